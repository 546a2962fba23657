"""Dev: point-contact debugging helper (one step, dumps of device state)."""
import sys, time, numpy as np
sys.path.insert(0, '/root/repo')
from paper_2008_03276_b200.ehl import EhlParams, PointContact
import oracle.ehl_point_oracle as P
for n in (128, 256, 512):
    p = EhlParams.point_from_moes(100.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
    c = P.point_case(100.0, 10.0); f = P.PointFilm(n, c)
    u0 = P.hertz_start(c, f)
    t = time.time(); ur, h0r, fr, rr, info = P.point_step(u0, c.h0, 0, c, f); t = time.time() - t
    for exact in (True, False):
        pc = PointContact(p, n, exact=exact); pc.step(); s = pc.snapshot()
        err = np.max(np.abs(s['u'] - ur)) / np.max(np.abs(ur))
        xr = [ {'scheme':0,'first-order':1,'diagonal':2}[r] for r in info['x_rungs']]
        print(n, exact, 'rel err', err, 'res', s['res'], rr, 'xr mism', int(np.sum(np.array(xr) != s['x_rungs'])),
              'yr>0', int((s['y_rungs']>0).sum()), 'oracle y>0', sum(1 for r in info['y_rungs'] if r != 'scheme'), 'oracle s', round(t,1), flush=True)
