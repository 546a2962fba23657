"""Dev: point / line drivers at edge-case grid sizes (8 .. 4096 intervals)."""
import sys; sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2008_03276_b200.ehl import EhlParams, PointContact, LineContactBatch, moes_convert, solve_ehl
from paper_2008_03276_b200.errors import NonConvergenceError, PaqifError
for n in (8, 9, 33, 50, 100):
    try:
        pc = PointContact(EhlParams.point_from_moes(100.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0), n)
        for _ in range(3): pc.step()
        print("point", n, "ok", pc.status()[1])
        pc.close()
    except Exception as e:
        print("point", n, "ERR", type(e).__name__, e)
u_, w_ = moes_convert(m=20.0, l=10.0, g=5000.0)
p = EhlParams.line_from_loads(5000.0, u_, w_, domain=(-4.5, 1.5))
for n in (4, 5, 7, 33, 2048, 4096):
    try:
        b = LineContactBatch([p], n)
        for _ in range(2): b.step()
        print("line", n, "ok", float(b.res[0].item()))
    except Exception as e:
        print("line", n, "ERR", type(e).__name__, str(e)[:100])
