"""Dev: runs of deferred (weighted) x-lines per outer iteration and their stability."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2008_03276_b200.ehl import EhlParams, PointContact
for n, m in ((512, 100.0), (2048, 1000.0)):
    pc = PointContact(EhlParams.point_from_moes(m, 10.0, domain=(-4.5, 1.5), lo_y=-3.0), n)
    prev = None
    for it in range(4 if n == 512 else 2):
        pc.step()
        s = pc.snapshot()
        nw = np.asarray(s["newton"])
        runs = np.diff(np.concatenate([[0], (nw == 0).astype(int), [0]]))
        starts = np.where(runs == 1)[0]; ends = np.where(runs == -1)[0]
        same = None if prev is None else int(np.sum(prev != nw))
        print(n, it, "weighted", int(np.sum(nw == 0)), "runs", list(zip(starts.tolist(), ends.tolist()))[:6], "changed vs prev", same, flush=True)
        prev = nw
