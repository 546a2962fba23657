"""Dev: rows / columns of the point contact that stay all-zero or unchanged per step."""
import sys
sys.path.insert(0, "/root/repo")
import numpy as np
from paper_2008_03276_b200.ehl import EhlParams, PointContact
for n, m in ((512, 100.0), (2048, 1000.0)):
    pc = PointContact(EhlParams.point_from_moes(m, 10.0, domain=(-4.5, 1.5), lo_y=-3.0), n)
    for it in range(2):
        u0 = pc.snapshot()["u"]
        pc.step()
        u1 = pc.snapshot()["u"]
        rows_zero = np.all(u1 == 0, axis=1).sum(); cols_zero = np.all(u1 == 0, axis=0).sum()
        rows_same = np.all(u1 == u0, axis=1).sum(); cols_same = np.all(u1 == u0, axis=0).sum()
        print(n, it, "rows all-zero", rows_zero, "cols all-zero", cols_zero, "rows unchanged", rows_same, "cols unchanged", cols_same, flush=True)
