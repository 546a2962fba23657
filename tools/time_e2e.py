"""Dev: the headline end-to-end path (paqif_lcp_batch_host, pinned host
buffers, H2D + solve + D2H per step) on the config-2 batch."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_03276_b200 import _native
from paper_2008_03276_b200.workloads import lcp_batch as gen
B = 4096
bands, f = gen(2024, B)
n, beta = bands.shape[2], (bands.shape[1] - 1) // 2
bp = torch.from_numpy(bands).pin_memory(); fp = torch.from_numpy(f).pin_memory()
u = torch.empty((B, n), dtype=torch.float64).pin_memory(); a = torch.empty((B, n), dtype=torch.uint8).pin_memory()
p = torch.empty(B, dtype=torch.int64).pin_memory(); r = torch.empty(B, dtype=torch.float64).pin_memory()
s = torch.empty(B, dtype=torch.int64).pin_memory()
L = _native.lib()
def run():
    _native.check(L.paqif_lcp_batch_host(B, n, beta, bp.data_ptr(), fp.data_ptr(), 1e-10, 100, 0, u.data_ptr(),
                                         a.data_ptr(), p.data_ptr(), r.data_ptr(), s.data_ptr()), "host")
for _ in range(3): run()
t0 = time.perf_counter()
for _ in range(10): run()
dt = (time.perf_counter() - t0) / 10
print(f"e2e {dt*1e3:.2f} ms/step, {B*1025/dt:.3e} rows/s")
