"""One warm-up + one profiled launch of the fused LCP kernel (ncu target)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2008_03276_b200.batch import LcpSolver
from paper_2008_03276_b200.workloads import lcp_batch as gen

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
exact = (sys.argv[2] != "fast") if len(sys.argv) > 2 else True
bands, f = gen(2024, B)
tb, tf = torch.from_numpy(bands).cuda(), torch.from_numpy(f).cuda()
s = LcpSolver(B, 1026, 8, exact)
s.launch(tb, tf)
s.launch(tb, tf)
torch.cuda.synchronize()
print("ok", int(s.status.max()), float(s.passes.double().mean()))
