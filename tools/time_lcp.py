"""Quick timing of the fused LCP kernel on the config-2 workload (dev tool)."""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_03276_b200.batch import LcpSolver
from paper_2008_03276_b200.workloads import lcp_batch as gen

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
t0 = time.time(); bands, f = gen(2024, B); print("gen", time.time() - t0, flush=True)
tb = torch.from_numpy(bands).cuda(); tf = torch.from_numpy(f).cuda()
for exact in (True, False):
    s = LcpSolver(B, 1026, 8, exact)
    for _ in range(2): s.launch(tb, tf)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5): s.launch(tb, tf)
    e1.record(); torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 5
    print(f"exact={exact} B={B} ms={ms:.3f} rows/s={B*1025/(ms*1e-3):.3e} "
          f"GB/s={B*155800/(ms*1e-3)/1e9:.1f} passes_mean={s.passes.double().mean().item():.3f} "
          f"status_max={int(s.status.max())} ws_MB={s.ws_bytes/1e6:.0f}", flush=True)
    pa = s.passes.cpu().numpy()
    print("  passes histogram", dict(zip(*np.unique(pa, return_counts=True))), flush=True)
    for bb in (64, 512, 1024, 2048):
        sb = LcpSolver(bb, 1026, 8, exact)
        sb.launch(tb[:bb], tf[:bb]); torch.cuda.synchronize()
        e0.record()
        for _ in range(3): sb.launch(tb[:bb], tf[:bb])
        e1.record(); torch.cuda.synchronize()
        print(f"  B={bb}: {e0.elapsed_time(e1)/3:.3f} ms, max passes {int(sb.passes.max())}", flush=True)
