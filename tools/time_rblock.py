"""Dev: one batched PAQIF solve (paqif_solve(L_b, f_b, r), all seven steps on
the device, csrc/rblock.cu) of the 4096 config-2 systems for several r, next
to the fused r=1 solve (solve-only LCP kernel)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2008_03276_b200 import _native
from paper_2008_03276_b200.batch import LcpSolver
from paper_2008_03276_b200.workloads import lcp_batch as gen

B = int(sys.argv[1]) if len(sys.argv) > 1 else 4096
bands, f = gen(2024, B)
tb, tf = torch.from_numpy(bands).cuda(), torch.from_numpy(f).cuda()
n, beta = bands.shape[2], (bands.shape[1] - 1) // 2
L = _native.lib()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for exact in (False, True):
    s = LcpSolver(B, n, beta, exact)
    x1, _ = s.solve_r1(tb, tf)
    torch.cuda.synchronize()
    e0.record()
    for _ in range(3): s.solve_r1(tb, tf)
    e1.record(); torch.cuda.synchronize()
    ref = x1.clone()
    print(f"exact={exact} r=1 fused: {e0.elapsed_time(e1)/3:.3f} ms", flush=True)
    for r in (3, 9, 19, 27):
        nbytes = L.paqif_solve_rblock_workspace_bytes(B, n, beta, r)
        if nbytes == 0:
            print(f"  r={r}: unsupported"); continue
        ws = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
        x = torch.zeros((B, n), dtype=torch.float64, device="cuda")
        st = torch.zeros(B, dtype=torch.int64, device="cuda")
        run = lambda: L.paqif_solve_rblock_batch(B, n, beta, r, tb.data_ptr(), tf.data_ptr(), x.data_ptr(), 0,
                                                 st.data_ptr(), _native.FLAG_EXACT if exact else 0,
                                                 ws.data_ptr(), nbytes, _native.stream_ptr())
        _native.check(run(), "rblock")
        torch.cuda.synchronize()
        e0.record()
        for _ in range(3): run()
        e1.record(); torch.cuda.synchronize()
        rel = ((x - ref).abs().max() / ref.abs().max()).item()
        print(f"  r={r}: {e0.elapsed_time(e1)/3:.3f} ms, status max {int(st.max())}, max rel vs r=1 {rel:.2e}", flush=True)
