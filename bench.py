#!/usr/bin/env python
"""Benchmark: batched PAQIF banded-LCP solve (BASELINE.json configs[1]).

Workload (per GPU, weak scaling): 4096 independent banded LCPs, n = 1025
(padded to 1026 with a pinned identity row), semibandwidth 8, seeded
synthetic inputs (paper_2008_03276_b200/workloads.py).  One "step" = one
fused-kernel launch that runs the reference's whole projected active-set
solve paqif_solve_lcp(r=1) on every system of the batch (2-4 factor + W + Z
passes each).  Rank r solves systems [4096 r, 4096 (r+1)) -- no collective on
the data path; NCCL only carries the max-over-ranks timing.

    python bench.py [--gpus N --steps K --warmup W] [--impl b200|reference] [--exact]

--gpus N > 1 without WORLD_SIZE in the environment re-launches itself under
torch.distributed.run (one rank per GPU, rendezvous on 127.0.0.1); under a
launcher WORLD_SIZE must equal N.

Prints ONE JSON line (rank 0).  Timing: CUDA events on the launching stream,
barrier + synchronize on both sides, max over ranks; inputs (571 MB of bands
per GPU) exceed the 126 MB L2, so no explicit flush is needed.
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import tempfile
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_ROWS = 1025          # unpadded order of one LCP (rows solved)
N_PAD = 1026
BETA = 8
B_PER_GPU = 4096
SEED = 2024
# algorithmic bytes per LCP: band (2beta+1)*n + f + u, float64
BYTES_PER_LCP = ((2 * BETA + 1) * N_ROWS + N_ROWS + N_ROWS) * 8
METRIC = "PAQIF banded-LCP rows solved/s"
UNIT = "rows/s"


def load_peaks():
    peaks = {"hbm_gbs": 6551.4, "src": "fallback"}
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as fh:
            d = json.load(fh)
        peaks["hbm_gbs"] = float(d.get("hbm_gbs", peaks["hbm_gbs"]))
        peaks["src"] = "MEASURED_PEAKS.json"
    peaks["fp64_tflops"] = 33.94  # DFMA microbenchmark, profiles/peaks_r01.json
    peaks["fp64_src"] = "tools/peaks.cu DFMA microbenchmark (fallback constant)"
    p2 = os.path.join(ROOT, "profiles", "peaks_r01.json")
    if os.path.exists(p2):
        with open(p2) as fh:
            peaks["fp64_tflops"] = float(json.load(fh)["dfma_tflops"])
        peaks["fp64_src"] = "tools/peaks.cu DFMA microbenchmark (profiles/peaks_r01.json)"
    return peaks


def ncu_traffic():
    """DRAM bytes per launch of the LCP kernel from the committed ncu capture."""
    p = os.path.join(ROOT, "profiles", "lcp_ncu_summary.json")
    if not os.path.exists(p):
        return None, None
    with open(p) as fh:
        d = json.load(fh)
    return d.get("dram_bytes_per_launch"), d.get("systems_per_launch")


class ClockSampler:
    """nvidia-smi clocks/throttle reasons sampled every 200 ms during the
    timed region (B200_PROFILING.md clocks line)."""

    def __init__(self, index: int):
        self.index = index
        self.proc = None
        self.path = None

    def __enter__(self):
        fd, self.path = tempfile.mkstemp(suffix=".csv")
        os.close(fd)
        q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
             "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
             "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--id={self.index}", f"--query-gpu={q}",
                 "--format=csv,noheader,nounits", "-lms", "200"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except OSError:
            self.proc = None
        time.sleep(0.3)
        return self

    def __exit__(self, *exc):
        if self.proc is not None:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        out = {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        try:
            lines = [l.strip() for l in open(self.path) if l.strip()]
        except OSError:
            return out
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for l in lines:
            f = [x.strip() for x in l.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                mx = float(f[2])
            except ValueError:
                continue
            for name, v in zip(names, f[5:9]):
                if v.lower() == "active":
                    reasons.add(name)
        if sm:
            out["sm_mhz"] = statistics.median(sm)
            out["sm_max_mhz"] = mx
            out["samples"] = len(sm)
        out["reasons"] = sorted(reasons)
        return out


def cpu_threads():
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


def cpu_reference_rate(bands, f, threads: int, min_core_seconds: float = 10.0):
    """The reference algorithm's CPU path (the C oracle port of
    paqif_solve_lcp(r=1), oracle/paqif_oracle.c) on the given config-2
    systems with `threads` host threads, repeated until at least
    `min_core_seconds` of CPU work.  Returns (rows/s, wall s, reps)."""
    import oracle
    reps, wall = 0, 0.0
    while reps == 0 or wall * threads < min_core_seconds:
        t0 = time.perf_counter()
        oracle.lcp_batch(bands, f, threads=threads)
        wall += time.perf_counter() - t0
        reps += 1
    return reps * bands.shape[0] * N_ROWS / wall, wall, reps


def _line_params(m, l):
    from paper_2008_03276_b200.ehl import EhlParams, moes_convert
    u, w = moes_convert(m=m, l=l, g=5000.0)
    return EhlParams.line_from_loads(5000.0, u, w, domain=(-4.5, 1.5))


def config3_cases(rank, count=1024, seed=SEED):
    """Config 3 load sweep: M log-uniform on [5, 200], L uniform on [5, 15];
    case c drawn from default_rng((seed, 3, c)) so shards are rank-invariant."""
    import numpy as np
    out = []
    for c in range(rank * count, (rank + 1) * count):
        g = np.random.default_rng((seed, 3, c))
        m = float(np.exp(g.uniform(np.log(5.0), np.log(200.0))))
        out.append((m, float(g.uniform(5.0, 15.0))))
    return out


def config3_flops(n_int=1024):
    """Algorithmic fp64 work of one config-3 case-iteration:
    two N x N direct deformation convolutions (2 flop per MAC), one beta=2
    AQIF factor + W + Z (the paper's CostModel count), ~200 flop per node
    twice (rheology, faces, assembly, residual)."""
    from paper_2008_03276_b200.parallel import CostModel
    n = n_int + 1
    return 2 * 2 * n * n + CostModel(n_int, 2, 1).serial_total() + 2 * 200 * n


def _c3_cpu_worker(job):
    """One host core: oracle line steps of config-3 case `c` for ~`secs`."""
    c, m, l, secs = job
    import oracle.ehl_oracle as E
    p = _line_params(m, l)
    case = E.LineCase(p_hertz=p.p_hertz, lam=p.lam)
    film = E.LineFilm(1024, case)
    u, h0 = E.hertz_start(case, film), case.h0
    t0 = time.perf_counter()
    k = 0
    while k < 3 or time.perf_counter() - t0 < secs:
        u, h0, _, _, _ = E.line_step(u, h0, k, case, film)
        k += 1
    return k, time.perf_counter() - t0


def config3_cpu_pool(cases, threads, secs=4.0):
    """Config-3 CPU baseline: a process pool over all host cores, each
    worker running the numpy oracle's line steps on its own case (BLAS /
    OpenMP threads pinned to 1 per worker).  Returns (case-iters/s, sample)."""
    import multiprocessing as mp
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS"):
        os.environ[v] = "1"
    jobs = [(c, m, l, secs) for c, (m, l) in enumerate(cases[:threads])]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(threads) as pool:
        res = pool.map(_c3_cpu_worker, jobs)
    wall = time.perf_counter() - t0
    steps = sum(k for k, _ in res)
    busy = max(t for _, t in res)
    return steps / busy, (f"{len(jobs)} cases x ~{secs:.0f} s of oracle line steps, one per "
                          f"process ({steps} case-iterations, {wall:.1f} s wall incl. start-up)")


def ehl_secondary(rank, world, with_cpu, max_over_ranks, barrier, steps1=200, steps3=5,
                  point_steps=(3, 1)):
    """EHL Newton-step throughput: config 1 (one line contact, N=513) and
    config 3 (1024 line contacts per GPU, N=1025), device-timed per outer
    iteration, plus the oracle CPU rate on this host.  With several ranks
    only the sharded config 3 runs (configs 1/4/5 and the TVD line are
    single-GPU workloads: replicas only)."""
    import numpy as np
    import torch
    from paper_2008_03276_b200.ehl import LineContactBatch
    out = {}
    stream = torch.cuda.current_stream()
    peaks = load_peaks()

    def timed(batch, k):
        for _ in range(3):
            batch.step()
        barrier()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(k):
            batch.step()
        e1.record(stream)
        e1.synchronize()
        return max_over_ranks(e0.elapsed_time(e1) / k)

    p1 = _line_params(20.0, 10.0)
    if world == 1:
        ms1 = timed(LineContactBatch([p1], 512), steps1)
        ms1f = timed(LineContactBatch([p1], 512, exact=False), steps1)
        out["config1"] = {"metric": "EHL Newton iters/s (line, N=513, M=20, L=10, B=1)",
                          "value": 1e3 / ms1, "unit": "iters/s", "us_per_iter": ms1 * 1e3,
                          "gpu_launches_per_iter": 1,
                          "fma": {"us_per_iter": ms1f * 1e3, "value": 1e3 / ms1f}}
        # end to end through the public solve_ehl (device-side stop tests, one
        # host synchronisation per 32 iterations; initial state uploaded, final
        # state read back inside the timed region)
        from paper_2008_03276_b200.ehl import solve_ehl
        from paper_2008_03276_b200.errors import NonConvergenceError
        k_e2e = max(steps1, 64)
        for rep in range(2):  # first call warms the caches
            t0 = time.perf_counter()
            try:
                solve_ehl(p1, 512, tol=0.0, tol_fb=0.0, max_outer=k_e2e)
            except NonConvergenceError:
                pass
            dt = time.perf_counter() - t0
        out["config1"]["e2e"] = {"value": k_e2e / dt, "unit": "iters/s",
                                 "path": f"solve_ehl(max_outer={k_e2e}), device-side stop tests",
                                 "h2d_bytes": 513 * 8 * 2, "d2h_bytes": 513 * 8 + 48}
    cases = config3_cases(rank)
    b3 = LineContactBatch([_line_params(m, l) for m, l in cases], 1024)
    ms3 = timed(b3, steps3)
    info = b3.info.cpu().numpy()
    ms3f = timed(LineContactBatch([_line_params(m, l) for m, l in cases], 1024, exact=False),
                 steps3)
    # the fused one-CTA-per-case kernel on the same batch, for comparison
    ms3_fused = timed(LineContactBatch([_line_params(m, l) for m, l in cases], 1024,
                                       path="fused"), steps3)
    fl3 = config3_flops()
    tf3 = len(cases) * fl3 / (ms3 * 1e-3) / 1e12
    tf3f = len(cases) * fl3 / (ms3f * 1e-3) / 1e12
    out["config3"] = {"metric": "EHL line-contact case-iterations/s (1024 cases/GPU, N=1025)",
                      "value": world * len(cases) * 1e3 / ms3, "unit": "case-iters/s",
                      "ms_per_iter": ms3, "scaling": "weak", "n_gpus": world,
                      "path": "split (phase A / batched rung solves / phase C)",
                      "fused_path_ms_per_iter": ms3_fused,
                      "gpu_launches_per_iter": 3,
                      "ladder_cases_last_iter": int(np.sum((info & 3) > 0)),
                      "roofline": {"bound": "fp64", "achieved": tf3,
                                   "peak": peaks["fp64_tflops"], "unit": "TFLOP/s",
                                   "frac": tf3 / peaks["fp64_tflops"],
                                   "flops_per_case_iter": fl3,
                                   "count": "2 N^2-MAC deformations + CostModel(1024,2,1) "
                                            "+ 400 flop/node (SURVEY.md 8(d))",
                                   "peak_src": peaks["fp64_src"]},
                      "fma": {"ms_per_iter": ms3f, "value": world * len(cases) * 1e3 / ms3f,
                              "roofline_frac": tf3f / peaks["fp64_tflops"]}}
    if with_cpu:
        import oracle.ehl_oracle as E
        c = E.LineCase(p_hertz=p1.p_hertz, lam=p1.lam)
        f = E.LineFilm(512, c)
        u, h0 = E.hertz_start(c, f), c.h0
        t0 = time.perf_counter()
        k = 0
        while k < 20 or time.perf_counter() - t0 < 3.0:
            u, h0, _, _, _ = E.line_step(u, h0, k, c, f)
            k += 1
        dt = (time.perf_counter() - t0) / k
        out["config1"]["cpu_baseline"] = {"value": 1.0 / dt, "unit": "iters/s", "cores": 1,
                                          "kind": "port",
                                          "sample": f"{k} oracle line steps (numpy restatement)"}
        threads = cpu_threads()
        rate, sample = config3_cpu_pool(cases, threads)
        out["config3"]["cpu_baseline"] = {"value": rate, "unit": "case-iters/s",
                                          "cores": threads, "kind": "port", "sample": sample}
    out.update(point_secondary(with_cpu, steps4=point_steps[0], steps5=point_steps[1],
                               world=world, max_over_ranks=max_over_ranks, barrier=barrier))
    for v in out.values():
        v["arith"] = "exact (reference rounding); 'fma' = FMA arithmetic (within 1e-9)"
    if world == 1:
        out["tvd"] = tvd_secondary()
    return out


def tvd_secondary(intervals=256, sweeps=4):
    """TVD linear study: Ls1 x-line sweeps of the
    manufactured quartic problem (kappa = 1/3), solve_by_sweeps on the
    device (csrc/tvd_sweep.cu), device-timed; bit-exact iterates."""
    import torch
    from paper_2008_03276_b200.tvdcd import KappaSchemeConfig, quartic_test_problem, solve_by_sweeps
    prob, _ = quartic_test_problem(intervals, KappaSchemeConfig(kappa=1.0 / 3.0, eps=1e-6))
    solve_by_sweeps(prob, "Ls1", tol=0.0, max_sweeps=1, cycle="x")
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    e0.record()
    _, hist = solve_by_sweeps(prob, "Ls1", tol=0.0, max_sweeps=sweeps, cycle="x")
    e1.record()
    e1.synchronize()
    ms = e0.elapsed_time(e1) / sweeps
    return {"metric": "TVD Ls1 x-line sweeps/s (quartic problem, kappa=1/3)",
            "value": 1e3 / ms, "unit": "sweeps/s", "ms_per_sweep": ms,
            "intervals": intervals, "lines_per_sweep": prob.grid.ny,
            "residual_last": hist[-1], "arith": "exact (reference rounding)"}


def fold_bytes(n):
    """Algorithmic HBM bytes of one full point deformation (the fold): read
    the pressure, write the deformation, read the kernel spectrum once
    ((P/2+1) x P complex, P = next power of two >= 2n)."""
    P = 32
    while P < 2 * n:
        P *= 2
    N = n + 1
    return 2 * N * N * 8 + (P // 2 + 1) * P * 16, P


def point_secondary(with_cpu, steps4=3, steps5=1, world=1, max_over_ranks=None, barrier=None):
    """EHL point contact, one outer iteration of solve_ehl per step through
    the native sweep driver (csrc/ehl_point.cu): config 4 (513^2, M=100) and
    config 5 (2049^2, M=1000), device-timed on the handle's stream; plus the
    full deformation (fold) alone with its HBM roofline fraction.  With
    several ranks only config 5 runs: every rank the same contact, each fold
    split over the ranks (PointContact.shard_folds, csrc/fft_shard.cuh)."""
    import torch
    from paper_2008_03276_b200.ehl import EhlParams, PointContact
    out = {}
    mor = max_over_ranks or (lambda x: x)
    bar = barrier or (lambda: None)
    peaks = load_peaks()

    def run(n, m, steps, warm, exact=True, shard=False, fold_reps=0):
        p = EhlParams.point_from_moes(m, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
        pc = PointContact(p, n, exact=exact)
        if shard:
            pc.shard_folds()
        stream = torch.cuda.ExternalStream(pc.stream_handle())
        for _ in range(warm):
            pc.step()
        pc.sync()
        bar()
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(steps):
            pc.step()
        e1.record(stream)
        e1.synchronize()
        ms = mor(e0.elapsed_time(e1) / steps)
        fold_ms = None
        if fold_reps:
            pc.fold_bench(2)
            pc.sync()
            bar()
            e0.record(stream)
            pc.fold_bench(fold_reps)
            e1.record(stream)
            e1.synchronize()
            fold_ms = mor(e0.elapsed_time(e1) / fold_reps)
        snap = pc.snapshot()
        pc.close()
        return ms, snap, fold_ms

    def fold_line(n, fold_ms):
        b, P = fold_bytes(n)
        gbs = b / (fold_ms * 1e-3) / 1e9
        return {"ms": fold_ms, "period": P, "algorithmic_bytes": b,
                "roofline": {"bound": "hbm", "achieved": gbs, "peak": peaks["hbm_gbs"],
                             "unit": "GB/s", "frac": gbs / peaks["hbm_gbs"]}}

    if steps4 > 0 and world == 1:
        ms4, s4, f4 = run(512, 100.0, steps4, 3, fold_reps=20)
        out["config4"] = {"metric": "EHL point Newton iters/s (513x513, M=100, L=10)",
                          "value": 1e3 / ms4, "unit": "iters/s", "ms_per_iter": ms4,
                          "lines_per_iter": 2 * 511, "newton_x_lines_last": int(s4["newton"].sum()),
                          "residual_last": s4["res"], "fold": fold_line(512, f4)}
        ms4f, s4f, _ = run(512, 100.0, steps4, 3, exact=False)
        out["config4"]["fma"] = {"ms_per_iter": ms4f, "value": 1e3 / ms4f,
                                 "newton_x_lines_last": int(s4f["newton"].sum())}
        if with_cpu:
            import oracle.ehl_point_oracle as P
            c = P.point_case(100.0, 10.0)
            f = P.PointFilm(512, c)
            t0 = time.perf_counter()
            P.point_step(P.hertz_start(c, f), c.h0, 0, c, f)
            dt = time.perf_counter() - t0
            out["config4"]["cpu_baseline"] = {"value": 1.0 / dt, "unit": "iters/s", "cores": 1,
                                              "kind": "port",
                                              "sample": "1 oracle point iteration (numpy/scipy)"}
    if steps5 > 0:
        ms5, s5, f5 = run(2048, 1000.0, steps5, 1, shard=world > 1, fold_reps=10)
        out["config5"] = {"metric": "EHL point Newton iters/s (2049x2049, M=1000, L=10)",
                          "value": 1e3 / ms5, "unit": "iters/s", "ms_per_iter": ms5,
                          "n_gpus": world, "scaling": "strong",
                          "folds": "split over the ranks (fft_shard.cuh)" if world > 1
                                   else "one GPU",
                          "lines_per_iter": 2 * 2047, "residual_last": s5["res"],
                          "fold": fold_line(2048, f5)}
        if with_cpu:
            out["config5"]["cpu_baseline"] = config5_cpu_baseline()
    for v in out.values():
        v["arith"] = "exact (reference rounding); 'fma' = FMA arithmetic (within 1e-9)"
    return out


def config5_cpu_baseline(budget_s=30.0):
    """Config 5's CPU baseline: the numpy oracle's x-sweep lines from the
    adapted Hertz start on one host core for ~budget_s, scaled to a whole
    outer iteration (2 x 2047 line solves plus their folds) by the line
    count.  One full reference iteration takes ~10 min on one core
    (SURVEY.md 6.3), too long for a bench run; the sample is named."""
    import oracle.ehl_point_oracle as P
    c = P.point_case(1000.0, 10.0)
    t0 = time.perf_counter()
    f = P.PointFilm(2048, c)
    u = P.hertz_start(c, f)
    f.deformation_full(u)
    setup = time.perf_counter() - t0
    t0 = time.perf_counter()
    lines = P.x_sweep_lines(u, c.h0, c, f, budget_s)
    dt = time.perf_counter() - t0
    per_line = dt / max(lines, 1)
    iter_s = per_line * 2 * 2047
    return {"value": 1.0 / iter_s, "unit": "iters/s", "cores": 1, "kind": "port",
            "sample": f"{lines} oracle x-sweep lines of the first iteration in {dt:.1f} s "
                      f"(+{setup:.1f} s set-up), scaled by 4094 lines per iteration"}


def shard_inputs(rank, B):
    """Rank r's config-2 shard: systems [r B, (r+1) B) of the rank-invariant
    seeded stream (workloads.lcp_batch draws system b from its own seed)."""
    from paper_2008_03276_b200.workloads import lcp_batch
    return lcp_batch(SEED, B, start=rank * B)


def make_max_over_ranks(dist, device):
    """max over ranks of a per-rank float (the device-timed step time):
    identity with one rank, an all_reduce(MAX) otherwise."""
    def max_over_ranks(x: float) -> float:
        if dist is None:
            return x
        import torch
        t = torch.tensor([x], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())
    return max_over_ranks


def headline_config(B):
    """The config dict of the headline line -- identical in both arms, so
    the driver can tell they ran the same workload."""
    return {"workload": "config2: banded LCP batch (4096 systems/GPU), n=1025 (pad 1026), "
                        "beta=8, paqif_solve_lcp(r=1) semantics",
            "systems_per_gpu": B, "n": N_ROWS, "beta": BETA, "seed": SEED,
            "generator": "workloads.lcp_batch(seed, B, start=rank*B)",
            "l2": "inputs larger than L2 (571 MB/GPU), no flush needed"}


def _ref_numba_worker(job):
    """One host core: the UNMODIFIED reference (baseline/_ref, numba) solving
    config-2 systems with paqif_solve_lcp(LcpProblem(L, f), r=1) for about
    `secs` after a JIT warm-up."""
    lo, hi, secs = job
    sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
    from paqif.bandcore import BandedMatrix
    from paqif.lcp import LcpProblem
    from paqif.parallel import paqif_solve_lcp
    from paper_2008_03276_b200.workloads import lcp_batch
    bands, f = lcp_batch(SEED, hi - lo, start=lo)
    solve = lambda b: paqif_solve_lcp(LcpProblem(BandedMatrix(N_PAD, BETA, bands[b]), f[b]), 1)
    solve(0)  # JIT compile / cache load
    t0 = time.perf_counter()
    k = 0
    while k < 1 or (time.perf_counter() - t0 < secs and k < hi - lo):
        solve(k)
        k += 1
    return k, time.perf_counter() - t0


def reference_code_rate(threads, secs=6.0):
    """Config 2 through the reference's own code (baseline/_ref, numba),
    one process per host core on its own slice of the batch.  None when
    baseline/_ref is absent."""
    if not os.path.isdir(os.path.join(ROOT, "baseline", "_ref", "paqif")):
        return None
    import multiprocessing as mp
    for v in ("OMP_NUM_THREADS", "OPENBLAS_NUM_THREADS", "MKL_NUM_THREADS", "NUMBA_NUM_THREADS"):
        os.environ[v] = "1"
    os.environ.setdefault("NUMBA_CACHE_DIR", tempfile.mkdtemp(prefix="numba_"))
    per = 256
    jobs = [(w * per, (w + 1) * per, secs) for w in range(threads)]
    t0 = time.perf_counter()
    with mp.get_context("spawn").Pool(threads) as pool:
        res = pool.map(_ref_numba_worker, jobs)
    wall = time.perf_counter() - t0
    solved = sum(k for k, _ in res)
    busy = max(t for _, t in res)
    return {"value": solved * N_ROWS / busy, "unit": UNIT, "cores": threads, "kind": "reference",
            "sample": f"{solved} config-2 systems through baseline/_ref paqif_solve_lcp(r=1) "
                      f"(numba), {threads} processes x ~{secs:.0f} s ({wall:.1f} s wall incl. "
                      f"JIT warm-up)"}


def relaunch_distributed(args) -> int:
    """--gpus N > 1 with no launcher: run this script under
    torch.distributed.run, one rank per GPU, and return its exit code."""
    import socket
    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr=127.0.0.1",
           f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def run_reference(args, rank, world):
    """--impl reference: the reference's CPU implementation of the path
    (oracle port, all host threads), rank 0 only."""
    if rank != 0:
        return
    import oracle
    from paper_2008_03276_b200.workloads import lcp_batch
    threads = cpu_threads()
    sample = B_PER_GPU  # one step = the same 4096-system batch the GPU step solves
    bands, f = lcp_batch(SEED, sample)
    for _ in range(args.warmup):
        oracle.lcp_batch(bands[:64], f[:64], threads=threads)
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        oracle.lcp_batch(bands, f, threads=threads)
        times.append(time.perf_counter() - t0)
    ms = 1e3 * sum(times) / len(times)
    value = sample * N_ROWS / (sum(times) / len(times))
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded, workloads.lcp_batch)",
        "config": headline_config(sample),
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads, "kind": "port",
                         "sample": f"{sample} config-2 systems per step (oracle/paqif_oracle.c "
                                   f"restating paqif_solve_lcp r=1), {threads} host threads"},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    # beside the port: the reference's own numba code path on the same cores
    ref_code = None if args.no_ref_code else reference_code_rate(threads)
    if ref_code is not None:
        line["reference_code"] = ref_code
    print(json.dumps(line), flush=True)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--exact", action="store_true",
                    help="headline in exact arithmetic (reference rounding, bit-exact vs the "
                         "oracle); default FMA arithmetic (within 1e-9, same passes/active sets)")
    ap.add_argument("--batch", type=int, default=B_PER_GPU)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-ehl", action="store_true", help="skip the config-1/3/4/5 EHL lines")
    ap.add_argument("--no-point", action="store_true", help="skip the config-4/5 point lines")
    ap.add_argument("--no-ref-code", action="store_true",
                    help="reference arm: skip timing the reference's numba code (baseline/_ref)")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)

    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        raise SystemExit(relaunch_distributed(args))
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    if args.impl == "reference":
        run_reference(args, rank, world)
        return

    import numpy as np
    import torch
    torch.cuda.set_device(local)
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))

    from paper_2008_03276_b200 import _native
    from paper_2008_03276_b200.batch import LcpSolver

    B = args.batch
    exact = args.exact
    bands_h, f_h = shard_inputs(rank, B)
    # pinned host copies: the e2e path reads these every step
    bands_pin = torch.from_numpy(bands_h).pin_memory()
    f_pin = torch.from_numpy(f_h).pin_memory()
    bands = bands_pin.to("cuda", non_blocking=True)
    f = f_pin.to("cuda", non_blocking=True)
    solver = LcpSolver(B, N_PAD, BETA, exact)
    stream = torch.cuda.current_stream()

    def barrier():
        torch.cuda.synchronize()
        if dist is not None:
            dist.barrier()
        torch.cuda.synchronize()

    max_over_ranks = make_max_over_ranks(dist, "cuda")

    for _ in range(args.warmup):
        solver.launch(bands, f)
    barrier()
    with ClockSampler(local) as clocks:
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        for _ in range(args.steps):
            solver.launch(bands, f)
        e1.record(stream)
        e1.synchronize()
        barrier()
    ms_step = max_over_ranks(e0.elapsed_time(e1) / args.steps)
    status = solver.status.cpu().numpy()
    passes = solver.passes.cpu().numpy()
    if np.any(status != 0):
        raise SystemExit(f"LCP status != 0 on {int(np.sum(status != 0))} systems")
    value = world * B * N_ROWS / (ms_step * 1e-3)

    # ---- the other arithmetic mode on the same batch: throughput + parity
    other = LcpSolver(B, N_PAD, BETA, not exact)
    other.launch(bands, f)
    torch.cuda.synchronize()
    o0 = torch.cuda.Event(enable_timing=True)
    o1 = torch.cuda.Event(enable_timing=True)
    o0.record(stream)
    for _ in range(3):
        other.launch(bands, f)
    o1.record(stream)
    o1.synchronize()
    ms_other = max_over_ranks(o0.elapsed_time(o1) / 3)
    ue, uf = (solver.u, other.u) if exact else (other.u, solver.u)
    scale = torch.clamp(ue.abs().amax(dim=1, keepdim=True), min=1.0)
    parity = {"max_rel_diff": float(((uf - ue).abs() / scale).max().item()),
              "same_passes": bool(torch.equal(solver.passes, other.passes)),
              "same_active_sets": bool(torch.equal(solver.active, other.active)),
              "systems": B}
    other_line = {"arith": "fma" if exact else "exact (bit-exact vs oracle)",
                  "ms_per_step": ms_other, "value": world * B * N_ROWS / (ms_other * 1e-3),
                  "parity_fma_vs_exact": parity}
    del other

    # ---- end to end through the C-ABI host entry (pinned host buffers in/out)
    L = _native.lib()
    u_h = torch.empty((B, N_PAD), dtype=torch.float64).pin_memory()
    a_h = torch.empty((B, N_PAD), dtype=torch.uint8).pin_memory()
    p_h = torch.empty(B, dtype=torch.int64).pin_memory()
    r_h = torch.empty(B, dtype=torch.float64).pin_memory()
    s_h = torch.empty(B, dtype=torch.int64).pin_memory()

    def host_call():
        rc = L.paqif_lcp_batch_host(B, N_PAD, BETA, bands_pin.data_ptr(), f_pin.data_ptr(),
                                    1e-10, 100, _native.FLAG_EXACT if exact else 0,
                                    u_h.data_ptr(), a_h.data_ptr(), p_h.data_ptr(),
                                    r_h.data_ptr(), s_h.data_ptr())
        _native.check(rc, "paqif_lcp_batch_host")

    host_call()
    barrier()
    t0 = time.perf_counter()
    e2e_steps = max(1, min(args.steps, 5))
    for _ in range(e2e_steps):
        host_call()
    barrier()
    e2e_s = max_over_ranks((time.perf_counter() - t0) / e2e_steps)
    e2e_value = world * B * N_ROWS / e2e_s
    if not np.array_equal(u_h.numpy(), solver.u.cpu().numpy()):
        raise SystemExit("host-entry result differs from device-entry result")
    h2d = bands_h.nbytes + f_h.nbytes
    d2h = u_h.numel() * 8 + a_h.numel() + 3 * B * 8

    # ---- roofline of the dominant (only) kernel
    peaks = load_peaks()
    achieved_gbs = B * BYTES_PER_LCP / (ms_step * 1e-3) / 1e9
    traffic, traffic_b = ncu_traffic()
    if traffic is not None and traffic_b:
        traffic = traffic * B / traffic_b
    from paper_2008_03276_b200.parallel import CostModel
    flops_pass = CostModel(N_PAD, BETA, 1).serial_total()  # paper's op count, one pass
    fp64_tflops = B * float(np.mean(passes)) * flops_pass / (ms_step * 1e-3) / 1e12
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded per system, workloads.lcp_batch; inputs 571 MB/GPU > L2, "
                "no flush needed)",
        "config": headline_config(B),
        "arith": "exact (reference rounding, bit-exact vs oracle)" if exact
                 else "fma (within 1e-9 of exact; same passes and active sets, see "
                      "other_arith.parity_fma_vs_exact)",
        "mean_passes": float(np.mean(passes)),
        "gpu_launches": args.steps,
        "e2e": {"value": e2e_value, "unit": UNIT, "h2d_bytes_per_step": int(h2d),
                "d2h_bytes_per_step": int(d2h),
                "path": "C ABI paqif_lcp_batch_host, pinned host buffers"},
        "roofline": {"bound": "hbm", "achieved": achieved_gbs, "peak": peaks["hbm_gbs"],
                     "unit": "GB/s", "frac": achieved_gbs / peaks["hbm_gbs"],
                     "traffic": traffic,
                     "peak_src": peaks["src"],
                     "algorithmic_bytes_per_launch": B * BYTES_PER_LCP},
        "fp64": {"achieved_tflops": fp64_tflops, "peak_tflops": peaks["fp64_tflops"],
                 "frac": fp64_tflops / peaks["fp64_tflops"],
                 "count": "CostModel(1026,8,1).serial_total() per pass x mean passes",
                 "peak_src": "tools/peaks.cu DFMA microbenchmark (profiles/peaks_r01.json)"},
        "clocks": clocks.summary(),
        "other_arith": other_line,
    }
    if not args.no_ehl:
        line["secondary"] = ehl_secondary(rank, world, with_cpu=(rank == 0 and world == 1
                                                                  and not args.no_cpu_baseline),
                                          max_over_ranks=max_over_ranks, barrier=barrier,
                                          point_steps=(0, 0) if args.no_point else (3, 1))
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        threads = cpu_threads()
        sample = 1024
        rate, secs, reps = cpu_reference_rate(bands_h[:sample], f_h[:sample], threads)
        line["cpu_baseline"] = {"value": rate, "unit": UNIT, "cores": threads, "kind": "port",
                                "sample": f"first {sample} systems of the GPU batch x {reps}, "
                                          f"oracle/paqif_oracle.c (C restatement of "
                                          f"paqif_solve_lcp r=1), {secs:.1f} s wall"}
    if rank == 0:
        print(json.dumps(line), flush=True)
    if dist is not None:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
