"""Host-side logic (no GPU): band storage, partitioning, cost model, kernel
tables and cache, parameter derivations, seeded workloads and the
multi-process sharding used by bench.py (gloo, world size 2)."""

import os
import socket

import numpy as np
import pytest

from paper_2008_03276_b200.bandcore import (BandedMatrix, band_matvec, cholesky_spd_solve,
                                            is_diagonally_dominant, project_nonneg)
from paper_2008_03276_b200.errors import (ContractViolationError, NotPositiveDefiniteError,
                                          PartitionError)
from paper_2008_03276_b200.parallel import CostModel, check_partition, predict_speedup
from paper_2008_03276_b200.workloads import lcp_batch, lcp_system, random_banded


class TestBandedMatrix:
    def test_entry_zero_outside_band(self, rng):
        a = BandedMatrix(12, 2, random_banded(12, 2, rng))
        for i in range(12):
            for j in range(12):
                if abs(i - j) > 2:
                    assert a.entry(i, j) == 0.0

    def test_dense_round_trip(self, rng):
        a = BandedMatrix(16, 3, random_banded(16, 3, rng))
        b = BandedMatrix.from_dense(a.to_dense(), 3)
        assert np.array_equal(a.bands, b.bands)

    def test_degenerate_order_rejected(self):
        with pytest.raises(ContractViolationError):
            BandedMatrix(2, 2)

    def test_matvec_matches_dense(self, rng):
        for n, beta in ((8, 1), (17, 2), (64, 3)):
            a = BandedMatrix(n, beta, random_banded(n, beta, rng, dominant=False))
            x = rng.standard_normal(n)
            np.testing.assert_allclose(band_matvec(a, x), a.to_dense() @ x, atol=1e-12)

    def test_dominance(self):
        assert is_diagonally_dominant(BandedMatrix.from_diagonals(8, {-1: -1.0, 0: 2.0, 1: -1.0}))
        assert not is_diagonally_dominant(
            BandedMatrix.from_diagonals(8, {-1: -1.0, 0: 1.5, 1: -1.0}))

    def test_projection(self, rng):
        x = rng.standard_normal(50)
        once = project_nonneg(x)
        assert np.all(once >= 0) and np.array_equal(project_nonneg(once), once)


def test_cholesky(rng):
    r = rng.standard_normal((8, 8)) + 4.0 * np.eye(8)
    a = r.T @ r
    b = rng.standard_normal(8)
    np.testing.assert_allclose(cholesky_spd_solve(a, b), np.linalg.solve(a, b), atol=1e-10)
    with pytest.raises(NotPositiveDefiniteError):
        cholesky_spd_solve(np.array([[1.0, 2.0], [2.0, 1.0]]), np.ones(2))


class TestPartition:
    """Block-split validation of paqif_solve(l, f, r): the reference's
    partition checks (parallel.py:106-125), same types, same order."""

    def test_block_size(self):
        assert check_partition(32, 2, 4) == 8
        assert check_partition(1026, 8, 1) == 1026

    def test_errors(self):
        with pytest.raises(PartitionError):
            check_partition(16, 2, 3)      # does not divide
        with pytest.raises(PartitionError):
            check_partition(16, 2, 4)      # t = 4 <= 2 beta
        with pytest.raises(PartitionError):
            check_partition(18, 1, 2)      # t = 9 odd
        with pytest.raises(PartitionError):
            check_partition(16, 2, 0)
        with pytest.raises(ContractViolationError):
            check_partition(16, 2, 2, rhs_len=15)

    def test_wide_band_rejected(self):
        """beta > 16 has no device engine: rejected before any compute (no
        host fallback)."""
        from paper_2008_03276_b200.parallel import paqif_solve, paqif_solve_lcp
        from paper_2008_03276_b200.lcp import LcpProblem
        l = BandedMatrix.identity(80, 17)
        with pytest.raises(ContractViolationError):
            paqif_solve(l, np.ones(80), 1)
        with pytest.raises(ContractViolationError):
            paqif_solve_lcp(LcpProblem(l, np.ones(80)), 1)


class TestCostModel:
    def test_speedup_formula(self):
        m = CostModel(512, 2, 4)
        assert predict_speedup(m) == pytest.approx(1.0 / (4.0 * (0.25 + (2.0 / 512.0) * 47.0)),
                                                   rel=1e-15)

    def test_counts_structure(self):
        c = CostModel(64, 2, 4)
        assert set(c.parallel_counts()) == {"fact", "y", "inv", "comp", "norm", "chol",
                                            "update", "sol"}
        # paper count used by bench.py's fp64 line
        assert CostModel(1026, 8, 1).serial_total() == pytest.approx(1.387e6, rel=1e-3)

    def test_serial_counts_closed_form(self):
        for n, b, r in ((64, 2, 1), (128, 3, 1), (256, 4, 2)):
            t = n // r
            got = CostModel(n, b, r).serial_counts()
            assert got["fact"] == (r * (t - 1) * (1 + 4 * b + 8 * b * b),
                                   r * (t - 1) * (2 + 8 * b + 8 * b * b), r * (t - 1) * 4 * b)
            assert got["norm"][0] == 36 * r * b ** 3 - 6 * r * b * b

    def test_invalid(self):
        with pytest.raises(ContractViolationError):
            CostModel(10, 2, 3)


class TestWorkloads:
    def test_config2_system_shape_and_dominance(self):
        bands, f = lcp_system(1, 0)
        assert bands.shape == (17, 1026) and f.shape == (1026,)
        assert bands[8, 1025] == 1.0 and f[1025] == 0.0
        assert np.all(bands[:, 1025][np.arange(17) != 8] == 0.0)
        a = BandedMatrix(1026, 8, bands)
        assert is_diagonally_dominant(a)
        off = np.abs(bands).sum(axis=0) - np.abs(bands[8])
        assert np.all(bands[8, :1025] - off[:1025] >= 0.1 - 1e-12)

    def test_shard_invariance(self):
        full_b, full_f = lcp_batch(5, 8, n=65, beta=8)
        part_b, part_f = lcp_batch(5, 4, n=65, beta=8, start=4)
        assert np.array_equal(full_b[4:], part_b) and np.array_equal(full_f[4:], part_f)

    def test_config3_cases_rank_invariant(self):
        import bench
        a = bench.config3_cases(0, count=8)
        b = bench.config3_cases(1, count=4)
        c = bench.config3_cases(0, count=12)
        assert a[4:] == b and c[:8] == a
        ms = np.array([m for m, _ in bench.config3_cases(0)])
        ls = np.array([l for _, l in bench.config3_cases(0)])
        assert ms.min() >= 5.0 and ms.max() <= 200.0 and ls.min() >= 5.0 and ls.max() <= 15.0


class TestEhlHost:
    def test_kernels_and_cache(self, tmp_path):
        from paper_2008_03276_b200.ehl import (kernel_line, kernel_point, load_kernel_cache,
                                               save_kernel_cache)
        kl = kernel_line(64, 0.05)
        assert kl.table.shape == (65,) and kl.table[0] < 0.0
        kp = kernel_point(8, 8, 0.1)
        assert kp.table.shape == (9, 9) and np.all(np.diff(kp.table[:, 0][1:]) <= 0.0)
        path = os.path.join(tmp_path, "k.npz")
        save_kernel_cache(path, kp)
        back = load_kernel_cache(path, "point", 0.1, 8, 8)
        assert back is not None and np.array_equal(back.table, kp.table)
        assert load_kernel_cache(path, "point", 0.2, 8, 8) is None
        assert load_kernel_cache(path, "line", 0.1, 8) is None

    def test_kernel_tables_vs_reference(self):
        # host tables bit-identical to the reference's (golden ehl_kernels.npz)
        from conftest import load_golden
        from paper_2008_03276_b200.ehl import kernel_line, kernel_point
        K = load_golden("ehl_kernels.npz")
        for k in (0, 1):
            t = kernel_line(int(K[f"line{k}_n"]), float(K[f"line{k}_h"])).table
            assert np.array_equal(t, K[f"line{k}_table"])
            t = kernel_point(int(K[f"point{k}_nx"]), int(K[f"point{k}_ny"]),
                             float(K[f"point{k}_h"])).table
            assert np.array_equal(t, K[f"point{k}_table"])

    def test_params(self):
        from paper_2008_03276_b200.ehl import EhlParams, moes_convert, moes_from_line
        u, w = moes_convert(m=20.0, l=10.0, g=5000.0)
        m, l = moes_from_line(5000.0, u, w)
        assert m == pytest.approx(20.0, rel=1e-12) and l == pytest.approx(10.0, rel=1e-12)
        p = EhlParams.line_from_loads(5000.0, u, w, domain=(-4.5, 1.5))
        assert p.load_target == pytest.approx(np.pi / 2)
        with pytest.raises(ContractViolationError):
            EhlParams(contact="line", moes_m=1, moes_l=1)
        with pytest.raises(ContractViolationError):
            EhlParams.point_from_moes(100, 10, relax_c=0.5)
        q = EhlParams.point_from_moes(100.0, 10.0)
        assert q.load_target == pytest.approx(1.5 * np.pi)

    def test_hybrid_select_and_nu(self):
        from paper_2008_03276_b200.ehl import hybrid_select, kernel_nu
        assert list(hybrid_select([0.5, 0.7], "Lhs1")) == ["Ls4", "Ls1"]
        assert list(hybrid_select([0.6, 0.61], "Lhs2")) == ["Ls5", "Ls0"]
        assert kernel_nu("Ls5", 1 / 3) == pytest.approx((2 - 1 / 3) / 2 + (1 - 1 / 3) / 4)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _shard_worker(rank, world, port, q):
    """One rank of bench.py's sharded configs, over gloo: its config-2 shard
    (bench.shard_inputs), its config-3 cases (bench.config3_cases) and the
    max-over-ranks reduction bench.py applies to the step times."""
    import torch.distributed as dist
    import oracle
    import bench
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    per = 3
    bands, f = bench.shard_inputs(rank, per)
    u, act, passes, res, st = oracle.lcp_batch(bands, f)
    cases = bench.config3_cases(rank, count=5)
    gathered = [None] * world
    dist.all_gather_object(gathered, (u, passes, cases))
    tmax = bench.make_max_over_ranks(dist, "cpu")(float(rank + 1))
    if rank == 0:
        q.put((gathered, tmax))
    dist.destroy_process_group()


def test_weak_scaling_shards_gloo():
    """Two ranks solve disjoint seeded shards with no data-path collective;
    gathering them reproduces the single-process batch exactly (config 2),
    the config-3 case lists tile the single-process list, and the
    max-over-ranks timing reduction returns the slowest rank's value."""
    import multiprocessing as mp
    import oracle
    import bench
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    gathered, tmax = q.get(timeout=180)
    for p in procs:
        p.join(timeout=60)
    assert tmax == 2.0
    bands, f = bench.shard_inputs(0, 6)
    u, act, passes, res, st = oracle.lcp_batch(bands, f)
    got_u = np.concatenate([g[0] for g in gathered])
    got_p = np.concatenate([g[1] for g in gathered])
    assert np.array_equal(got_u, u) and np.array_equal(got_p, passes)
    assert gathered[0][2] + gathered[1][2] == bench.config3_cases(0, count=10)
    assert gathered[0][2] != gathered[1][2]


def test_bench_launcher_spawns_ranks():
    """bench.py --gpus 2 without a launcher re-executes itself under
    torch.distributed.run; the reference arm prints one line from rank 0
    with n_gpus = 2 and the same config dict as the GPU arm."""
    import json
    import subprocess
    import sys
    import bench
    env = dict(os.environ)
    for k in ("WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, os.path.join(bench.ROOT, "bench.py"), "--impl",
                        "reference", "--gpus", "2", "--steps", "1", "--warmup", "3",
                        "--no-ref-code"], capture_output=True, text=True, timeout=600, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    line = lines[0]
    assert line["impl"] == "reference" and line["n_gpus"] == 2
    assert line["config"] == bench.headline_config(bench.B_PER_GPU)
    assert line["e2e"]["h2d_bytes_per_step"] == 0


class TestTvdHost:
    """Host set-up of the TVD study (tvdcd.py mirror): the operator and
    residual norm reproduce the reference's residual norms bit for bit
    (golden tvd.npz), plus the contract errors and study helpers."""

    def test_residual_norm_vs_reference(self):
        from conftest import load_golden
        from paper_2008_03276_b200.tvdcd import (ConvectionDiffusionProblem, Grid2D,
                                                 KappaSchemeConfig)
        T = load_golden("tvd.npz")
        prob = ConvectionDiffusionProblem(Grid2D(0.0, 1.0, 0.0, 1.0, 19, 19),
                                          KappaSchemeConfig(kappa=0.0, eps=1e-4, a=1.0, b=0.7),
                                          T["c_upwind_ls0__f"], T["c_upwind_ls0__boundary"],
                                          closure="upwind")
        assert prob.residual_norm(T["c_upwind_ls0__u1"]) == T["c_upwind_ls0__res"][0]
        assert prob.residual_norm(T["c_upwind_ls0__u2"]) == T["c_upwind_ls0__res"][1]

    def test_contracts_and_helpers(self):
        from paper_2008_03276_b200.tvdcd import (Grid2D, KappaSchemeConfig, convergence_order,
                                                 error_norms, transposed_problem,
                                                 quartic_test_problem)
        g = Grid2D.square(16)
        assert g.h == pytest.approx(2.0 / 16) and g.nx == 15
        with pytest.raises(ContractViolationError):
            Grid2D(0.0, 1.0, 0.0, 2.0, 7, 7)
        with pytest.raises(ContractViolationError):
            KappaSchemeConfig(kappa=1.5)
        with pytest.raises(ContractViolationError):
            quartic_test_problem(4, KappaSchemeConfig())
        u = np.ones((4, 4))
        assert error_norms(u, u, 0.1) == (0.0, 0.0, 0.0)
        assert convergence_order([1.0, 0.5, 0.25]) == pytest.approx([1.0, 1.0])
        prob, exact = quartic_test_problem(16, KappaSchemeConfig(kappa=1 / 3, eps=1e-6))
        twin = transposed_problem(prob)
        r1 = prob.residual_field(exact)
        r2 = twin.residual_field(np.ascontiguousarray(exact.T))
        assert np.allclose(r1, r2.T, atol=1e-12)


def _shard_attach_worker(rank, world, port, q):
    """One rank of PointContact.shard_folds over gloo with the native calls
    mocked: every rank must receive all ranks' IPC handles in rank order."""
    import ctypes
    import torch.distributed as dist
    from paper_2008_03276_b200.ehl.point import PointContact
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)

    class FakeL:
        attached = None

        def paqif_ehl_point_ipc_handles(self, ptr, buf):
            ctypes.memmove(buf, bytes([rank + 1]) * 192, 192)
            return 0

        def paqif_ehl_point_attach_peers(self, ptr, r, w, blob):
            FakeL.attached = (r, w, bytes(blob.raw))
            return 0

    class FakeH:
        ptr = 1

    pc = object.__new__(PointContact)
    pc.L, pc._h = FakeL(), FakeH()
    pc.sync = lambda: None
    w = pc.shard_folds()
    q.put((rank, w, FakeL.attached))
    dist.destroy_process_group()


def test_shard_folds_handle_exchange_gloo():
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_attach_worker, args=(r, 3, port, q)) for r in range(3)]
    for p in procs:
        p.start()
    got = [q.get(timeout=180) for _ in range(3)]
    for p in procs:
        p.join(timeout=60)
    expect = b"".join(bytes([r + 1]) * 192 for r in range(3))
    for rank, w, (r, wa, blob) in got:
        assert w == 3 and wa == 3 and r == rank
        assert blob == expect
