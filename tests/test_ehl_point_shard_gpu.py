"""Sharded point-contact fold (config 5 on several GPUs, csrc/fft_shard.cuh).

The slab decomposition -- row FFTs, column FFTs x kernel spectrum, inverse
row FFTs, each rank its slab -- is checked with the ranks emulated one after
another on one GPU (every "peer" buffer the local one): the deformation must
be bit-identical to the one-kernel fold for any number of ranks, since every
row and column runs the same device function.  The multi-rank plumbing
(IPC handles, peer stores, barriers) runs only with several GPUs
(bench.py --gpus N); its host logic has CPU tests in test_host_logic.py.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("n", [64, 512, 2048])
def test_sharded_fold_bit_identical_emulated(n):
    from paper_2008_03276_b200.ehl import EhlParams
    from paper_2008_03276_b200.ehl.point import PointDevice, point_grid
    from paper_2008_03276_b200.ehl.kernels import kernel_point
    p = EhlParams.point_from_moes(1000.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
    x, y, h = point_grid(p, n)
    gx, gy = np.meshgrid(x, y)
    dev = PointDevice(kernel_point(n, n, h).table, 0.5 * (gx ** 2 + gy ** 2))
    rng = np.random.default_rng(n)
    u = np.maximum(0.0, rng.standard_normal((n + 1, n + 1)))
    ref = dev.deformation(u)
    for world in (1, 2, 3, 5, 8):
        got = dev.fold_emulated(world, u)
        assert np.array_equal(got.view(np.uint64), ref.view(np.uint64)), world


def test_single_rank_shard_is_noop():
    """Without torch.distributed (or with one rank) shard_folds leaves the
    contact on the one-kernel fold."""
    from paper_2008_03276_b200.ehl import EhlParams, PointContact
    p = EhlParams.point_from_moes(100.0, 10.0, domain=(-4.5, 1.5), lo_y=-3.0)
    pc = PointContact(p, 32)
    assert pc.shard_folds() == 1
    pc.step()
    assert np.isfinite(pc.status()[1])
    pc.close()
