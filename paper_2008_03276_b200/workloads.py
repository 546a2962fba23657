"""Seeded synthetic inputs for the BASELINE.json configurations.

No public dataset is involved: every input is drawn on
the host from ``numpy.random.default_rng`` so the CPU oracle and the GPU see
identical bits.  System ``b`` of a batch is drawn from its own generator
``default_rng((seed, b))`` so a shard computed on rank r of N is bit-identical
to the same system of an unsharded run.

Config 2 ("4096 banded LCPs, n=1025, beta=8"): per system, in this order,
  1. off-diagonals for offsets -beta..-1, 1..beta (ascending), each a vector of
     n draws U(-1, 1); entries that fall outside the matrix are zeroed;
  2. diagonal = sum_o |off_o(i)| + U(0.1, 1)   (strict diagonal dominance);
  3. right side f ~ N(0, 1) (n draws).
n = 1025 is odd and AQIF needs an even order (aqif.py:121-122), so the
system is padded to 1026 with a pinned identity row and f = 0, exactly as the
reference's line systems pad (ehl/sweeps.py:143-154).
"""

from __future__ import annotations

import numpy as np


def padded_order(n: int) -> int:
    return n if n % 2 == 0 else n + 1


def lcp_system(seed: int, b: int, n: int = 1025, beta: int = 8):
    """One config-2 system: (bands (2beta+1, n_pad), f (n_pad,))."""
    rng = np.random.default_rng((seed, b))
    npad = padded_order(n)
    bands = np.zeros((2 * beta + 1, npad))
    offs = [o for o in range(-beta, beta + 1) if o != 0]
    vals = rng.uniform(-1.0, 1.0, (len(offs), n))
    for k, o in enumerate(offs):
        row = bands[beta + o, :n]
        row[:] = vals[k]
        # zero entries whose column leaves the (unpadded) matrix
        if o > 0:
            row[n - o:] = 0.0
        else:
            row[:-o] = 0.0
    off = np.abs(bands[:, :n]).sum(axis=0) - np.abs(bands[beta, :n])
    bands[beta, :n] = off + rng.uniform(0.1, 1.0, n)
    f = np.zeros(npad)
    f[:n] = rng.standard_normal(n)
    if npad != n:
        bands[beta, n:] = 1.0
    return bands, f


def lcp_batch(seed: int, count: int, n: int = 1025, beta: int = 8, start: int = 0):
    """Systems ``start .. start+count-1`` of the seeded config-2 batch."""
    npad = padded_order(n)
    bands = np.empty((count, 2 * beta + 1, npad))
    f = np.empty((count, npad))
    for k in range(count):
        bands[k], f[k] = lcp_system(seed, start + k, n, beta)
    return bands, f


def random_banded(n: int, beta: int, rng, dominant: bool = True, m_matrix: bool = False):
    """Diagonal-major random banded matrix with the construction the
    reference's test fixture uses (tests/conftest.py:7-28): off-diagonals
    U(0.2,1) with random signs (or all negative for M-matrices), diagonal =
    row |off| sum + U(0.5, 2), or U(-1,1) when not dominant."""
    bands = np.zeros((2 * beta + 1, n))
    for o in range(-beta, beta + 1):
        if o == 0:
            continue
        vals = rng.uniform(0.2, 1.0, n)
        if not m_matrix:
            vals *= rng.choice([-1.0, 1.0], n)
        else:
            vals = -vals
        bands[beta + o] = vals
    zero_out_of_range(bands)
    if dominant:
        off = np.zeros(n)
        for o in range(-beta, beta + 1):
            if o != 0:
                off += np.abs(bands[beta + o])
        bands[beta] = off + rng.uniform(0.5, 2.0, n)
    else:
        bands[beta] = rng.uniform(-1.0, 1.0, n)
    return bands


def zero_out_of_range(bands: np.ndarray) -> np.ndarray:
    """Force entries mapping outside the matrix to exact zero
    (bandcore.py:48-55 semantics) on a (..., 2beta+1, n) array."""
    beta = (bands.shape[-2] - 1) // 2
    n = bands.shape[-1]
    for o in range(-beta, beta + 1):
        if o > 0:
            bands[..., beta + o, n - o:] = 0.0
        elif o < 0:
            bands[..., beta + o, :-o] = 0.0
    return bands
