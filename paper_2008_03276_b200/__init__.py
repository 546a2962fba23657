"""paper_2008_03276_b200 -- B200-native (sm_100a, fp64) PAQIF solvers and the
EHL Newton step of arXiv 2008.03276, behind the reference package's API.

The module layout mirrors the reference package ``paqif`` so it drops in:

    paqif                 -> paper_2008_03276_b200
    paqif._kernels        -> paper_2008_03276_b200._kernels   (CUDA, bit-exact)
    paqif.aqif / parallel / lcp / bandcore / errors           (same names)
    paqif.ehl             -> paper_2008_03276_b200.ehl

Batched device entry points (the GPU-native granularity) live in
``paper_2008_03276_b200.batch``.  All compute goes through
``_build/libpaqif_b200.so``; there is no CPU fallback.
"""

from .bandcore import (BandedMatrix, band_matvec, cholesky_spd_solve, is_diagonally_dominant,
                       project_nonneg)
from .aqif import WZFactors, aqif_solve, factorize_wz, solve_w, solve_z
from .errors import (ContractViolationError, FactorizationBreakdownError, NonConvergenceError,
                     NotPositiveDefiniteError, PaqifError, PartitionError,
                     UnsupportedOrderError)

__version__ = "0.1.0"
