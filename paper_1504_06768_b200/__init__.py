"""rhosolve-b200: B200-native steady-state solver for Lindblad Liouvillians
(arXiv 1504.06768), a drop-in for the reference `rhosolve` hot path.

Host code mirrors the reference API; every stage on the n x n Liouvillian
runs as hand-written sm_100a CUDA behind the C ABI in
include/rhosolve_b200.h (library: _lib/librhosolve_b200.so).  There is no
CPU fallback: without the library or a GPU the solver entry points raise.
"""

from .sparse import CSRMatrix, Permutation, DeviceCSR, PinnedBatchCSR, from_host, pin_batch
from .operators import QuantumOperator, destroy, spin_ops, embed, identity_operator
from .liouville import (LiouvillianSystem, build_liouvillian, build_liouvillian_batch, shift,
                        build_modified, default_weight, DEFAULT_SIGMA)
from .ordering import rcm, band_profile, BandProfile
from .factor import (LUFactors, lu, ilutp, solve_lu, condest, SingularMatrixError,
                     PreconditionerBreakdownError)
from .krylov import IterOptions, IterResult, gmres, bicgstab
from .steady import (SteadyStateResult, solve_direct, solve_iterative, inverse_power,
                     inverse_power_batch, solve_batch, InnerSolverError, PowerIterationError,
                     DEFAULT_SEED, MAX_OUTER)

KERNEL_BACKEND = "cuda-sm_100a"
__version__ = "0.1.0"
