"""B200-native batched one-sided Jacobi SVD (arXiv 2601.17979 hot path).

Drop-in for the reference package's batch entry point
(/root/reference/pkg/src/bsvd/batch.py:85 ``batch_svd``) and the solver
records it returns.  Every solve runs in hand-written sm_100a CUDA kernels
behind the C-ABI in include/bsvd_b200.h (paper_2601_17979_b200/_lib/
libbsvd_b200.so); there is no CPU fallback.
"""

from . import backend
from .backend import Backend, active, select, use
from .batch import BatchState, batch_svd, convergence_scan
from .core import (
    SUPPORTED_DTYPES,
    DomainError,
    ShapeError,
    check_dtype,
    fmatrix,
    is_complex,
    real_dtype,
    unit_roundoff,
)
from .eig import EigInfo, Rotation, batch_hermitian_eig, compute_rotation, jacobi_hermitian_eig
from .kernels import compute_gram, eig_sweeps, fused_pair_update, householder_qr, onesided_sweeps
from .ordering import Schedule, round_robin_schedule, schedule_arrays
from .solver import DeviceResult, solve_tensor
from . import fileio
from .fileio import (
    DTYPE_CODES,
    FormatError,
    ResultRecord,
    read_matrices,
    read_results,
    write_matrices,
    write_results,
)
from .matgen import FAMILIES, make_sigma
from .verify import (
    ErrorReport,
    error_report,
    orthogonality_e2_e3,
    residual_e1,
    sigma_error_e4,
    threshold,
    verify_tensor,
)
from .svd import (
    JacobiOptions,
    SolveInfo,
    SvdResult,
    WorkCounters,
    finalize,
    svd_blocked,
    svd_dispatch,
    svd_qr_preprocessed,
    svd_unblocked,
)

__version__ = "0.1.0"

__all__ = [
    "BatchState",
    "DeviceResult",
    "DomainError",
    "EigInfo",
    "ErrorReport",
    "JacobiOptions",
    "Rotation",
    "Schedule",
    "ShapeError",
    "SolveInfo",
    "SUPPORTED_DTYPES",
    "SvdResult",
    "WorkCounters",
    "batch_hermitian_eig",
    "batch_svd",
    "check_dtype",
    "compute_gram",
    "compute_rotation",
    "convergence_scan",
    "error_report",
    "fileio",
    "fmatrix",
    "fused_pair_update",
    "is_complex",
    "jacobi_hermitian_eig",
    "onesided_sweeps",
    "real_dtype",
    "round_robin_schedule",
    "schedule_arrays",
    "solve_tensor",
    "svd_blocked",
    "svd_dispatch",
    "svd_qr_preprocessed",
    "svd_unblocked",
    "threshold",
    "unit_roundoff",
    "verify_tensor",
    "finalize",
    "householder_qr",
    "eig_sweeps",
    "Backend",
    "active",
    "select",
    "use",
    "backend",
    "residual_e1",
    "orthogonality_e2_e3",
    "sigma_error_e4",
    "DTYPE_CODES",
    "FormatError",
    "ResultRecord",
    "read_matrices",
    "read_results",
    "write_matrices",
    "write_results",
    "FAMILIES",
    "make_sigma",
    "__version__",
]
