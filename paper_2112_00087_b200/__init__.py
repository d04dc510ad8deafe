"""B200-native complex-FP64 Krylov / Schwarz-DDM Helmholtz solver.

Drop-in for the reference's solve path (cavac: numkit + krylov + schwarz);
see DESIGN.md.  The compute runs in libcavac_b200.so (hand-written sm_100a
CUDA behind the C ABI in include/cavac_b200.h).
"""
from .cavac import (  # noqa: F401
    CsrMatrix, Device, ExecMode, InvalidArgument, LogicError, Preconditioner, SolveReport,
    SolveResult, SolverId, SolverOptions, axpy, axpy_inplace, bicgstab, bicgstab_l, cocg,
    csr_from_triplets, csr_identity, dot_hermitian, exec_mode, gmres, identity_preconditioner, ilu0,
    ilu0_factor,
    jacobi, norm2, option, path_options, scale_inplace, set_exec_mode, solve, solver_from_name, solver_id,
    solver_name, spmv,
    tfqmr, true_relative_residual, xpay_inplace,
)
