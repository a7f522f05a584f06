"""B200-native (sm_100a) two-level-preconditioned CG — the hot path of NeuraLSP
(arXiv 2601.20174, reference `nlsp`), behind the reference's solver /
preconditioner interface. See DESIGN.md."""
from .nlsp import (  # noqa: F401
    ConvergenceError,
    Context,
    CudaError,
    DeviceCsr,
    DeviceDense,
    IdentityPreconditioner,
    JacobiPreconditioner,
    JacobiSmoother,
    NotSpdError,
    NumericError,
    PcgResult,
    RankDeficiencyError,
    SolveReport,
    SparseCsrMatrix,
    TwoLevelPreconditioner,
    ValidationError,
    apply_two_level,
    build_preconditioner,
    default_context,
    generate_smoothed_vectors,
    pcg,
    smooth_vectors,
    spmv,
    svd_basis,
)
