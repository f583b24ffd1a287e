"""paper_1207_1114_b200 — B200-native FastPFP hot path (arXiv 1207.1114).

Public API (thin wrapper over the C-ABI in include/fastpfp.h):
    Solver(n, n_prime, d)          fastpfp_create
    .set_graphs(A, Ap, B, Bp)      fastpfp_set_graphs   (numpy on host or torch CUDA tensors)
    .set_x0(X0) / .reset()         fastpfp_set_x0 / fastpfp_reset
    .iterate(alpha, lam, eps1, eps2, max_iter1, max_iter2) -> (X, report)
    .discretize() / .objective(lam)
The shared library is loaded lazily on first use; there is no CPU fallback.
"""
from ._native import (  # noqa: F401
    EINVAL, ENCCL, ENONFINITE, EPOISONED, ESTATE, ESYM, OPT_CHECK_EVERY, OPT_NCCL_TIMEOUT_MS, OPT_GEMM_CTA_GROUP, OPT_METHOD, OPT_PRECISION, OPT_PROFILE, OPT_PROJ_KERNEL,
    METHOD_FASTPFP, METHOD_PG, METHOD_FASTGA, OPT_RESCALE,
    OPT_SLACK_MODE, OPT_STREAM, PREC_FP32_SIMT, PREC_INT8_OZAKI, PREC_TF32, PREC_TF32X3, FastPFPError,
    BatchedSolver, BatchReport, IterReport, Solver, gemm_nt, gemm_nt_blocked, lib, nccl_unique_id, project,
)
