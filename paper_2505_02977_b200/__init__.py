"""B200-native (sm_100a) randomized approximate Cholesky (rchol / ParAC,
arXiv 2505.02977) for graph-Laplacian preconditioning, plus the PCG solve that
consumes it. Drop-in for the reference library `parac`'s factor / solve entry
points; see include/parac_gpu.h (C ABI) and rchol.py (host mirror)."""
from .rchol import (  # noqa: F401
    Errc, Error, LaplacianGraph, Ordering, LdlFactor, FactorStats, GpuOptions, GpuContext,
    SolveConfig, SolveReport, factor_gpu, pcg_solve_gpu, apply_preconditioner_gpu,
    laplacian_apply_gpu, schedule_levels_gpu, dependency_counts, make_rhs, gen_poisson3d,
    gen_poisson2d, gen_poisson27, gen_rmat, gen_random_connected, gen_random_components,
    ordering_random, ordering_nnz_sort, ordering_nnz_sort_gpu, default_context, device_count, factor_batch_gpu,
    read_laplacian, write_matrix_market, write_factor, read_factor, write_vector, read_vector,
    write_permutation, ordering_from_file,
)
from ._lib import LIB_PATH  # noqa: F401
