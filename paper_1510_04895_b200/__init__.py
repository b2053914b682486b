"""chebfd_b200: B200-native ChebFD hot path (arXiv 1510.04895).

The product is libchebfd_b200.so (csrc/, sm_100a kernels + C ABI declared in
include/chebfd_b200.h).  This package mirrors the reference's driver API on
top of that ABI; it never computes on the CPU.
"""
from .api import (  # noqa: F401
    BlockVector, ChebfdError, Context, ConvergenceReport, CudaError, DomainError, DosEstimate,
    FilterPolynomial, Interval, InvalidArgument, Kernel, LatticeSpec, MomentTable, NcclError,
    NumericalError, OutOfRange, RitzSet, SolverOptions, SparseMatrix, SvqbResult, Unsupported,
    apply_filter, apply_filter_host, block_axpy_scal, block_mult_small, column_dots, column_norms,
    csr_graphene, csr_topological_insulator, estimate_count, eval_scalar, gram, intensity_model,
    kernel_coeffs, kpm_dos, lanczos_bounds, make_filter, per_row_bytes, per_row_flops,
    plan_all4, plan_complete_sends, plan_map_column, plan_partition, plan_sends,
    rayleigh_ritz, recurrence_step, solve, spmmvm, spmmvm_fused, svqb_orthonormalize,
    window_coeffs, DesignResult, choose_parameters, damping_factor, invert_search_margin,
    optimize_degree, quality, host_randomize, read_matrix_market, write_matrix_market,
    save_block, load_block, BenchPoint, BenchReport, bandwidth_probe, bandwidth_probe_min_bytes,
    bench_filter, FilterPipe, host_array, experimental_build,
    filter_schedule_bytes, WeightDensity, weight_density, VirtualGroup,
)
from ._lib import LIB_PATH, load  # noqa: F401

__version__ = "0.2.0"
