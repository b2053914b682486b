"""ctypes binding of libchebfd_b200.so (the C ABI in include/chebfd_b200.h).

The shared library is built in tree (``make -C paper_1510_04895_b200/csrc``
or ``__graft_entry__.build()``).  There is no fallback: if the library is
missing or a call fails, an exception is raised.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CHEBFD_B200_LIB overrides the library path (A/B builds); default: the in-tree build
LIB_PATH = os.environ.get("CHEBFD_B200_LIB", os.path.join(HERE, "libchebfd_b200.so"))

_i64 = C.c_int64
_u64 = C.c_uint64
_dbl = C.c_double
_vp = C.c_void_p
_int = C.c_int
_pp = C.POINTER(C.c_void_p)


class chebfd_lattice(C.Structure):
    _fields_ = [("lx", _i64), ("ly", _i64), ("lz", _i64), ("t", _dbl), ("disorder", _dbl),
                ("boundary", _int), ("seed", _u64)]


class chebfd_partition(C.Structure):
    _fields_ = [("dim", _i64), ("row_begin", _i64), ("local_rows", _i64), ("halo_lo", _i64),
                ("halo_hi", _i64), ("lo_src_begin", _i64), ("hi_src_begin", _i64),
                ("lo_rank", _int), ("hi_rank", _int), ("bnd_lo", _i64), ("bnd_hi", _i64),
                ("send_lo_begin", _i64), ("send_lo_n", _i64), ("send_hi_begin", _i64),
                ("send_hi_n", _i64)]


class chebfd_matrix_info(C.Structure):
    _fields_ = [("kind", _int), ("dim", _i64), ("nnz", _i64), ("local_rows", _i64),
                ("row_begin", _i64), ("local_nnz", _i64), ("sell_entries", _i64),
                ("halo_lo", _i64), ("halo_hi", _i64), ("chunk", _int), ("max_row_len", _int),
                ("stage_rows", _int)]


class chebfd_design(C.Structure):
    _fields_ = [("np_opt", _int), ("eta_opt", _dbl), ("sigma", _dbl), ("predicted_mvms", _dbl),
                ("predicted_iters", _int), ("delta_prime", _dbl), ("n_target_estimate", _dbl),
                ("below_recommended_search_space", _int)]


class chebfd_bench_point(C.Structure):
    _fields_ = [("n_b", _int), ("seconds", _dbl), ("flops", _dbl), ("gflops", _dbl),
                ("gbs_proxy", _dbl), ("intensity", _dbl), ("roofline", _dbl), ("efficiency", _dbl)]


class chebfd_solver_options(C.Structure):
    _fields_ = [("target_lo", _dbl), ("target_hi", _dbl), ("epsilon", _dbl), ("n_search", _int),
                ("degree", _int), ("kernel", _int), ("kernel_mu", _int), ("max_iters", _int),
                ("seed", _u64), ("dos_moments", _int), ("dos_samples", _int),
                ("bounds_lo", _dbl), ("bounds_hi", _dbl), ("collect_weight_density", _int)]


class chebfd_solve_report(C.Structure):
    _fields_ = [("converged", _int), ("iterations", _int), ("n_search", _int), ("degree", _int),
                ("n_values", _int), ("total_spmvms", _dbl), ("sigma", _dbl), ("eta", _dbl),
                ("bounds_lo", _dbl), ("bounds_hi", _dbl), ("matrix_norm_est", _dbl),
                ("n_target_estimate", _dbl), ("seconds", _dbl), ("weight_integral", _dbl),
                ("t_bounds", _dbl), ("t_dos", _dbl), ("t_design", _dbl), ("t_filter", _dbl),
                ("t_ortho", _dbl), ("t_rr", _dbl), ("t_start", _dbl)]


_SIGS = {
    "chebfd_last_error": (C.c_char_p, []),
    "chebfd_version": (C.c_char_p, []),
    "chebfd_build_features": (_int, []),
    "chebfd_vgroup_create": (_int, [_int, _int, _pp]),
    "chebfd_vgroup_destroy": (_int, [_vp]),
    "chebfd_vgroup_context": (_int, [_vp, _int, _pp]),
    "chebfd_vgroup_set_option": (_int, [_vp, _int, _i64]),
    "chebfd_vgroup_matrix_lattice": (_int, [_vp, _int, _vp, _vp]),
    "chebfd_vgroup_apply_filter": (_int, [_vp, _vp, _vp, _vp, _int, _dbl, _dbl, _vp]),
    "chebfd_vgroup_spmmvm_fused": (_int, [_vp, _vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _vp]),
    "chebfd_vgroup_gram": (_int, [_vp, _vp, _vp, _vp]),
    "chebfd_vgroup_halo_rows": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "chebfd_nccl_unique_id": (_int, [_vp]),
    "chebfd_ctx_create": (_int, [_int, _pp]),
    "chebfd_ctx_create_dist": (_int, [_int, _int, _int, _vp, _pp]),
    "chebfd_ctx_destroy": (_int, [_vp]),
    "chebfd_ctx_synchronize": (_int, [_vp]),
    "chebfd_ctx_stream": (_int, [_vp, _pp]),
    "chebfd_ctx_info": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "chebfd_ctx_launch_count": (_int, [_vp, _vp]),
    "chebfd_ctx_set_option": (_int, [_vp, _int, _i64]),
    "chebfd_ctx_band_launches": (_int, [_vp, _vp]),
    "chebfd_ctx_group_launches": (_int, [_vp, _vp]),
    "chebfd_ctx_ring_launches": (_int, [_vp, _vp]),
    "chebfd_ctx_event_record": (_int, [_vp, _int]),
    "chebfd_ctx_event_elapsed": (_int, [_vp, _int, _int, _vp]),
    "chebfd_host_alloc": (_int, [C.c_size_t, _pp]),
    "chebfd_host_free": (_int, [_vp]),
    "chebfd_csr_graphene": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "chebfd_csr_topological_insulator": (_int, [_vp, _i64, _i64, _vp, _vp, _vp, _vp, _vp]),
    "chebfd_plan_partition": (_int, [_vp, _int, _int, _int, _vp]),
    "chebfd_plan_sends": (_int, [_vp, _int, _int, _vp]),
    "chebfd_plan_map_column": (_i64, [_vp, _i64]),
    "chebfd_matrix_from_csr": (_int, [_vp, _int, _i64, _vp, _vp, _vp, _pp]),
    "chebfd_matrix_graphene": (_int, [_vp, _vp, _pp]),
    "chebfd_matrix_topological_insulator": (_int, [_vp, _vp, _pp]),
    "chebfd_matrix_destroy": (_int, [_vp]),
    "chebfd_matrix_get_info": (_int, [_vp, _vp]),
    "chebfd_block_create": (_int, [_vp, _i64, _pp]),
    "chebfd_block_create_dim": (_int, [_vp, _int, _i64, _i64, _pp]),
    "chebfd_block_create_like": (_int, [_vp, _i64, _pp]),
    "chebfd_block_destroy": (_int, [_vp]),
    "chebfd_block_info": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "chebfd_block_upload": (_int, [_vp, _vp]),
    "chebfd_block_download": (_int, [_vp, _vp]),
    "chebfd_block_copy": (_int, [_vp, _vp]),
    "chebfd_block_zero": (_int, [_vp]),
    "chebfd_block_randomize": (_int, [_vp, _u64]),
    "chebfd_block_randomize_device": (_int, [_vp, _u64]),
    "chebfd_host_randomize": (_int, [_int, _u64, _i64, _i64, _vp]),
    "chebfd_block_scale_columns": (_int, [_vp, _vp]),
    "chebfd_block_copy_columns": (_int, [_vp, _i64, _vp, _i64, _i64]),
    "chebfd_block_device_ptr": (_int, [_vp, _pp]),
    "chebfd_intensity_model": (_int, [_dbl, _int, _int, _int, _int, _int, C.POINTER(_dbl)]),
    "chebfd_bandwidth_probe_min_bytes": (_int, [_vp, C.POINTER(_u64)]),
    "chebfd_bandwidth_probe": (_int, [_vp, _u64, _int, C.POINTER(_dbl)]),
    "chebfd_bench_filter": (_int, [_vp, _vp, _int, _int, _dbl, _vp, C.POINTER(_dbl)]),
    "chebfd_read_matrix_market": (_int, [C.c_char_p, _vp, _vp, _vp, _vp, _vp, _vp, _vp]),
    "chebfd_write_matrix_market": (_int, [C.c_char_p, _int, _i64, _vp, _vp, _vp, _int]),
    "chebfd_matrix_from_matrix_market": (_int, [_vp, C.c_char_p, _pp]),
    "chebfd_cbfd_save": (_int, [C.c_char_p, _int, _u64, C.c_uint32, _vp]),
    "chebfd_cbfd_load": (_int, [C.c_char_p, _vp, _vp, _vp, _vp]),
    "chebfd_block_save": (_int, [_vp, C.c_char_p]),
    "chebfd_block_load": (_int, [_vp, C.c_char_p, _pp]),
    "chebfd_spmmvm": (_int, [_vp, _vp, _vp, _dbl, _dbl]),
    "chebfd_spmmvm_fused": (_int, [_vp, _vp, _vp, _vp, _dbl, _dbl, _dbl, _vp]),
    "chebfd_recurrence_step": (_int, [_vp, _vp, _vp, _dbl, _dbl]),
    "chebfd_block_axpy_scal": (_int, [_vp, _vp, _vp, _dbl, _dbl, _dbl]),
    "chebfd_column_dots": (_int, [_vp, _vp, _vp]),
    "chebfd_column_norms": (_int, [_vp, _vp]),
    "chebfd_gram": (_int, [_vp, _vp, _vp]),
    "chebfd_block_mult_small": (_int, [_vp, _vp, _i64, _vp]),
    "chebfd_window_coeffs": (_int, [_dbl, _dbl, _dbl, _dbl, _int, _vp]),
    "chebfd_kernel_coeffs": (_int, [_int, _int, _int, _vp]),
    "chebfd_make_filter": (_int, [_dbl, _dbl, _dbl, _dbl, _int, _int, _int, _vp, _vp, _vp]),
    "chebfd_eval_scalar": (_int, [_vp, _int, _dbl, _dbl, _dbl, _dbl, _dbl, _vp]),
    "chebfd_apply_filter": (_int, [_vp, _vp, _vp, _int, _dbl, _dbl, _vp]),
    "chebfd_apply_filter_host": (_int, [_vp, _vp, _i64, _vp, _int, _dbl, _dbl, _vp]),
    "chebfd_filter_pipe_create": (_int, [_vp, _i64, _pp]),
    "chebfd_filter_pipe_submit": (_int, [_vp, _vp, _vp, _vp, _int, _dbl, _dbl]),
    "chebfd_filter_pipe_submit_gram": (_int, [_vp, _vp, _vp, _vp, _int, _dbl, _dbl, _vp]),
    "chebfd_filter_pipe_wait": (_int, [_vp]),
    "chebfd_filter_pipe_destroy": (_int, [_vp]),
    "chebfd_svqb": (_int, [_vp, _dbl, _vp, _vp]),
    "chebfd_rayleigh_ritz": (_int, [_vp, _vp, _vp, _vp, _vp]),
    "chebfd_lanczos_bounds": (_int, [_vp, _int, _u64, _vp, _vp]),
    "chebfd_kpm_dos": (_int, [_vp, _dbl, _dbl, _int, _int, _u64, _vp]),
    "chebfd_dos_count": (_int, [_vp, _int, _dbl, _dbl, _dbl, _dbl, _vp]),
    "chebfd_dos_density": (_int, [_vp, _int, _dbl, _dbl, _dbl, _vp]),
    "chebfd_weight_density": (_int, [_vp, _int, _i64, _vp]),
    "chebfd_damping_factor": (_int, [_dbl, _dbl, _dbl, _dbl, _dbl, _int, _int, _int, _vp]),
    "chebfd_optimize_degree": (_int, [_dbl, _dbl, _dbl, _dbl, _dbl, _int, _int, _dbl, _vp]),
    "chebfd_invert_search_margin": (_int, [_vp, _int, _dbl, _dbl, _dbl, _dbl, _dbl, _vp]),
    "chebfd_choose_parameters": (_int, [_vp, _int, _dbl, _dbl, _dbl, _dbl, _dbl, _int, _int, _dbl,
                                        _vp]),
    "chebfd_solver_options_default": (None, [_vp]),
    "chebfd_solve": (_int, [_vp, _vp, _vp, _int, _vp, _vp, _vp, _vp, _pp]),
    "chebfd_solve_ex": (_int, [_vp, _vp, _vp, _int, _vp, _vp, _vp, _vp, _pp, _int, _vp, _vp]),
}

EXPORTED = tuple(_SIGS)

_lib = None


def load(path: str = LIB_PATH):
    """Load the library once; raise ImportError if it has not been built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(path):
        raise ImportError(
            f"{path} not found: build the CUDA library first "
            "(python -c 'import __graft_entry__ as g; g.build()' or "
            "make -C paper_1510_04895_b200/csrc)")
    lib = C.CDLL(path)
    for name, (res, args) in _SIGS.items():
        try:
            fn = getattr(lib, name)
        except AttributeError:
            # an older build (CHEBFD_B200_LIB A/B runs): calling the symbol raises
            if path == os.path.join(HERE, "libchebfd_b200.so"):
                raise
            continue
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib
