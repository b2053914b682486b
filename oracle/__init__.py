"""CPU oracle for the ChebFD hot path -- TEST INFRASTRUCTURE ONLY.

Two legs, both CPU:

* ``Oracle`` -- ctypes view of ``oracle/_build/libchebfd_oracle.so``, our C
  restatement of the reference algorithm (``oracle/chebfd_oracle.c``; every
  function cites the reference file:line it follows).
* ``Ref`` -- ctypes view of ``oracle/_ref/libchebfd_ref.so``, the UNMODIFIED
  reference (``/root/reference/proj``) compiled in place by
  ``oracle/Makefile`` with an Eigen-subset shim.  Present wherever it was
  built (this container; it travels to the GPU box as a prebuilt .so).

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package, and
only as the checker or the timed reference arm -- never as the product path.

Block vectors are numpy arrays of shape (D, nb), dtype float64 or
complex128, C-contiguous (row-major, ``block_vector.hpp:15-16``).
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_SO = os.path.join(HERE, "_build", "libchebfd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libchebfd_ref.so")

_i64 = C.c_int64
_u64 = C.c_uint64
_dbl = C.c_double
_vp = C.c_void_p

BOUNDARY = {"periodic_xy_open_z": 0, "periodic_all": 1, "open_all": 2}
KERNEL = {"none": 0, "fejer": 1, "jackson": 2, "lanczos": 3}


def _ptr(a):
    return None if a is None else a.ctypes.data_as(_vp)


def _kind(a):
    return 1 if np.iscomplexobj(a) else 0


def _kernel_code(kernel):
    """'lanczos2' / 'jackson' / ('lanczos', mu) -> (kind, mu)."""
    if isinstance(kernel, tuple):
        return KERNEL[kernel[0]], int(kernel[1])
    if kernel.startswith("lanczos"):
        mu = int(kernel[7:]) if len(kernel) > 7 else 2
        return 3, mu
    return KERNEL[kernel], 0


class CSR:
    """Plain CSR triple as the reference stores it (sparse_matrix.hpp:15-107)."""

    def __init__(self, offs, cols, vals):
        self.offs = np.ascontiguousarray(offs, dtype=np.int64)
        self.cols = np.ascontiguousarray(cols, dtype=np.int64)
        self.vals = np.ascontiguousarray(vals)
        self.dim = len(self.offs) - 1

    @property
    def kind(self):
        return _kind(self.vals)

    @property
    def nnz(self):
        return len(self.cols)

    def to_dense(self):
        d = np.zeros((self.dim, self.dim), dtype=self.vals.dtype)
        rows = np.repeat(np.arange(self.dim), np.diff(self.offs))
        np.add.at(d, (rows, self.cols), self.vals)
        return d


def build(quiet=True):
    """Build both legs with oracle/Makefile (the ref leg needs /root/reference)."""
    subprocess.run(["make", "-s", "-C", HERE, "all"], check=True,
                   stdout=subprocess.DEVNULL if quiet else None)


class _CsrStruct(C.Structure):
    _fields_ = [("kind", C.c_int), ("dim", _i64), ("offs", _vp), ("cols", _vp), ("vals", _vp)]


class OracleError(RuntimeError):
    pass


class Oracle:
    """C restatement (oracle/chebfd_oracle.c)."""

    def __init__(self, path=ORACLE_SO):
        if not os.path.exists(path):
            build()
        self.lib = C.CDLL(path)
        L = self.lib
        L.orc_rng_seed.argtypes = [_vp, _u64]
        L.orc_rng_next.restype = _u64
        L.orc_rng_next.argtypes = [_vp]
        L.orc_rng_normal.restype = _dbl
        L.orc_rng_normal.argtypes = [_vp]
        L.orc_randomize.argtypes = [C.c_int, _i64, _i64, _u64, _vp]
        L.orc_graphene.argtypes = [_i64, _i64, _dbl, _dbl, C.c_int, _u64, _vp, _vp, _vp, _vp, _vp]
        L.orc_topological_insulator.argtypes = [_i64, _i64, _i64, _dbl, _dbl, C.c_int, _u64,
                                                _vp, _vp, _vp, _vp, _vp]
        L.orc_window_coeffs.argtypes = [_dbl, _dbl, _dbl, _dbl, C.c_int, _vp]
        L.orc_kernel_coeffs.argtypes = [C.c_int, C.c_int, C.c_int, _vp]
        L.orc_make_filter.argtypes = [_dbl, _dbl, _dbl, _dbl, C.c_int, C.c_int, C.c_int, _vp,
                                      _vp, _vp]
        L.orc_eval_scalar.restype = _dbl
        L.orc_eval_scalar.argtypes = [_vp, C.c_int, _dbl, _dbl, _dbl]
        L.orc_spmmvm.argtypes = [_vp, _vp, _i64, _dbl, _dbl, _vp]
        L.orc_spmmvm_fused.argtypes = [_vp, _vp, _vp, _vp, _i64, _dbl, _dbl, _dbl, _vp]
        L.orc_recurrence_step.argtypes = [_vp, _vp, _vp, _i64, _dbl, _dbl]
        L.orc_block_axpy_scal.argtypes = [C.c_int, _i64, _i64, _vp, _vp, _vp, _dbl, _dbl, _dbl]
        L.orc_column_dots.argtypes = [C.c_int, _i64, _i64, _vp, _vp, _vp]
        L.orc_gram.argtypes = [C.c_int, _i64, _vp, _i64, _vp, _i64, _vp]
        L.orc_block_mult_small.argtypes = [C.c_int, _i64, _i64, _vp, _vp, _i64, _vp]
        L.orc_column_norms.argtypes = [C.c_int, _i64, _i64, _vp, _vp]
        L.orc_apply_filter.argtypes = [_vp, _vp, _i64, _vp, C.c_int, _dbl, _dbl, _vp]
        L.orc_per_row_flops.restype = _dbl
        L.orc_per_row_flops.argtypes = [_dbl, C.c_int, C.c_int]
        L.orc_per_row_bytes.restype = _dbl
        L.orc_per_row_bytes.argtypes = [_dbl, C.c_int, C.c_int, C.c_int]

    # -- RNG --------------------------------------------------------------
    def mt19937_64(self, seed, n):
        st = C.create_string_buffer(312 * 8 + 64)
        self.lib.orc_rng_seed(st, seed)
        return np.array([self.lib.orc_rng_next(st) for _ in range(n)], dtype=np.uint64)

    def randomize(self, dim, width, seed, complex_=False):
        out = np.empty((dim, width), dtype=np.complex128 if complex_ else np.float64)
        self.lib.orc_randomize(int(complex_), dim, width, seed, _ptr(out))
        return out

    # -- models -----------------------------------------------------------
    def _model(self, fn, args, cplx):
        dim, nnz = _i64(), _i64()
        rc = fn(*args, C.byref(dim), C.byref(nnz), None, None, None)
        if rc:
            raise ValueError("LatticeSpec: invalid lattice")
        offs = np.empty(dim.value + 1, np.int64)
        cols = np.empty(nnz.value, np.int64)
        vals = np.empty(nnz.value, np.complex128 if cplx else np.float64)
        fn(*args, C.byref(dim), C.byref(nnz), _ptr(offs), _ptr(cols), _ptr(vals))
        return CSR(offs, cols, vals)

    def graphene(self, lx, ly, t=1.0, disorder=0.0, boundary="periodic_xy_open_z", seed=1):
        return self._model(self.lib.orc_graphene,
                           (lx, ly, t, disorder, BOUNDARY[boundary], seed), False)

    def topological_insulator(self, lx, ly, lz, t=1.0, disorder=0.0,
                              boundary="periodic_xy_open_z", seed=1):
        return self._model(self.lib.orc_topological_insulator,
                           (lx, ly, lz, t, disorder, BOUNDARY[boundary], seed), True)

    # -- filter coefficients -----------------------------------------------
    def window_coeffs(self, target, bounds, degree):
        out = np.empty(degree + 1)
        if self.lib.orc_window_coeffs(target[0], target[1], bounds[0], bounds[1], degree, _ptr(out)):
            raise ValueError("window_coeffs: invalid configuration")
        return out

    def kernel_coeffs(self, kernel, degree):
        k, mu = _kernel_code(kernel)
        out = np.empty(degree + 1)
        if self.lib.orc_kernel_coeffs(k, mu, degree, _ptr(out)):
            raise ValueError("kernel_coeffs: invalid configuration")
        return out

    def make_filter(self, target, bounds, degree, kernel="lanczos2"):
        k, mu = _kernel_code(kernel)
        comb = np.empty(degree + 1)
        a, b = _dbl(), _dbl()
        if self.lib.orc_make_filter(target[0], target[1], bounds[0], bounds[1], degree, k, mu,
                                    _ptr(comb), C.byref(a), C.byref(b)):
            raise ValueError("make_filter: invalid configuration")
        return comb, a.value, b.value

    def eval_scalar(self, combined, alpha, beta, x):
        c = np.ascontiguousarray(combined, dtype=np.float64)
        return self.lib.orc_eval_scalar(_ptr(c), len(c) - 1, alpha, beta, x)

    # -- kernels ------------------------------------------------------------
    @staticmethod
    def _csr(a):
        s = _CsrStruct(a.kind, a.dim, _ptr(a.offs), _ptr(a.cols), _ptr(a.vals))
        return s

    def spmmvm(self, a, x, alpha, beta):
        x = np.ascontiguousarray(x)
        y = np.empty_like(x)
        s = self._csr(a)
        self.lib.orc_spmmvm(C.byref(s), _ptr(x), x.shape[1], alpha, beta, _ptr(y))
        return y

    def spmmvm_fused(self, a, u, w, x, alpha, beta, coeff, want_dots=False):
        """In place on w and x (like the reference); returns dots or None."""
        nb = u.shape[1]
        dots = np.empty(nb, dtype=u.dtype) if want_dots else None
        s = self._csr(a)
        if self.lib.orc_spmmvm_fused(C.byref(s), _ptr(u), _ptr(w), _ptr(x), nb, alpha, beta,
                                     coeff, _ptr(dots)):
            raise ValueError("spmmvm_fused: U, W, X must not alias")
        return dots

    def recurrence_step(self, a, u, w, alpha, beta):
        s = self._csr(a)
        self.lib.orc_recurrence_step(C.byref(s), _ptr(u), _ptr(w), u.shape[1], alpha, beta)

    def block_axpy_scal(self, x, u, w, c0, c1, c2):
        self.lib.orc_block_axpy_scal(_kind(x), x.shape[0], x.shape[1], _ptr(x), _ptr(u), _ptr(w),
                                     c0, c1, c2)

    def column_dots(self, x, y):
        d = np.empty(x.shape[1], dtype=x.dtype)
        self.lib.orc_column_dots(_kind(x), x.shape[0], x.shape[1], _ptr(x), _ptr(y), _ptr(d))
        return d

    def gram(self, x, y):
        g = np.empty((x.shape[1], y.shape[1]), dtype=x.dtype)
        self.lib.orc_gram(_kind(x), x.shape[0], _ptr(x), x.shape[1], _ptr(y), y.shape[1], _ptr(g))
        return g

    def block_mult_small(self, x, b):
        b = np.ascontiguousarray(b, dtype=x.dtype)
        y = np.empty((x.shape[0], b.shape[1]), dtype=x.dtype)
        self.lib.orc_block_mult_small(_kind(x), x.shape[0], x.shape[1], _ptr(x), _ptr(b),
                                      b.shape[1], _ptr(y))
        return y

    def column_norms(self, x):
        out = np.empty(x.shape[1])
        self.lib.orc_column_norms(_kind(x), x.shape[0], x.shape[1], _ptr(x), _ptr(out))
        return out

    def apply_filter(self, a, x, combined, alpha, beta, want_moments=False):
        """Returns (filtered copy of x, moments or None)."""
        x = np.array(x, copy=True, order="C")
        comb = np.ascontiguousarray(combined, dtype=np.float64)
        degree = len(comb) - 1
        mom = np.empty((degree + 1, x.shape[1])) if want_moments else None
        s = self._csr(a)
        if self.lib.orc_apply_filter(C.byref(s), _ptr(x), x.shape[1], _ptr(comb), degree, alpha,
                                     beta, _ptr(mom)):
            raise ValueError("apply_filter: degree must be >= 2")
        return x, mom

    def per_row_flops(self, n_nzr, f_a, f_m):
        return self.lib.orc_per_row_flops(n_nzr, f_a, f_m)

    def per_row_bytes(self, n_nzr, s_d, s_i, n_b):
        return self.lib.orc_per_row_bytes(n_nzr, s_d, s_i, n_b)


class RefError(RuntimeError):
    pass


_REF_EXC = {1: ValueError, 2: RuntimeError, 3: ArithmeticError, 4: IndexError, 9: RuntimeError}


class _RefSolveOptions(C.Structure):
    _fields_ = [("target_lo", _dbl), ("target_hi", _dbl), ("epsilon", _dbl),
                ("n_search", C.c_int), ("degree", C.c_int), ("kernel_kind", C.c_int),
                ("kernel_mu", C.c_int), ("max_iters", C.c_int), ("seed", _u64),
                ("dos_moments", C.c_int), ("dos_samples", C.c_int), ("bounds_lo", _dbl),
                ("bounds_hi", _dbl), ("collect_weight_density", C.c_int)]


class _RefSolveReport(C.Structure):
    _fields_ = [("converged", C.c_int), ("iterations", C.c_int), ("n_search", C.c_int),
                ("degree", C.c_int), ("n_values", C.c_int), ("total_spmvms", _dbl),
                ("sigma", _dbl), ("eta", _dbl), ("bounds_lo", _dbl), ("bounds_hi", _dbl),
                ("matrix_norm_est", _dbl), ("n_target_estimate", _dbl), ("seconds", _dbl),
                ("weight_integral", _dbl)]


class RefMatrix:
    def __init__(self, ref, handle):
        self.ref = ref
        self.h = handle
        kind, dim, nnz = C.c_int(), _i64(), _i64()
        ref._chk(ref.lib.ref_matrix_info(self.h, C.byref(kind), C.byref(dim), C.byref(nnz)))
        self.kind, self.dim, self.nnz = kind.value, dim.value, nnz.value

    def __del__(self):
        try:
            self.ref.lib.ref_matrix_free(self.h)
        except Exception:
            pass

    @property
    def dtype(self):
        return np.complex128 if self.kind else np.float64

    def csr(self):
        offs = np.empty(self.dim + 1, np.int64)
        cols = np.empty(self.nnz, np.int64)
        vals = np.empty(self.nnz, self.dtype)
        self.ref._chk(self.ref.lib.ref_matrix_csr(self.h, _ptr(offs), _ptr(cols), _ptr(vals)))
        return CSR(offs, cols, vals)


class Ref:
    """The compiled reference (oracle/_ref/libchebfd_ref.so)."""

    def __init__(self, path=REF_SO, threads=1):
        if not os.path.exists(path):
            raise FileNotFoundError(path)
        self.lib = C.CDLL(path)
        L = self.lib
        L.ref_last_error.restype = C.c_char_p
        L.ref_matrix_free.argtypes = [_vp]
        for name in ("ref_graphene", "ref_topological_insulator", "ref_diag_flat",
                     "ref_diag_linear", "ref_matrix_from_csr"):
            getattr(L, name).restype = C.c_int
        L.ref_graphene.argtypes = [_i64, _i64, _dbl, _dbl, C.c_int, _u64, _vp]
        L.ref_topological_insulator.argtypes = [_i64, _i64, _i64, _dbl, _dbl, C.c_int, _u64, _vp]
        L.ref_diag_flat.argtypes = [_i64, _dbl, _dbl, _vp]
        L.ref_diag_linear.argtypes = [_i64, _vp]
        L.ref_matrix_from_csr.argtypes = [C.c_int, _i64, _vp, _vp, _vp, _vp]
        L.ref_matrix_info.argtypes = [_vp, _vp, _vp, _vp]
        L.ref_matrix_csr.argtypes = [_vp, _vp, _vp, _vp]
        L.ref_randomize.argtypes = [C.c_int, _i64, _i64, _u64, _vp]
        L.ref_window_coeffs.argtypes = [_dbl, _dbl, _dbl, _dbl, C.c_int, _vp]
        L.ref_kernel_coeffs.argtypes = [C.c_int, C.c_int, C.c_int, _vp]
        L.ref_make_filter.argtypes = [_dbl, _dbl, _dbl, _dbl, C.c_int, C.c_int, C.c_int, _vp, _vp,
                                      _vp]
        L.ref_spmmvm.argtypes = [_vp, _vp, _i64, _dbl, _dbl, _vp]
        L.ref_spmmvm_fused.argtypes = [_vp, _vp, _vp, _vp, _i64, _dbl, _dbl, _dbl, _vp]
        L.ref_recurrence_step.argtypes = [_vp, _vp, _vp, _i64, _dbl, _dbl]
        L.ref_block_axpy_scal.argtypes = [C.c_int, _i64, _i64, _vp, _vp, _vp, _dbl, _dbl, _dbl]
        L.ref_gram.argtypes = [C.c_int, _i64, _vp, _i64, _vp, _i64, _vp]
        L.ref_column_dots.argtypes = [C.c_int, _i64, _i64, _vp, _vp, _vp]
        L.ref_column_norms.argtypes = [C.c_int, _i64, _i64, _vp, _vp]
        L.ref_block_mult_small.argtypes = [C.c_int, _i64, _i64, _vp, _vp, _i64, _vp]
        L.ref_apply_filter.argtypes = [_vp, _vp, _i64, _vp, C.c_int, _dbl, _dbl, _vp]
        L.ref_time_fused_steps.argtypes = [_vp, _i64, C.c_int, _dbl, _dbl, _dbl, _u64, _vp]
        L.ref_fused_session_create.argtypes = [_vp, _i64, _vp]
        L.ref_fused_session_run.argtypes = [_vp, C.c_int, _dbl, _dbl, _dbl, _vp]
        L.ref_fused_session_apply.argtypes = [_vp, _vp, C.c_int, _dbl, _dbl, _vp]
        L.ref_fused_session_gram.argtypes = [_vp, _vp]
        L.ref_fused_session_free.argtypes = [_vp]
        L.ref_fused_session_free.restype = None
        L.ref_svqb.argtypes = [C.c_int, _i64, _i64, _vp, _dbl, _vp, _vp]
        L.ref_rayleigh_ritz.argtypes = [_vp, _vp, _i64, _vp, _vp, _vp]
        L.ref_lanczos_bounds.argtypes = [_vp, C.c_int, _u64, _vp, _vp]
        L.ref_kpm_dos.argtypes = [_vp, _dbl, _dbl, C.c_int, C.c_int, _u64, _vp]
        L.ref_dos_count.argtypes = [_vp, C.c_int, _dbl, _dbl, _dbl, _dbl, _vp]
        L.ref_choose_parameters.argtypes = [_vp, C.c_int, _dbl, _dbl, _dbl, _dbl, _dbl, C.c_int,
                                            C.c_int, _dbl, _vp, _vp, _vp, _vp]
        L.ref_solve.argtypes = [_vp, _vp, _vp, C.c_int, _vp, _vp, _vp, _vp]
        L.ref_intensity_model.argtypes = [_dbl, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, _vp]
        L.ref_set_threads.argtypes = [C.c_int]
        L.ref_read_matrix_market.argtypes = [C.c_char_p, _vp, _vp]
        L.ref_write_matrix_market.argtypes = [_vp, C.c_char_p, C.c_int]
        L.ref_block_save.argtypes = [C.c_int, _i64, _i64, _vp, C.c_char_p]
        L.ref_block_load.argtypes = [C.c_int, C.c_char_p, _vp, _vp, _vp]
        L.ref_bench_filter.argtypes = [_vp, _vp, C.c_int, C.c_int, _dbl, _vp]
        L.ref_damping_factor.argtypes = [_dbl, _dbl, _dbl, _dbl, _dbl, C.c_int, C.c_int, C.c_int,
                                         _vp]
        if threads is not None:
            L.ref_set_threads(threads)

    def set_threads(self, n):
        self.lib.ref_set_threads(n)

    def num_threads(self):
        return self.lib.ref_num_threads()

    def _chk(self, rc):
        if rc:
            raise _REF_EXC.get(rc, RuntimeError)(self.lib.ref_last_error().decode())

    def _mat(self, fn, *args):
        h = _vp()
        self._chk(fn(*args, C.byref(h)))
        return RefMatrix(self, h)

    def graphene(self, lx, ly, t=1.0, disorder=0.0, boundary="periodic_xy_open_z", seed=1):
        return self._mat(self.lib.ref_graphene, lx, ly, t, disorder, BOUNDARY[boundary], seed)

    def topological_insulator(self, lx, ly, lz, t=1.0, disorder=0.0,
                              boundary="periodic_xy_open_z", seed=1):
        return self._mat(self.lib.ref_topological_insulator, lx, ly, lz, t, disorder,
                         BOUNDARY[boundary], seed)

    def diag_flat(self, dim, lo, hi):
        return self._mat(self.lib.ref_diag_flat, dim, lo, hi)

    def diag_linear(self, dim):
        return self._mat(self.lib.ref_diag_linear, dim)

    def from_csr(self, csr):
        return self._mat(self.lib.ref_matrix_from_csr, csr.kind, csr.dim, _ptr(csr.offs),
                         _ptr(csr.cols), _ptr(csr.vals))

    def randomize(self, dim, width, seed, complex_=False):
        out = np.empty((dim, width), dtype=np.complex128 if complex_ else np.float64)
        self._chk(self.lib.ref_randomize(int(complex_), dim, width, seed, _ptr(out)))
        return out

    def window_coeffs(self, target, bounds, degree):
        out = np.empty(degree + 1)
        self._chk(self.lib.ref_window_coeffs(target[0], target[1], bounds[0], bounds[1], degree,
                                             _ptr(out)))
        return out

    def kernel_coeffs(self, kernel, degree):
        k, mu = _kernel_code(kernel)
        out = np.empty(degree + 1)
        self._chk(self.lib.ref_kernel_coeffs(k, mu, degree, _ptr(out)))
        return out

    def make_filter(self, target, bounds, degree, kernel="lanczos2"):
        k, mu = _kernel_code(kernel)
        comb = np.empty(degree + 1)
        a, b = _dbl(), _dbl()
        self._chk(self.lib.ref_make_filter(target[0], target[1], bounds[0], bounds[1], degree, k,
                                           mu, _ptr(comb), C.byref(a), C.byref(b)))
        return comb, a.value, b.value

    def spmmvm(self, m, x, alpha, beta):
        x = np.ascontiguousarray(x)
        y = np.empty_like(x)
        self._chk(self.lib.ref_spmmvm(m.h, _ptr(x), x.shape[1], alpha, beta, _ptr(y)))
        return y

    def spmmvm_fused(self, m, u, w, x, alpha, beta, coeff, want_dots=False):
        dots = np.empty(u.shape[1], dtype=u.dtype) if want_dots else None
        self._chk(self.lib.ref_spmmvm_fused(m.h, _ptr(u), _ptr(w), _ptr(x), u.shape[1], alpha,
                                            beta, coeff, _ptr(dots)))
        return dots

    def recurrence_step(self, m, u, w, alpha, beta):
        self._chk(self.lib.ref_recurrence_step(m.h, _ptr(u), _ptr(w), u.shape[1], alpha, beta))

    def block_axpy_scal(self, x, u, w, c0, c1, c2):
        self._chk(self.lib.ref_block_axpy_scal(_kind(x), x.shape[0], x.shape[1], _ptr(x), _ptr(u),
                                               _ptr(w), c0, c1, c2))

    def gram(self, x, y):
        g = np.empty((x.shape[1], y.shape[1]), dtype=x.dtype)
        self._chk(self.lib.ref_gram(_kind(x), x.shape[0], _ptr(x), x.shape[1], _ptr(y),
                                    y.shape[1], _ptr(g)))
        return g

    def column_dots(self, x, y):
        d = np.empty(x.shape[1], dtype=x.dtype)
        self._chk(self.lib.ref_column_dots(_kind(x), x.shape[0], x.shape[1], _ptr(x), _ptr(y),
                                           _ptr(d)))
        return d

    def column_norms(self, x):
        out = np.empty(x.shape[1])
        self._chk(self.lib.ref_column_norms(_kind(x), x.shape[0], x.shape[1], _ptr(x), _ptr(out)))
        return out

    def block_mult_small(self, x, b):
        b = np.ascontiguousarray(b, dtype=x.dtype)
        y = np.empty((x.shape[0], b.shape[1]), dtype=x.dtype)
        self._chk(self.lib.ref_block_mult_small(_kind(x), x.shape[0], x.shape[1], _ptr(x), _ptr(b),
                                                b.shape[1], _ptr(y)))
        return y

    def apply_filter(self, m, x, combined, alpha, beta, want_moments=False):
        x = np.array(x, copy=True, order="C")
        comb = np.ascontiguousarray(combined, dtype=np.float64)
        degree = len(comb) - 1
        mom = np.empty((degree + 1, x.shape[1])) if want_moments else None
        self._chk(self.lib.ref_apply_filter(m.h, _ptr(x), x.shape[1], _ptr(comb), degree, alpha,
                                            beta, _ptr(mom)))
        return x, mom

    def time_fused_steps(self, m, width, steps, alpha=0.5, beta=0.0, coeff=0.25, seed=7):
        sec = _dbl()
        self._chk(self.lib.ref_time_fused_steps(m.h, width, steps, alpha, beta, coeff, seed,
                                                C.byref(sec)))
        return sec.value

    def fused_session(self, m, width):
        """Persistent U, W, X reference blocks for steady-state spmmvm_fused timing
        (timed reference arm / cpu_baseline): session.run(steps) -> seconds."""
        ref = self
        h = _vp()
        self._chk(self.lib.ref_fused_session_create(m.h, width, C.byref(h)))

        class _Session:
            def run(self, steps, alpha=0.37, beta=0.0, coeff=0.25):
                sec = _dbl()
                ref._chk(ref.lib.ref_fused_session_run(h, steps, alpha, beta, coeff,
                                                       C.byref(sec)))
                return sec.value

            def apply_filter(self, combined, alpha, beta):
                comb = np.ascontiguousarray(combined, dtype=np.float64)
                sec = _dbl()
                ref._chk(ref.lib.ref_fused_session_apply(h, _ptr(comb), len(comb) - 1, alpha,
                                                         beta, C.byref(sec)))
                return sec.value

            def gram(self):
                sec = _dbl()
                ref._chk(ref.lib.ref_fused_session_gram(h, C.byref(sec)))
                return sec.value

            def close(self):
                if h.value:
                    ref.lib.ref_fused_session_free(h)
                    h.value = None

            def __del__(self):
                self.close()

        return _Session()

    def svqb(self, y, drop_tol=1e-14):
        y = np.ascontiguousarray(y)
        q = np.empty_like(y)
        rank = _i64()
        self._chk(self.lib.ref_svqb(_kind(y), y.shape[0], y.shape[1], _ptr(y), drop_tol, _ptr(q),
                                    C.byref(rank)))
        return q[:, :rank.value].copy() if rank.value < y.shape[1] else q, rank.value

    def rayleigh_ritz(self, m, q):
        q = np.ascontiguousarray(q)
        v = np.empty_like(q)
        vals = np.empty(q.shape[1])
        res = np.empty(q.shape[1])
        self._chk(self.lib.ref_rayleigh_ritz(m.h, _ptr(q), q.shape[1], _ptr(v), _ptr(vals),
                                             _ptr(res)))
        return vals, v, res

    def lanczos_bounds(self, m, iters=30, seed=1):
        lo, hi = _dbl(), _dbl()
        self._chk(self.lib.ref_lanczos_bounds(m.h, iters, seed, C.byref(lo), C.byref(hi)))
        return lo.value, hi.value

    def kpm_dos(self, m, bounds, order, samples, seed=1):
        mu = np.empty(order + 1)
        self._chk(self.lib.ref_kpm_dos(m.h, bounds[0], bounds[1], order, samples, seed, _ptr(mu)))
        return mu

    def dos_count(self, mu, bounds, lo, hi):
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        out = _dbl()
        self._chk(self.lib.ref_dos_count(_ptr(mu), len(mu) - 1, bounds[0], bounds[1], lo, hi,
                                         C.byref(out)))
        return out.value

    def choose_parameters(self, mu, bounds, target, n_search, kernel="lanczos2", epsilon=1e-12):
        mu = np.ascontiguousarray(mu, dtype=np.float64)
        k, kmu = _kernel_code(kernel)
        np_opt, sigma, eta, dp = C.c_int(), _dbl(), _dbl(), _dbl()
        self._chk(self.lib.ref_choose_parameters(_ptr(mu), len(mu) - 1, bounds[0], bounds[1],
                                                 target[0], target[1], n_search, k, kmu, epsilon,
                                                 C.byref(np_opt), C.byref(sigma), C.byref(eta),
                                                 C.byref(dp)))
        return dict(np_opt=np_opt.value, sigma=sigma.value, eta=eta.value,
                    delta_prime=dp.value)

    def solve(self, m, target, epsilon=1e-10, n_search=0, degree=0, kernel="lanczos2",
              max_iters=40, seed=1, dos_moments=2000, dos_samples=32, bounds=(0.0, 0.0),
              collect_weight_density=True):
        k, mu = _kernel_code(kernel)
        o = _RefSolveOptions(target[0], target[1], epsilon, n_search, degree, k, mu, max_iters,
                             seed, dos_moments, dos_samples, bounds[0], bounds[1],
                             int(collect_weight_density))
        rep = _RefSolveReport()
        cap = 4096
        vals = np.zeros(cap)
        res = np.zeros(cap)
        acc = np.zeros(cap, dtype=np.int32)
        hist = np.zeros((max_iters, 5))
        self._chk(self.lib.ref_solve(m.h, C.byref(o), C.byref(rep), cap, _ptr(vals), _ptr(res),
                                     _ptr(acc), _ptr(hist)))
        n = rep.n_values
        out = {f: getattr(rep, f) for f, _ in _RefSolveReport._fields_}
        out.update(values=vals[:n].copy(), residual_norms=res[:n].copy(),
                   accepted=acc[:n].astype(bool), history=hist[:rep.iterations].copy())
        return out

    def intensity_model(self, n_nzr, s_d, s_i, f_a, f_m, n_b):
        out = _dbl()
        self._chk(self.lib.ref_intensity_model(n_nzr, s_d, s_i, f_a, f_m, n_b, C.byref(out)))
        return out.value

    # -- on-disk formats (matrix_market.cpp, block_vector.hpp:63-96) ------
    def read_matrix_market(self, path):
        """-> (RefMatrix, hermitian flag)"""
        h, herm = _vp(), C.c_int()
        self._chk(self.lib.ref_read_matrix_market(os.fsencode(path), C.byref(h), C.byref(herm)))
        return RefMatrix(self, h), bool(herm.value)

    def write_matrix_market(self, m, path, hermitian=True):
        self._chk(self.lib.ref_write_matrix_market(m.h, os.fsencode(path), int(hermitian)))

    def block_save(self, block, path):
        a = np.ascontiguousarray(block)
        kind = int(np.iscomplexobj(a))
        self._chk(self.lib.ref_block_save(kind, a.shape[0], a.shape[1], _ptr(a), os.fsencode(path)))

    def block_load(self, path, complex_=False):
        d, w = _i64(), _i64()
        self._chk(self.lib.ref_block_load(int(complex_), os.fsencode(path), C.byref(d), C.byref(w),
                                          None))
        out = np.empty((d.value, w.value), np.complex128 if complex_ else np.float64)
        self._chk(self.lib.ref_block_load(int(complex_), os.fsencode(path), C.byref(d), C.byref(w),
                                          _ptr(out)))
        return out

    def bench_filter(self, m, sizes, degree, bandwidth):
        """-> (n, 8) rows: n_b, seconds, flops, gflops, gbs_proxy, intensity, roofline,
        efficiency (bench.cpp:71-126)"""
        sz = np.ascontiguousarray(sizes, dtype=np.int32)
        out = np.zeros((len(sz), 8))
        self._chk(self.lib.ref_bench_filter(m.h, _ptr(sz), len(sz), degree, bandwidth, _ptr(out)))
        return out

    def damping_factor(self, target, delta_prime, bounds, degree, kernel="lanczos2"):
        k, kmu = _kernel_code(kernel)
        out = _dbl()
        self._chk(self.lib.ref_damping_factor(target[0], target[1], delta_prime, bounds[0],
                                              bounds[1], degree, k, kmu, C.byref(out)))
        return out.value


def ref_available():
    return os.path.exists(REF_SO)
