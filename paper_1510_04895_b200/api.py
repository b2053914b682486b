"""Python mirror of the reference's ChebFD driver API, backed by the sm_100a
library through its C ABI (include/chebfd_b200.h).

Names, argument meaning and error behaviour follow the reference's C++ API
(/root/reference/proj/include/chebfd/*.hpp); every device call goes through
libchebfd_b200.so -- there is no CPU fallback.  C++ exception types map to
Python exceptions: std::invalid_argument -> InvalidArgument (ValueError),
std::runtime_error -> NumericalError (RuntimeError), std::domain_error ->
DomainError (ValueError), std::out_of_range -> OutOfRange (IndexError).
"""
from __future__ import annotations

import ctypes as C
import os
import weakref
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib as L

REAL64, COMPLEX128 = 0, 1
BOUNDARY = {"periodic_xy_open_z": 0, "periodic_all": 1, "open_all": 2}
KERNELS = {"none": 0, "fejer": 1, "jackson": 2, "lanczos": 3}


# ------------------------------------------------------------------ errors --
class ChebfdError(Exception):
    code = -1


class InvalidArgument(ChebfdError, ValueError):
    code = 1


class NumericalError(ChebfdError, RuntimeError):
    code = 2


class DomainError(ChebfdError, ValueError):
    code = 3


class OutOfRange(ChebfdError, IndexError):
    code = 4


class CudaError(ChebfdError, RuntimeError):
    code = 5


class NcclError(ChebfdError, RuntimeError):
    code = 6


class Unsupported(ChebfdError, NotImplementedError):
    code = 7


_EXC = {c.code: c for c in (InvalidArgument, NumericalError, DomainError, OutOfRange, CudaError,
                            NcclError, Unsupported)}


def _lib():
    return L.load()


def _check(rc):
    if rc:
        msg = _lib().chebfd_last_error().decode()
        raise _EXC.get(rc, ChebfdError)(msg)


def experimental_build() -> bool:
    """True when the library was built with the opt-in slower kernel variants
    (make EXPERIMENTAL=1): the pair kernel and kernel variant 2."""
    return bool(_lib().chebfd_build_features() & 1)


def _ptr(a):
    return None if a is None else a.ctypes.data_as(C.c_void_p)


# ----------------------------------------------------------------- context --
class Context:
    """One GPU, one stream (replaces the reference's OpenMP runtime,
    parallel.hpp:18-54).  ``Context.distributed(rank, nranks, uid)`` joins a
    row-partitioned multi-GPU context (one process per GPU)."""

    def __init__(self, device: int = 0, _handle=None, _borrowed=False):
        self._h = C.c_void_p()
        self._children = weakref.WeakSet()  # matrices / blocks to release first
        self._borrowed = _borrowed  # a virtual group's rank context: the group destroys it
        if _handle is None:
            _check(_lib().chebfd_ctx_create(device, C.byref(self._h)))
        else:
            self._h = _handle

    def _adopt(self, obj):
        self._children.add(obj)

    @staticmethod
    def nccl_unique_id() -> bytes:
        buf = (C.c_ubyte * 128)()
        _check(_lib().chebfd_nccl_unique_id(buf))
        return bytes(buf)

    @classmethod
    def distributed(cls, device: int, rank: int, nranks: int, uid: bytes):
        h = C.c_void_p()
        buf = (C.c_ubyte * 128).from_buffer_copy(uid)
        _check(_lib().chebfd_ctx_create_dist(device, rank, nranks, buf, C.byref(h)))
        return cls(_handle=h)

    def close(self):
        """Release every block and matrix of this context, then the context."""
        if getattr(self, "_h", None) and self._h.value:
            kids = list(self._children)
            for k in kids:  # blocks before matrices (blocks reference matrices)
                if isinstance(k, BlockVector):
                    k.close()
            for k in kids:
                k.close()
            if not self._borrowed:
                _lib().chebfd_ctx_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def synchronize(self):
        _check(_lib().chebfd_ctx_synchronize(self._h))

    @property
    def stream(self) -> int:
        s = C.c_void_p()
        _check(_lib().chebfd_ctx_stream(self._h, C.byref(s)))
        return s.value or 0

    def info(self):
        d, r, n, s = C.c_int(), C.c_int(), C.c_int(), C.c_int()
        _check(_lib().chebfd_ctx_info(self._h, C.byref(d), C.byref(r), C.byref(n), C.byref(s)))
        return dict(device=d.value, rank=r.value, nranks=n.value, num_sms=s.value)

    @property
    def launch_count(self) -> int:
        v = C.c_int64()
        _check(_lib().chebfd_ctx_launch_count(self._h, C.byref(v)))
        return v.value

    @property
    def group_launches(self) -> int:
        """Step launches that ran the row-group kernel (option "grouped")."""
        v = C.c_int64()
        _check(_lib().chebfd_ctx_group_launches(self._h, C.byref(v)))
        return v.value

    @property
    def ring_launches(self) -> int:
        """Step launches that ran the site-ring kernel (option "ring")."""
        v = C.c_int64()
        _check(_lib().chebfd_ctx_ring_launches(self._h, C.byref(v)))
        return v.value

    @property
    def band_launches(self) -> int:
        """Step launches that ran in the band (2.5D) tile order."""
        v = C.c_int64()
        _check(_lib().chebfd_ctx_band_launches(self._h, C.byref(v)))
        return v.value

    def record(self, slot: int):
        """Record CUDA event `slot` (0..15) on the context stream."""
        _check(_lib().chebfd_ctx_event_record(self._h, slot))

    def elapsed_ms(self, a: int, b: int) -> float:
        ms = C.c_float()
        _check(_lib().chebfd_ctx_event_elapsed(self._h, a, b, C.byref(ms)))
        return ms.value

    def set_option(self, name: str, value):
        """graphs (bool), overlap (bool), kernel ("gather" | "tma"),
        slab_units (int, 0 = 256), pair (0 off | 1 auto | 2 force: two fused
        steps per wavefront launch), pair_tile_rows / pair_threads /
        pair_extra (pair-kernel tuning, 0 / 0 / -1 = automatic), moments
        ("direct" | "doubling": how filter / KPM moments are formed)."""
        code = {"graphs": 1, "overlap": 2, "kernel": 3, "slab_units": 5, "pair": 6,
                "pair_tile_rows": 7, "pair_threads": 8, "pair_extra": 9, "pair_hints": 10,
                "pair_slab": 11, "moments": 12, "pdl": 14, "delayed_x": 15,
                "band_bytes": 16, "async_start": 17, "tiles_per_cta": 18,
                "compact_halo": 19, "gram": 20, "grouped": 21, "group_lines": 22,
                "ring": 23, "ring_segx": 24, "ring_no": 25, "ring_nz": 26,
                "ring_rows": 27, "ring_consts": 28, "ring_tmap": 29,
                "ring_order": 30, "ring_unit": 31, "ring_dots": 32}[name]
        if name == "moments" and isinstance(value, str):
            value = {"direct": 0, "doubling": 1}[value]
        if name == "kernel" and isinstance(value, str):
            value = {"gather": 0, "tma": 1, "stage": 2, "tma2": 3}[value]
        _check(_lib().chebfd_ctx_set_option(self._h, code, int(value)))


# ------------------------------------------------------------- intervals --
@dataclass
class Interval:
    """filter.hpp:19-26"""
    lo: float = 0.0
    hi: float = 0.0

    def width(self):
        return self.hi - self.lo

    def half_width(self):
        return 0.5 * (self.hi - self.lo)

    def center(self):
        return 0.5 * (self.lo + self.hi)

    def contains(self, x):
        if isinstance(x, Interval):
            return self.lo <= x.lo and x.hi <= self.hi
        return self.lo <= x <= self.hi


def _iv(x) -> Interval:
    return x if isinstance(x, Interval) else Interval(float(x[0]), float(x[1]))


@dataclass
class Kernel:
    """Damping kernel (filter.hpp:12-17): kind in none/fejer/jackson/lanczos."""
    kind: str = "lanczos"
    mu: int = 2

    def name(self) -> str:
        return f"lanczos{self.mu}" if self.kind == "lanczos" else self.kind

    @staticmethod
    def parse(s: str) -> "Kernel":
        if s in ("none", "fejer", "jackson"):
            return Kernel(s, 0)
        if s.startswith("lanczos"):
            mu = int(s[7:]) if len(s) > 7 else 2
            if mu < 1:
                raise InvalidArgument("lanczos kernel needs mu >= 1")
            return Kernel("lanczos", mu)
        raise InvalidArgument("unknown kernel: " + s)

    def code(self):
        return KERNELS[self.kind], self.mu


def _kernel(k) -> Kernel:
    return k if isinstance(k, Kernel) else Kernel.parse(k)


@dataclass
class LatticeSpec:
    """models.hpp:19-29 (onsite_potential not supported)."""
    lx: int = 1
    ly: int = 1
    lz: int = 1
    t: float = 1.0
    disorder: float = 0.0
    boundary: str = "periodic_xy_open_z"
    seed: int = 1

    def _c(self):
        return L.chebfd_lattice(self.lx, self.ly, self.lz, self.t, self.disorder,
                                BOUNDARY[self.boundary], self.seed)


# ---------------------------------------------------------- host CSR gen --
def csr_graphene(spec: LatticeSpec, row_begin=0, row_end=None):
    """Host CSR of graphene() rows (models.cpp:142-178), stencil-direct."""
    return _csr(_lib().chebfd_csr_graphene, spec, row_begin, row_end, np.float64)


def csr_topological_insulator(spec: LatticeSpec, row_begin=0, row_end=None):
    """Host CSR of topological_insulator() rows (models.cpp:80-140)."""
    return _csr(_lib().chebfd_csr_topological_insulator, spec, row_begin, row_end, np.complex128)


def _csr(fn, spec, r0, r1, dtype):
    s = spec._c()
    dim, nnz = C.c_int64(), C.c_int64()
    if r1 is None:
        _check(fn(C.byref(s), 0, 0, C.byref(dim), C.byref(nnz), None, None, None))
        r1 = dim.value
    _check(fn(C.byref(s), r0, r1, C.byref(dim), C.byref(nnz), None, None, None))
    offs = np.empty(r1 - r0 + 1, np.int64)
    cols = np.empty(nnz.value, np.int64)
    vals = np.empty(nnz.value, dtype)
    _check(fn(C.byref(s), r0, r1, C.byref(dim), C.byref(nnz), _ptr(offs), _ptr(cols), _ptr(vals)))
    return offs, cols, vals


# --------------------------------------------------------- virtual ranks --
class VirtualGroup:
    """The distributed filter's ranks on ONE GPU (chebfd_vgroup_*, vgroup.cu): each rank
    a Context with its row partition and halos, all ranks' steps enqueued in lockstep
    with the halo rows pulled from the neighbours' blocks (optionally one CUDA graph).
    Results equal the single-rank path's bits; dots / moments / Gram summed over ranks."""

    def __init__(self, nranks: int, device: int = 0):
        self._h = C.c_void_p()
        _check(_lib().chebfd_vgroup_create(device, nranks, C.byref(self._h)))
        self.nranks = nranks
        self.ranks = []
        for r in range(nranks):
            h = C.c_void_p()
            _check(_lib().chebfd_vgroup_context(self._h, r, C.byref(h)))
            self.ranks.append(Context(_handle=h, _borrowed=True))

    def set_option(self, name: str, value):
        code = {"graphs": 1}.get(name)
        if code is not None:
            _check(_lib().chebfd_vgroup_set_option(self._h, code, int(value)))
            return
        for c in self.ranks:
            c.set_option(name, value)

    def _lattice(self, model, spec):
        hs = (C.c_void_p * self.nranks)()
        s = spec._c()
        _check(_lib().chebfd_vgroup_matrix_lattice(self._h, model, C.byref(s), hs))
        return [SparseMatrix(self.ranks[r], C.c_void_p(hs[r])) for r in range(self.nranks)]

    def topological_insulator(self, spec: "LatticeSpec"):
        return self._lattice(1, spec)

    def graphene(self, spec: "LatticeSpec"):
        return self._lattice(0, spec)

    @staticmethod
    def _arr(objs):
        a = (C.c_void_p * len(objs))()
        for i, o in enumerate(objs):
            a[i] = o._h.value
        return a

    def apply_filter(self, As, Xs, p: "FilterPolynomial", want_moments=False):
        comb = np.ascontiguousarray(p.combined, dtype=np.float64)
        nb = Xs[0].width_
        mom = np.empty((p.degree + 1, nb)) if want_moments else None
        _check(_lib().chebfd_vgroup_apply_filter(self._h, self._arr(As), self._arr(Xs), _ptr(comb),
                                                 p.degree, p.alpha, p.beta, _ptr(mom)))
        return MomentTable(p.degree, nb, mom) if want_moments else None

    def spmmvm_fused(self, As, Us, Ws, Xs, alpha, beta, coeff, dots=False):
        d = np.empty(Us[0].width_, dtype=Us[0].dtype) if dots else None
        _check(_lib().chebfd_vgroup_spmmvm_fused(self._h, self._arr(As), self._arr(Us),
                                                 self._arr(Ws), self._arr(Xs), alpha, beta, coeff,
                                                 _ptr(d)))
        return d

    def gram(self, Xs, Ys):
        g = np.empty((Xs[0].width_, Ys[0].width_), dtype=Xs[0].dtype)
        _check(_lib().chebfd_vgroup_gram(self._h, self._arr(Xs), self._arr(Ys), _ptr(g)))
        return g

    @staticmethod
    def halo_rows(A):
        v = [C.c_int64() for _ in range(4)]
        _check(_lib().chebfd_vgroup_halo_rows(A._h, *[C.byref(x) for x in v]))
        return dict(halo_lo=v[0].value, halo_hi=v[1].value, send_lo=v[2].value, send_hi=v[3].value)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            for c in self.ranks:
                c.close()
            _lib().chebfd_vgroup_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ----------------------------------------------------------- sparse matrix --
class SparseMatrix:
    """Device SELL-C-sigma matrix (C = 32, sigma = 1); replaces
    SparseMatrix<S> (sparse_matrix.hpp:15-107)."""

    def __init__(self, ctx: Context, handle):
        self.ctx = ctx
        self._h = handle
        ctx._adopt(self)
        info = L.chebfd_matrix_info()
        _check(_lib().chebfd_matrix_get_info(self._h, C.byref(info)))
        self.info = {f: getattr(info, f) for f, _ in L.chebfd_matrix_info._fields_}

    @classmethod
    def from_csr(cls, ctx, dim, row_offsets, col_indices, values):
        offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
        cols = np.ascontiguousarray(col_indices, dtype=np.int64)
        vals = np.ascontiguousarray(values)
        if len(offs) != dim + 1:
            raise InvalidArgument("SparseMatrix: row_offsets length must be dim+1")
        if len(cols) != len(vals):
            raise InvalidArgument("SparseMatrix: col/value length mismatch")
        if offs[-1] != len(vals):
            raise InvalidArgument("SparseMatrix: invalid row_offsets range")
        kind = COMPLEX128 if np.iscomplexobj(vals) else REAL64
        vals = vals.astype(np.complex128 if kind else np.float64, copy=False)
        h = C.c_void_p()
        _check(_lib().chebfd_matrix_from_csr(ctx._h, kind, dim, _ptr(offs), _ptr(cols), _ptr(vals),
                                              C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def from_matrix_market(cls, ctx, path):
        """read_matrix_market (matrix_market.cpp:98-115) straight to the device."""
        h = C.c_void_p()
        _check(_lib().chebfd_matrix_from_matrix_market(ctx._h, os.fsencode(path), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def graphene(cls, ctx, spec: LatticeSpec):
        h = C.c_void_p()
        s = spec._c()
        _check(_lib().chebfd_matrix_graphene(ctx._h, C.byref(s), C.byref(h)))
        return cls(ctx, h)

    @classmethod
    def topological_insulator(cls, ctx, spec: LatticeSpec):
        h = C.c_void_p()
        s = spec._c()
        _check(_lib().chebfd_matrix_topological_insulator(ctx._h, C.byref(s), C.byref(h)))
        return cls(ctx, h)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib().chebfd_matrix_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def dim(self):
        return self.info["dim"]

    def nnz(self):
        return self.info["nnz"]

    @property
    def kind(self):
        return self.info["kind"]

    @property
    def dtype(self):
        return np.complex128 if self.kind else np.float64

    def avg_nonzeros_per_row(self):
        return self.nnz() / self.dim() if self.dim() else 0.0

    @property
    def local_rows(self):
        return self.info["local_rows"]

    @property
    def row_begin(self):
        return self.info["row_begin"]


# ------------------------------------------------------------ block vector --
class BlockVector:
    """Device D x n_b row-major block (block_vector.hpp:17-102).  Created
    conforming to a matrix (owned rows of this rank, halo storage for
    gathers) or free-standing by (ctx, dim, width, kind)."""

    def __init__(self, A: Optional[SparseMatrix] = None, width: int = 1, *, ctx=None, dim=None,
                 kind=None, _handle=None):
        self.A = A
        if _handle is not None:
            self._h = _handle
        elif A is not None:
            self._h = C.c_void_p()
            _check(_lib().chebfd_block_create(A._h, width, C.byref(self._h)))
        else:
            self._h = C.c_void_p()
            _check(_lib().chebfd_block_create_dim(ctx._h, kind, dim, width, C.byref(self._h)))
        self.ctx = ctx if ctx is not None else A.ctx
        self.ctx._adopt(self)
        k, r, w, rb = C.c_int(), C.c_int64(), C.c_int64(), C.c_int64()
        _check(_lib().chebfd_block_info(self._h, C.byref(k), C.byref(r), C.byref(w), C.byref(rb)))
        self.kind, self.rows, self.width_, self.row_begin = k.value, r.value, w.value, rb.value

    @classmethod
    def like(cls, other: "BlockVector", width=None):
        w = other.width_ if width is None else width
        if other.A is not None:
            return cls(other.A, w)
        return cls(ctx=other.ctx, dim=other.rows, width=w, kind=other.kind)

    def close(self):
        if getattr(self, "_h", None) and self._h.value:
            _lib().chebfd_block_destroy(self._h)
            self._h = C.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def dim(self):
        return self.rows

    def width(self):
        return self.width_

    @property
    def dtype(self):
        return np.complex128 if self.kind else np.float64

    @property
    def shape(self):
        return (self.rows, self.width_)

    def upload(self, host: np.ndarray):
        a = np.ascontiguousarray(host, dtype=self.dtype)
        if a.shape != self.shape:
            raise InvalidArgument(f"upload: shape {a.shape} != {self.shape}")
        _check(_lib().chebfd_block_upload(self._h, _ptr(a)))
        return self

    def to_numpy(self) -> np.ndarray:
        out = np.empty(self.shape, dtype=self.dtype)
        _check(_lib().chebfd_block_download(self._h, _ptr(out)))
        return out

    def save(self, path):
        """BlockVector::save (block_vector.hpp:65-78): .cbfd dump of the block."""
        _check(_lib().chebfd_block_save(self._h, os.fsencode(path)))

    @classmethod
    def load(cls, A: SparseMatrix, path) -> "BlockVector":
        """BlockVector::load (block_vector.hpp:80-95) into a block conforming to A."""
        h = C.c_void_p()
        _check(_lib().chebfd_block_load(A._h, os.fsencode(path), C.byref(h)))
        return cls(A, _handle=h)

    def copy_from(self, other: "BlockVector"):
        _check(_lib().chebfd_block_copy(self._h, other._h))
        return self

    def zero(self):
        _check(_lib().chebfd_block_zero(self._h))
        return self

    def randomize(self, seed: int):
        """BlockVector::randomize (block_vector.hpp:42-51), same stream."""
        _check(_lib().chebfd_block_randomize(self._h, seed))
        return self

    def randomize_device(self, seed: int):
        """Fast device Gaussian fill (Philox) -- not the reference stream."""
        _check(_lib().chebfd_block_randomize_device(self._h, seed))
        return self

    def scale_columns(self, s):
        s = np.ascontiguousarray(s, dtype=np.float64)
        _check(_lib().chebfd_block_scale_columns(self._h, _ptr(s)))
        return self

    def copy_columns(self, d0, src: "BlockVector", s0, n):
        _check(_lib().chebfd_block_copy_columns(self._h, d0, src._h, s0, n))
        return self

    @property
    def device_ptr(self) -> int:
        p = C.c_void_p()
        _check(_lib().chebfd_block_device_ptr(self._h, C.byref(p)))
        return p.value


# ------------------------------------------------------------------ kernels --
def spmmvm(A: SparseMatrix, X: BlockVector, alpha: float, beta: float) -> BlockVector:
    """Y = (alpha A + beta I) X  (kernels.hpp:45-69)."""
    Y = BlockVector.like(X)
    _check(_lib().chebfd_spmmvm(A._h, X._h, Y._h, alpha, beta))
    return Y


def spmmvm_fused(A, U, W, X, alpha, beta, coeff, dots: bool = False):
    """W <- 2(alpha A + beta)U - W;  X <- X + coeff W  (kernels.hpp:71-118).
    Returns d_k = <x_k(before), w_k(after)> when dots=True."""
    d = np.empty(U.width_, dtype=U.dtype) if dots else None
    _check(_lib().chebfd_spmmvm_fused(A._h, U._h, W._h, X._h, alpha, beta, coeff, _ptr(d)))
    return d


def recurrence_step(A, U, W, alpha, beta):
    """W <- 2(alpha A + beta)U - W  (kernels.hpp:120-145)."""
    _check(_lib().chebfd_recurrence_step(A._h, U._h, W._h, alpha, beta))


def block_axpy_scal(X, U, W, c0, c1, c2):
    """X <- c0 X + c1 U + c2 W  (kernels.hpp:147-162)."""
    _check(_lib().chebfd_block_axpy_scal(X._h, U._h, W._h, c0, c1, c2))


def column_dots(X, Y) -> np.ndarray:
    """d_k = <x_k, y_k>  (kernels.hpp:194-213)."""
    d = np.empty(X.width_, dtype=X.dtype)
    _check(_lib().chebfd_column_dots(X._h, Y._h, _ptr(d)))
    return d


def column_norms(X) -> np.ndarray:
    out = np.empty(X.width_)
    _check(_lib().chebfd_column_norms(X._h, _ptr(out)))
    return out


def gram(X, Y) -> np.ndarray:
    """G(k,l) = <x_k, y_l>  (kernels.hpp:164-192)."""
    g = np.empty((X.width_, Y.width_), dtype=X.dtype)
    _check(_lib().chebfd_gram(X._h, Y._h, _ptr(g)))
    return g


def block_mult_small(X, B) -> BlockVector:
    """Y = X B with a small dense B  (kernels.hpp:215-232)."""
    B = np.ascontiguousarray(B, dtype=X.dtype)
    if B.ndim != 2 or B.shape[0] != X.width_:
        raise InvalidArgument("block_mult_small: shape mismatch")
    Y = BlockVector.like(X, width=B.shape[1])
    _check(_lib().chebfd_block_mult_small(X._h, _ptr(B), B.shape[1], Y._h))
    return Y


# ------------------------------------------------------------------ filter --
def window_coeffs(target, bounds, degree: int) -> np.ndarray:
    t, b = _iv(target), _iv(bounds)
    out = np.empty(max(degree, 0) + 1)
    _check(_lib().chebfd_window_coeffs(t.lo, t.hi, b.lo, b.hi, degree, _ptr(out)))
    return out


def kernel_coeffs(kernel, degree: int) -> np.ndarray:
    k, mu = _kernel(kernel).code()
    out = np.empty(max(degree, 0) + 1)
    _check(_lib().chebfd_kernel_coeffs(k, mu, degree, _ptr(out)))
    return out


@dataclass
class FilterPolynomial:
    """filter.hpp:39-46"""
    degree: int = 0
    combined: np.ndarray = field(default_factory=lambda: np.zeros(0))
    alpha: float = 1.0
    beta: float = 0.0
    target: Interval = field(default_factory=Interval)
    bounds: Interval = field(default_factory=Interval)
    kernel: Kernel = field(default_factory=Kernel)


def make_filter(target, bounds, degree: int, kernel="lanczos2") -> FilterPolynomial:
    """combined[n] = g_n c_n  (filter.cpp:86-99)."""
    t, b, k = _iv(target), _iv(bounds), _kernel(kernel)
    kk, mu = k.code()
    comb = np.empty(max(degree, 0) + 1)
    a, be = C.c_double(), C.c_double()
    _check(_lib().chebfd_make_filter(t.lo, t.hi, b.lo, b.hi, degree, kk, mu, _ptr(comb),
                                     C.byref(a), C.byref(be)))
    return FilterPolynomial(degree, comb, a.value, be.value, t, b, k)


def eval_scalar(p: FilterPolynomial, x: float) -> float:
    out = C.c_double()
    comb = np.ascontiguousarray(p.combined, dtype=np.float64)
    _check(_lib().chebfd_eval_scalar(_ptr(comb), p.degree, p.alpha, p.beta, p.bounds.lo,
                                     p.bounds.hi, x, C.byref(out)))
    return out.value


@dataclass
class MomentTable:
    """filter.hpp:61-68: m(n,k) = <x_k, T_n(alpha A + beta) x_k>."""
    degree: int
    width: int
    m: np.ndarray  # (degree+1, width)

    def __call__(self, n, k):
        return self.m[n, k]


def apply_filter(A: SparseMatrix, X: BlockVector, p: FilterPolynomial,
                 want_moments: bool = False) -> Optional[MomentTable]:
    """X <- p[A] X in exactly Np*n_b column spMVMs (filter.hpp:73-116)."""
    comb = np.ascontiguousarray(p.combined, dtype=np.float64)
    if len(comb) < p.degree + 1 and p.degree >= 2:
        raise InvalidArgument("apply_filter: coefficient array shorter than degree+1")
    mom = np.empty((max(p.degree, 0) + 1, X.width_)) if want_moments else None
    _check(_lib().chebfd_apply_filter(A._h, X._h, _ptr(comb), p.degree, p.alpha, p.beta,
                                      _ptr(mom)))
    return MomentTable(p.degree, X.width_, mom) if want_moments else None


def apply_filter_host(A: SparseMatrix, x: np.ndarray, p: FilterPolynomial,
                      want_moments: bool = False):
    """End-to-end filter of a HOST block (in place): H2D, filter, D2H."""
    if x.dtype != A.dtype or not x.flags.c_contiguous:
        raise InvalidArgument("apply_filter_host: x must be C-contiguous of the matrix dtype")
    if x.ndim != 2 or x.shape[0] != A.local_rows or x.shape[1] < 1:
        raise InvalidArgument("apply_filter_host: x must be (local rows x width) "
                              f"= ({A.local_rows}, n_b), got {x.shape}")
    comb = np.ascontiguousarray(p.combined, dtype=np.float64)
    if p.degree >= 2 and len(comb) < p.degree + 1:
        raise InvalidArgument("apply_filter: coefficient array shorter than degree+1")
    mom = np.empty((p.degree + 1, x.shape[1])) if want_moments else None
    _check(_lib().chebfd_apply_filter_host(A._h, _ptr(x), x.shape[1], _ptr(comb), p.degree,
                                           p.alpha, p.beta, _ptr(mom)))
    return MomentTable(p.degree, x.shape[1], mom) if want_moments else None


class FilterPipe:
    """Streamed end-to-end filtering of host blocks (chebfd_filter_pipe_*): the
    H2D copy of job k and the D2H copy of job k-2 overlap the filter of job k-1.
    Host arrays must stay alive until wait(); pinned ones (host_array) copy at
    full PCIe speed."""

    def __init__(self, A: SparseMatrix, width: int):
        self.A = A
        self.width_ = int(width)
        self._h = C.c_void_p()
        _check(_lib().chebfd_filter_pipe_create(A._h, self.width_, C.byref(self._h)))
        self._keep = []

    def submit(self, x_in: np.ndarray, p: "FilterPolynomial", x_out: Optional[np.ndarray] = None,
               gram_out: Optional[np.ndarray] = None):
        """Queue one filter of x_in (result in x_out, default in place); with gram_out
        (width x width, matrix dtype) also the Gram X^H X of the filtered block.  Pass
        pinned arrays (host_array): copies to or from pageable memory block the host until
        the stream reaches them, which serialises the pipeline."""
        x_out = x_in if x_out is None else x_out
        for x in (x_in, x_out):
            if x.dtype != self.A.dtype or not x.flags.c_contiguous or x.shape != (self.A.local_rows, self.width_):
                raise InvalidArgument("filter_pipe: host block must be C-contiguous "
                                      "(local rows x width) of the matrix dtype")
        comb = np.ascontiguousarray(p.combined, dtype=np.float64)
        if p.degree >= 2 and len(comb) < p.degree + 1:
            raise InvalidArgument("apply_filter: coefficient array shorter than degree+1")
        if gram_out is not None:
            if (gram_out.dtype != self.A.dtype or not gram_out.flags.c_contiguous
                    or gram_out.shape != (self.width_, self.width_)):
                raise InvalidArgument("filter_pipe: gram_out must be C-contiguous (width x width)")
            self._keep.append((x_in, x_out, gram_out))
            _check(_lib().chebfd_filter_pipe_submit_gram(self._h, _ptr(x_in), _ptr(x_out),
                                                         _ptr(comb), p.degree, p.alpha, p.beta,
                                                         _ptr(gram_out)))
            return
        self._keep.append((x_in, x_out))
        _check(_lib().chebfd_filter_pipe_submit(self._h, _ptr(x_in), _ptr(x_out), _ptr(comb),
                                                p.degree, p.alpha, p.beta))

    def wait(self):
        _check(_lib().chebfd_filter_pipe_wait(self._h))
        self._keep.clear()

    def close(self):
        if self._h:
            _check(_lib().chebfd_filter_pipe_destroy(self._h))
            self._h = None
        self._keep.clear()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def host_array(shape, dtype):
    """A numpy array over pinned host memory (chebfd_host_alloc); freed with the array."""
    dt = np.dtype(dtype)
    nbytes = int(np.prod(shape)) * dt.itemsize
    ptr = C.c_void_p()
    _check(_lib().chebfd_host_alloc(max(nbytes, 1), C.byref(ptr)))
    buf = (C.c_char * max(nbytes, 1)).from_address(ptr.value)
    arr = np.frombuffer(buf, dtype=dt, count=int(np.prod(shape))).reshape(shape)
    weakref.finalize(buf, _lib().chebfd_host_free, C.c_void_p(ptr.value))
    return arr


# ------------------------------------------------------------------ solver --
@dataclass
class SvqbResult:
    q: BlockVector
    rank: int


def svqb_orthonormalize(Y: BlockVector, drop_tol: float = 1e-14) -> SvqbResult:
    """solver.cpp:32-61.  q keeps Y's width; columns >= rank are zero."""
    Q = BlockVector.like(Y)
    r = C.c_int64()
    _check(_lib().chebfd_svqb(Y._h, drop_tol, Q._h, C.byref(r)))
    return SvqbResult(Q, r.value)


@dataclass
class RitzSet:
    """solver.hpp:27-33"""
    values: np.ndarray
    vectors: Optional[BlockVector]
    residual_norms: np.ndarray
    accepted: np.ndarray


def rayleigh_ritz(A: SparseMatrix, Q: BlockVector) -> RitzSet:
    """solver.cpp:63-91"""
    V = BlockVector.like(Q)
    vals = np.empty(Q.width_)
    res = np.empty(Q.width_)
    _check(_lib().chebfd_rayleigh_ritz(A._h, Q._h, V._h, _ptr(vals), _ptr(res)))
    return RitzSet(vals, V, res, np.zeros(Q.width_, dtype=bool))


def lanczos_bounds(A: SparseMatrix, iters: int = 30, seed: int = 1) -> Interval:
    """spectral.cpp:96-154"""
    lo, hi = C.c_double(), C.c_double()
    _check(_lib().chebfd_lanczos_bounds(A._h, iters, seed, C.byref(lo), C.byref(hi)))
    return Interval(lo.value, hi.value)


@dataclass
class DosEstimate:
    """spectral.hpp:55-79 (Jackson-damped Chebyshev moments)."""
    moments: np.ndarray
    bounds: Interval
    num_samples: int = 0
    matrix_dim: int = 0

    def count(self, lo, hi) -> float:
        mu = np.ascontiguousarray(self.moments, dtype=np.float64)
        out = C.c_double()
        _check(_lib().chebfd_dos_count(_ptr(mu), len(mu) - 1, self.bounds.lo, self.bounds.hi,
                                       lo, hi, C.byref(out)))
        return out.value

    def density(self, lam) -> float:
        """ChebSeriesDensity::density (spectral.cpp:31-44)."""
        mu = np.ascontiguousarray(self.moments, dtype=np.float64)
        out = C.c_double()
        _check(_lib().chebfd_dos_density(_ptr(mu), len(mu) - 1, self.bounds.lo, self.bounds.hi,
                                         float(lam), C.byref(out)))
        return out.value


@dataclass
class WeightDensity:
    """Search-space weight density w(lambda) (spectral.hpp:57-72): the summed filter
    moments as a Jackson-damped Chebyshev series; integrates to N_S."""
    moments: np.ndarray
    bounds: Interval

    def _series(self):
        return DosEstimate(self.moments, self.bounds)

    def density(self, lam) -> float:
        return self._series().density(lam)

    def count(self, lo, hi) -> float:
        return self._series().count(lo, hi)

    def integral(self) -> float:
        return float(self.moments[0]) if len(self.moments) else 0.0


def weight_density(moments: "MomentTable", bounds) -> WeightDensity:
    """spectral.cpp:81-88: mu[n] = sum_k m(n, k)."""
    m = np.ascontiguousarray(moments.m, dtype=np.float64)
    mu = np.empty(max(int(moments.degree), 0) + 1)
    _check(_lib().chebfd_weight_density(_ptr(m), int(moments.degree), int(moments.width), _ptr(mu)))
    return WeightDensity(mu, _iv(bounds))


def kpm_dos(A: SparseMatrix, bounds, order: int, num_samples: int, seed: int = 1) -> DosEstimate:
    """spectral.cpp:156-205"""
    b = _iv(bounds)
    mu = np.empty(max(order, 0) + 1)
    _check(_lib().chebfd_kpm_dos(A._h, b.lo, b.hi, order, num_samples, seed, _ptr(mu)))
    return DosEstimate(mu, b, num_samples, A.dim())


def estimate_count(dos: DosEstimate, interval) -> float:
    """spectral.cpp:90-94"""
    iv = _iv(interval)
    if not dos.bounds.contains(iv):
        raise InvalidArgument("estimate_count: interval outside DOS bounds")
    return dos.count(iv.lo, iv.hi)


@dataclass
class SolverOptions:
    """solver.hpp:12-25"""
    target: Interval = field(default_factory=Interval)
    epsilon: float = 1e-10
    n_search: int = 0
    degree: int = 0
    kernel: Kernel = field(default_factory=lambda: Kernel("lanczos", 2))
    max_iters: int = 40
    seed: int = 1
    dos_moments: int = 2000
    dos_samples: int = 32
    deterministic: bool = True
    bounds: Interval = field(default_factory=Interval)
    collect_weight_density: bool = True


@dataclass
class ConvergenceReport:
    """solver.hpp:43-60"""
    converged: bool
    iterations: int
    total_spmvms: float
    n_search: int
    degree: int
    sigma: float
    eta: float
    bounds: Interval
    matrix_norm_est: float
    n_target_estimate: float
    ritz: RitzSet
    history: np.ndarray
    weight_integral: float
    have_weight: bool
    seconds: float
    timings: dict = field(default_factory=dict)  # wall seconds per solve phase
    weight: Optional["WeightDensity"] = None     # ConvergenceReport::weight (solver.cpp:158-162)


def solve(A: SparseMatrix, opts: SolverOptions) -> ConvergenceReport:
    """Full ChebFD iteration (solver.cpp:93-214) driven from host C++ with all
    block work on the device."""
    o = L.chebfd_solver_options()
    _lib().chebfd_solver_options_default(C.byref(o))
    t = _iv(opts.target)
    b = _iv(opts.bounds)
    kk, mu = _kernel(opts.kernel).code()
    o.target_lo, o.target_hi = t.lo, t.hi
    o.epsilon = opts.epsilon
    o.n_search = opts.n_search
    o.degree = opts.degree
    o.kernel, o.kernel_mu = kk, mu
    o.max_iters = opts.max_iters
    o.seed = opts.seed
    o.dos_moments = opts.dos_moments
    o.dos_samples = opts.dos_samples
    o.bounds_lo, o.bounds_hi = b.lo, b.hi
    o.collect_weight_density = int(opts.collect_weight_density)
    rep = L.chebfd_solve_report()
    cap = max(4096, 2 * opts.n_search)
    vals = np.zeros(cap)
    res = np.zeros(cap)
    acc = np.zeros(cap, dtype=np.int32)
    hist = np.zeros((opts.max_iters, 5))
    vh = C.c_void_p()
    wcap = 1 << 20
    wmu = np.zeros(wcap)
    wlen = C.c_int()
    _check(_lib().chebfd_solve_ex(A._h, C.byref(o), C.byref(rep), cap, _ptr(vals), _ptr(res),
                                  _ptr(acc), _ptr(hist), C.byref(vh), wcap, _ptr(wmu),
                                  C.byref(wlen)))
    weight = (WeightDensity(wmu[:wlen.value].copy(), Interval(rep.bounds_lo, rep.bounds_hi))
              if wlen.value > 0 else None)
    n = rep.n_values
    V = BlockVector(A, _handle=vh) if vh.value else None
    ritz = RitzSet(vals[:n].copy(), V, res[:n].copy(), acc[:n].astype(bool))
    return ConvergenceReport(bool(rep.converged), rep.iterations, rep.total_spmvms, rep.n_search,
                             rep.degree, rep.sigma, rep.eta, Interval(rep.bounds_lo, rep.bounds_hi),
                             rep.matrix_norm_est, rep.n_target_estimate, ritz,
                             hist[:rep.iterations].copy(), rep.weight_integral,
                             bool(opts.collect_weight_density), rep.seconds,
                             {k: getattr(rep, "t_" + k) for k in
                              ("bounds", "dos", "design", "filter", "ortho", "rr", "start")},
                             weight)


# ----------------------------------------------------- bench conventions --
def per_row_flops(n_nzr, f_a, f_m):
    """bench.cpp:28-30"""
    return n_nzr * (f_a + f_m) + np.ceil(9.0 * f_a / 2.0) + np.ceil(11.0 * f_m / 2.0)


def per_row_bytes(n_nzr, s_d, s_i, n_b):
    """bench.cpp:32-34"""
    return n_nzr / n_b * (s_d + s_i) + 5.0 * s_d


def filter_schedule_bytes(dim, nnz, n_b, cplx, degree, group=3):
    """Minimal DRAM bytes of one apply_filter as this library schedules it (no moments):
    the matrix (S_d + 4 bytes per entry) once per step plus the block streams each step
    kind moves -- start-up spmmvm (X gathered, U written: 2 streams), start-up step 2 (U
    gathered, X read, W and X written: 4), then groups of `group` steps (CHEBFD_OPT_DELAYED_X):
    V_n-only steps (U gathered, W read and written: 3) and the group's last step, which
    also reads and writes X (5).  The reference's model (bench.cpp:32-34) charges 5
    streams to every step; this is the byte count the kernels can at best move."""
    s_d = 16 if cplx else 8
    mat = nnz * (s_d + 4)
    blk = dim * n_b * s_d
    total = (mat + 2 * blk) + (mat + 4 * blk)
    n = 3
    while n <= degree:
        g = min(max(group, 1), degree - n + 1)
        total += (g - 1) * (mat + 3 * blk) + (mat + 5 * blk)
        n += g
    return total


def intensity_model(n_nzr, s_d, s_i, f_a, f_m, n_b):
    """intensity_model (bench.cpp:37-41) through the C ABI."""
    out = C.c_double()
    _check(_lib().chebfd_intensity_model(float(n_nzr), int(s_d), int(s_i), int(f_a), int(f_m),
                                         int(n_b), C.byref(out)))
    return out.value


# ------------------------------------------------- distributed planning --
def plan_partition(spec: LatticeSpec, model: str, rank: int, nranks: int):
    """Rows and halos of `rank` for a lattice model ("graphene" | "ti"),
    partitioned on lattice planes; send ranges via plan_complete_sends."""
    out = L.chebfd_partition()
    s = spec._c()
    _check(_lib().chebfd_plan_partition(C.byref(s), {"graphene": 0, "ti": 1}[model], rank, nranks,
                                        C.byref(out)))
    return out


def plan_all4(plan) -> list:
    """This rank's (halo_lo, halo_hi, lo_rank, hi_rank) -- what ranks all-gather."""
    return [plan.halo_lo, plan.halo_hi, plan.lo_rank, plan.hi_rank]


def plan_sends(plan, rank: int, all4) -> None:
    """Fill plan's send ranges from every rank's plan_all4 (flattened)."""
    arr = np.ascontiguousarray(np.asarray(all4, dtype=np.int64).reshape(-1))
    _check(_lib().chebfd_plan_sends(C.byref(plan), rank, len(arr) // 4, _ptr(arr)))


def plan_complete_sends(plans) -> None:
    """Single-process helper: complete the send ranges of all ranks' plans."""
    all4 = [v for p in plans for v in plan_all4(p)]
    for r, p in enumerate(plans):
        plan_sends(p, r, all4)


def plan_map_column(plan, g: int) -> int:
    """Extended-row index of global column g on this rank (-2: not held)."""
    return int(_lib().chebfd_plan_map_column(C.byref(plan), int(g)))


# --------------------------------------------------------- filter design --
@dataclass
class DesignResult:
    """filter_design.hpp:21-28 (+ the margin and N_T used)."""
    np_opt: int
    eta_opt: float
    sigma: float
    predicted_mvms: float
    predicted_iters: int
    delta_prime: float
    n_target_estimate: float = 0.0
    below_recommended_search_space: bool = False


def _design(d):
    return DesignResult(d.np_opt, d.eta_opt, d.sigma, d.predicted_mvms, d.predicted_iters,
                        d.delta_prime, d.n_target_estimate, bool(d.below_recommended_search_space))


def damping_factor(p: FilterPolynomial, delta_prime: float) -> float:
    """sigma of filter p for the search margin delta' (filter_design.cpp:178-184)."""
    k, mu = p.kernel.code()
    s = C.c_double()
    _check(_lib().chebfd_damping_factor(p.target.lo, p.target.hi, delta_prime, p.bounds.lo,
                                        p.bounds.hi, p.degree, k, mu, C.byref(s)))
    return s.value


def optimize_degree(target, delta_prime, bounds, kernel="lanczos2", epsilon=1e-12) -> DesignResult:
    """filter_design.cpp:204-277"""
    t, b = _iv(target), _iv(bounds)
    k, mu = _kernel(kernel).code()
    d = L.chebfd_design()
    _check(_lib().chebfd_optimize_degree(t.lo, t.hi, delta_prime, b.lo, b.hi, k, mu, epsilon,
                                         C.byref(d)))
    return _design(d)


def invert_search_margin(dos: DosEstimate, target, n_search: float) -> float:
    """filter_design.cpp:330-354"""
    t = _iv(target)
    mu = np.ascontiguousarray(dos.moments, dtype=np.float64)
    out = C.c_double()
    _check(_lib().chebfd_invert_search_margin(_ptr(mu), len(mu) - 1, dos.bounds.lo, dos.bounds.hi,
                                              t.lo, t.hi, n_search, C.byref(out)))
    return out.value


def choose_parameters(dos: DosEstimate, target, n_search: float, kernel="lanczos2",
                      epsilon=1e-12) -> DesignResult:
    """filter_design.cpp:356-369"""
    t = _iv(target)
    k, kmu = _kernel(kernel).code()
    mu = np.ascontiguousarray(dos.moments, dtype=np.float64)
    d = L.chebfd_design()
    _check(_lib().chebfd_choose_parameters(_ptr(mu), len(mu) - 1, dos.bounds.lo, dos.bounds.hi,
                                           t.lo, t.hi, n_search, k, kmu, epsilon, C.byref(d)))
    return _design(d)


def quality(degree: int, sigma: float) -> float:
    """filter_design.cpp:186-190"""
    if not sigma > 0.0:
        raise DomainError("quality: sigma must be positive")
    if sigma >= 1.0:
        raise DomainError("quality: sigma >= 1, filter does not damp")
    return -degree / np.log10(sigma)


def host_randomize(dim: int, width: int, seed: int, complex_: bool = False, first_row: int = 0,
                   rows=None) -> np.ndarray:
    """Rows [first_row, first_row+rows) of BlockVector(dim, width).randomize(seed)
    (block_vector.hpp:42-51) -- the reference's exact stream, generated on the
    host in parallel (mt19937_64 jump-ahead)."""
    rows = dim - first_row if rows is None else rows
    out = np.empty((rows, width), dtype=np.complex128 if complex_ else np.float64)
    _check(_lib().chebfd_host_randomize(int(complex_), seed, first_row * width, rows * width,
                                        _ptr(out)))
    return out


# ------------------------------------------------------------ on-disk formats --
def read_matrix_market(path):
    """Host CSR of a Matrix Market file (read_matrix_market, matrix_market.cpp:
    98-115): returns (dim, offs, cols, vals, hermitian); vals complex128 for a
    complex field, float64 for real / integer."""
    lib, bpath = _lib(), os.fsencode(path)
    kind, dim, nnz, herm = C.c_int(), C.c_int64(), C.c_int64(), C.c_int()
    _check(lib.chebfd_read_matrix_market(bpath, C.byref(kind), C.byref(dim), C.byref(nnz),
                                         None, None, None, C.byref(herm)))
    offs = np.empty(dim.value + 1, np.int64)
    cols = np.empty(nnz.value, np.int64)
    vals = np.empty(nnz.value, np.complex128 if kind.value else np.float64)
    _check(lib.chebfd_read_matrix_market(bpath, C.byref(kind), C.byref(dim), C.byref(nnz),
                                         _ptr(offs), _ptr(cols), _ptr(vals), C.byref(herm)))
    return dim.value, offs, cols, vals, bool(herm.value)


def write_matrix_market(path, dim, row_offsets, col_indices, values, hermitian=True):
    """write_matrix_market (matrix_market.cpp:63-95): lower triangle for a
    Hermitian matrix, 17 significant digits."""
    offs = np.ascontiguousarray(row_offsets, dtype=np.int64)
    cols = np.ascontiguousarray(col_indices, dtype=np.int64)
    vals = np.ascontiguousarray(values)
    kind = COMPLEX128 if np.iscomplexobj(vals) else REAL64
    vals = vals.astype(np.complex128 if kind else np.float64, copy=False)
    if len(offs) != dim + 1 or offs[-1] != len(cols) or len(cols) != len(vals):
        raise InvalidArgument("write_matrix_market: inconsistent CSR arrays")
    _check(_lib().chebfd_write_matrix_market(os.fsencode(path), kind, dim, _ptr(offs), _ptr(cols),
                                             _ptr(vals), int(bool(hermitian))))


def save_block(path, block: np.ndarray):
    """.cbfd dump of a host D x nb block (BlockVector::save format)."""
    a = np.ascontiguousarray(block)
    if a.ndim != 2:
        raise InvalidArgument("save_block: expects a 2-D block")
    kind = COMPLEX128 if np.iscomplexobj(a) else REAL64
    a = a.astype(np.complex128 if kind else np.float64, copy=False)
    _check(_lib().chebfd_cbfd_save(os.fsencode(path), kind, a.shape[0], a.shape[1], _ptr(a)))


def load_block(path) -> np.ndarray:
    """Host block from a .cbfd file (BlockVector::load format)."""
    lib, bpath = _lib(), os.fsencode(path)
    kind, dim, width = C.c_int(), C.c_uint64(), C.c_uint32()
    _check(lib.chebfd_cbfd_load(bpath, C.byref(kind), C.byref(dim), C.byref(width), None))
    out = np.empty((dim.value, width.value), np.complex128 if kind.value else np.float64)
    _check(lib.chebfd_cbfd_load(bpath, C.byref(kind), C.byref(dim), C.byref(width), _ptr(out)))
    return out


# ------------------------------------------------------------ bench front end --
@dataclass
class BenchPoint:
    """bench.hpp:49-58"""
    n_b: int
    seconds: float
    flops: float
    gflops: float
    gbs_proxy: float
    intensity: float
    roofline: float
    efficiency: float


@dataclass
class BenchReport:
    """bench.hpp:60-66; to_json() gives bench_report.json's schema (chebfd.cpp:336-357)."""
    points: list
    bandwidth_gbs: float
    degree: int
    dim: int
    traffic_overhead: str = "not measured"  # hardware counters: see profiles/ (ncu)

    def to_json(self):
        return {"bandwidth_gbs": self.bandwidth_gbs, "degree": self.degree, "dim": self.dim,
                "traffic_overhead": self.traffic_overhead,
                "points": [{"n_b": p.n_b, "seconds": p.seconds, "flops": p.flops,
                            "gflops": p.gflops, "gbs_proxy": p.gbs_proxy,
                            "intensity": p.intensity, "roofline_gflops": p.roofline,
                            "efficiency": p.efficiency} for p in self.points]}

    def table(self):
        """The CLI's text table (chebfd.cpp:329-343)."""
        lines = [f"bandwidth: {self.bandwidth_gbs:g} GB/s   traffic overhead: "
                 f"{self.traffic_overhead}",
                 "  n_b   Gflop/s      GB/s  I(n_b)    P*(Gflop/s)  efficiency"]
        for p in self.points:
            lines.append(f"{p.n_b:5d} {p.gflops:9.3f} {p.gbs_proxy:9.3f} {p.intensity:7.4f} "
                         f"{p.roofline:14.3f} {p.efficiency:11.3f}")
        return "\n".join(lines)


def bandwidth_probe_min_bytes(ctx: Context) -> int:
    """8 x the GPU's L2 (bench.cpp:42 uses 8 x the LLC)."""
    out = C.c_uint64()
    _check(_lib().chebfd_bandwidth_probe_min_bytes(ctx._h, C.byref(out)))
    return out.value


def bandwidth_probe(ctx: Context, size_bytes: Optional[int] = None, reps: int = 5) -> float:
    """bandwidth_probe (bench.cpp:44-67) on HBM: median GB/s of read-only sweeps."""
    if size_bytes is None:
        size_bytes = bandwidth_probe_min_bytes(ctx)
    out = C.c_double()
    _check(_lib().chebfd_bandwidth_probe(ctx._h, int(size_bytes), int(reps), C.byref(out)))
    return out.value


def bench_filter(A: SparseMatrix, block_sizes=(1, 2, 4, 8, 16, 32), degree: int = 100,
                 bandwidth_gbs: float = 0.0) -> BenchReport:
    """bench_filter (bench.cpp:71-126) on the device."""
    sizes = np.ascontiguousarray(list(block_sizes), dtype=np.int32)
    pts = (L.chebfd_bench_point * max(len(sizes), 1))()
    bw = C.c_double()
    _check(_lib().chebfd_bench_filter(A._h, _ptr(sizes), len(sizes), int(degree),
                                      float(bandwidth_gbs), pts, C.byref(bw)))
    points = [BenchPoint(*(getattr(pts[i], f) for f, _ in L.chebfd_bench_point._fields_))
              for i in range(len(sizes))]
    return BenchReport(points=points, bandwidth_gbs=bw.value, degree=int(degree), dim=A.dim())
