"""Restatement of the reference's on-disk formats -- TEST INFRASTRUCTURE ONLY.

Pure Python / numpy, for the checker side of tests on the GPU box (where the
compiled reference is absent).  Pinned against the compiled reference's own
reader / writer in tests/test_formats.py.

* ``read_matrix_market`` follows matrix_market.cpp:19-61 (read_body) and
  :98-115 (banner checks): '%' lines skipped, 1-based indices, mirrored
  entries for symmetric (same value) and hermitian (conjugate) storage,
  duplicates summed in insertion order (SparseMatrix::Builder,
  sparse_matrix.hpp:58-79 -- a std::map per row starting from S{}).
* ``cbfd_bytes`` / ``parse_cbfd`` follow BlockVector::save / load
  (block_vector.hpp:63-96).
"""
from __future__ import annotations

import struct

import numpy as np

CBFD_MAGIC = 0x44464243  # "CBFD"


def read_matrix_market(path):
    """-> (dim, offs, cols, vals, hermitian); raises ValueError with the
    reference's message text (runtime_error) or IndexError (out_of_range)."""
    with open(path) as f:
        lines = f.read().split("\n")
    if not lines or not lines[0].startswith("%%MatrixMarket"):
        raise ValueError(f"{path}: missing MatrixMarket banner")
    words = lines[0][2:].lower().split()
    words += [""] * (5 - len(words))
    _, obj, fmt, field, sym = words[:5]
    if obj != "matrix" or fmt != "coordinate":
        raise ValueError(f"{path}: only coordinate matrices are supported")
    if sym not in ("general", "symmetric", "hermitian"):
        raise ValueError(f"{path}: unsupported symmetry '{sym}'")
    if field in ("real", "integer"):
        cplx = False
    elif field == "complex":
        cplx = True
    else:
        raise ValueError(f"{path}: unsupported field '{field}'")
    body = iter(lines[1:])
    data = (ln for ln in body if ln and ln[0] != "%")
    rows = cols = nnz = 0
    for ln in data:
        t = ln.split()
        try:
            rows, cols, nnz = int(t[0]), int(t[1]), int(t[2])
        except (ValueError, IndexError):
            raise ValueError(f"{path}: malformed size line")
        break
    if rows != cols:
        raise ValueError(f"{path}: matrix is not square")
    acc = [dict() for _ in range(rows)]  # row -> {col: value}, insertion-order sums
    zero = 0j if cplx else 0.0

    def add(i, j, v):
        if i < 0 or i >= rows or j < 0 or j >= rows:
            raise IndexError("SparseMatrix::Builder: index out of range")
        acc[i][j] = acc[i].get(j, zero) + v

    seen = 0
    for ln in data:
        if seen >= nnz:
            break
        t = ln.split()
        try:
            i, j = int(t[0]) - 1, int(t[1]) - 1
        except (ValueError, IndexError):
            raise ValueError(f"{path}: malformed entry line")
        if len(t) < 3:
            raise ValueError(f"{path}: missing value")
        re = float(t[2])
        if cplx:
            if len(t) < 4:
                raise ValueError(f"{path}: missing imaginary part")
            v = complex(re, float(t[3]))
        else:
            v = re
        add(i, j, v)
        if i != j:
            if sym == "symmetric":
                add(j, i, v)
            elif sym == "hermitian":
                add(j, i, v.conjugate() if cplx else v)
        seen += 1
    if seen != nnz:
        raise ValueError(f"{path}: fewer entries than declared")
    offs = np.zeros(rows + 1, np.int64)
    cl, vl = [], []
    for i in range(rows):
        for j in sorted(acc[i]):
            cl.append(j)
            vl.append(acc[i][j])
        offs[i + 1] = len(cl)
    vals = np.array(vl, np.complex128 if cplx else np.float64)
    return rows, offs, np.array(cl, np.int64), vals, sym != "general"


def cbfd_bytes(block):
    """BlockVector::save (block_vector.hpp:65-78) as bytes."""
    a = np.ascontiguousarray(block)
    kind = 1 if np.iscomplexobj(a) else 0
    a = a.astype(np.complex128 if kind else np.float64, copy=False)
    return struct.pack("<IQII", CBFD_MAGIC, a.shape[0], a.shape[1], kind) + a.tobytes()


def parse_cbfd(raw):
    """BlockVector::load (block_vector.hpp:80-95) from bytes."""
    if len(raw) < 20:
        raise ValueError("BlockVector::load: bad header")
    magic, dim, width, kind = struct.unpack_from("<IQII", raw)
    if magic != CBFD_MAGIC:
        raise ValueError("BlockVector::load: bad header")
    dt = np.complex128 if kind else np.float64
    n = dim * width * np.dtype(dt).itemsize
    if len(raw) - 20 < n:
        raise ValueError("BlockVector::load: truncated payload")
    return np.frombuffer(raw[20:20 + n], dt).reshape(dim, width).copy()
