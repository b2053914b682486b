"""GPU: files -> device objects through the C ABI.

Matrix Market files the reference wrote (tests/golden/formats/) load straight
into device SELL matrices whose SpMMV is bit-identical to the oracle's on the
same CSR; .cbfd dumps round-trip device blocks byte for byte and reproduce
the reference's files.
"""
import os

import numpy as np
import pytest

import paper_1510_04895_b200 as cf
from oracle import CSR, formats

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "formats")


def bits(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and a.dtype == b.dtype and a.tobytes() == b.tobytes()


@pytest.mark.parametrize("name", ["graphene_6x5_symmetric.mtx", "graphene_6x5_general.mtx",
                                  "ti_2x2x3_hermitian.mtx"])
def test_matrix_market_to_device_spmmv_bitexact(ctx, orc, name):
    path = os.path.join(GOLDEN, name)
    dim, offs, cols, vals, _ = formats.read_matrix_market(path)
    A = cf.SparseMatrix.from_matrix_market(ctx, path)
    assert A.dim() == dim and A.nnz() == len(cols)
    assert A.dtype == vals.dtype
    x = orc.randomize(dim, 5, 13, np.iscomplexobj(vals))
    y = cf.spmmvm(A, cf.BlockVector(A, 5).upload(x), 0.31, -0.07).to_numpy()
    assert bits(y, orc.spmmvm(CSR(offs, cols, vals), x, 0.31, -0.07))


def test_matrix_market_errors_on_device_path(ctx, tmp_path):
    p = tmp_path / "bad.mtx"
    p.write_text("%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1\n")
    with pytest.raises(cf.OutOfRange):
        cf.SparseMatrix.from_matrix_market(ctx, str(p))
    with pytest.raises(cf.NumericalError):
        cf.SparseMatrix.from_matrix_market(ctx, str(tmp_path / "missing.mtx"))


@pytest.mark.parametrize("cplx", [False, True])
def test_block_save_load_round_trip(ctx, orc, tmp_path, cplx):
    spec = cf.LatticeSpec(4, 4, 4, disorder=0.5, seed=2)
    A = (cf.SparseMatrix.topological_insulator(ctx, spec) if cplx
         else cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(16, 8, disorder=0.5, seed=2)))
    X = cf.BlockVector(A, 7).randomize(9)
    p = tmp_path / "x.cbfd"
    X.save(str(p))
    host = X.to_numpy()
    assert p.read_bytes() == formats.cbfd_bytes(host)
    Y = cf.BlockVector.load(A, str(p))
    assert Y.shape == X.shape and bits(Y.to_numpy(), host)


def test_block_load_golden_and_errors(ctx, tmp_path):
    path = os.path.join(GOLDEN, "block_real_30x4.cbfd")
    want = formats.parse_cbfd(open(path, "rb").read())
    A = cf.SparseMatrix.from_csr(ctx, 30, np.arange(31), np.arange(30), np.linspace(-1, 1, 30))
    assert bits(cf.BlockVector.load(A, path).to_numpy(), want)
    B = cf.SparseMatrix.from_csr(ctx, 31, np.arange(32), np.arange(31), np.linspace(-1, 1, 31))
    with pytest.raises(cf.InvalidArgument):  # dimension does not match the matrix
        cf.BlockVector.load(B, path)
    Z = cf.SparseMatrix.from_csr(ctx, 30, np.arange(31), np.arange(30),
                                 np.linspace(-1, 1, 30) + 0j)
    with pytest.raises(cf.NumericalError, match="kind mismatch"):
        cf.BlockVector.load(Z, path)
