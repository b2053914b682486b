"""The hand-written FP64 tensor-core kernels (csrc/gram.cu): gram X^H Y (kernels.hpp:165-192)
and block_mult_small Y = X B (kernels.hpp:216-232) against the CPU oracle's restatement,
over widths that fill, split and pad the 64 x 64 super-tiles, Hermitian (Y^H Y) and
general (X^H Y) products, row counts that do not fill the 16-row stages, and the real
path (forced with CHEBFD_OPT_GRAM = 2).  Reduction order differs from the reference's
Kahan chunks: 1e-13 of the largest entry; the rotation has no cross-row sums and
matches to 1e-14."""
import numpy as np
import pytest

import paper_1510_04895_b200 as cf

pytestmark = pytest.mark.gpu


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


@pytest.mark.parametrize("l,nx,ny", [((7, 5, 9), 64, 64), ((7, 5, 9), 100, 100), ((3, 3, 5), 130, 48),
                                     ((6, 6, 6), 48, 193), ((2, 3, 1), 64, 64)])
@pytest.mark.parametrize("mode", [1, 2])
def test_dmma_gram_complex(ctx, orc, l, nx, ny, mode):
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(*l, disorder=0.5, seed=1))
    x = orc.randomize(A.dim(), nx, 4, True)
    y = orc.randomize(A.dim(), ny, 5, True)
    X = cf.BlockVector(A, nx).upload(x)
    Y = cf.BlockVector(A, ny).upload(y)
    ctx.set_option("gram", mode)
    try:
        assert rel(cf.gram(X, Y), orc.gram(x, y)) <= 1e-13
        g = cf.gram(X, X)  # Hermitian: upper super-tiles computed, lower mirrored
        assert rel(g, orc.gram(x, x)) <= 1e-13
        assert np.array_equal(g, g.conj().T) or rel(g, g.conj().T) <= 1e-15
    finally:
        ctx.set_option("gram", 1)


@pytest.mark.parametrize("nb,m", [(64, 64), (100, 37), (48, 130), (256, 256)])
def test_dmma_block_mult_small(ctx, orc, nb, m):
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(5, 5, 7, disorder=0.5, seed=2))
    x = orc.randomize(A.dim(), nb, 6, True)
    rng = np.random.default_rng(nb + m)
    B = rng.standard_normal((nb, m)) + 1j * rng.standard_normal((nb, m))
    X = cf.BlockVector(A, nb).upload(x)
    ctx.set_option("gram", 2)
    try:
        Y = cf.block_mult_small(X, B).to_numpy()
    finally:
        ctx.set_option("gram", 1)
    assert rel(Y, orc.block_mult_small(x, B)) <= 1e-14


@pytest.mark.parametrize("nx,ny", [(64, 64), (40, 66)])
def test_dmma_gram_real_forced(ctx, orc, nx, ny):
    A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(31, 17, disorder=0.3, seed=2))
    x = orc.randomize(A.dim(), nx, 7, False)
    y = orc.randomize(A.dim(), ny, 8, False)
    X = cf.BlockVector(A, nx).upload(x)
    Y = cf.BlockVector(A, ny).upload(y)
    ctx.set_option("gram", 2)
    try:
        assert rel(cf.gram(X, Y), orc.gram(x, y)) <= 1e-13
        assert rel(cf.gram(X, X), orc.gram(x, x)) <= 1e-13
    finally:
        ctx.set_option("gram", 1)


def test_rayleigh_ritz_with_hermitian_half_projection(ctx, orc):
    """Rayleigh-Ritz computes only the upper half of Q^H A Q on Hermitian operators
    (DMMA path, n_b >= 48): Ritz values equal the dense projection's eigenvalues."""
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(6, 6, 5, disorder=0.5, seed=3))
    csr = orc.topological_insulator(6, 6, 5, disorder=0.5, seed=3)
    nb = 72
    x = orc.randomize(A.dim(), nb, 9, True)
    q, _ = np.linalg.qr(x)
    Q = cf.BlockVector(A, nb).upload(np.ascontiguousarray(q))
    r = cf.rayleigh_ritz(A, Q)
    H = csr.to_dense()
    want = np.linalg.eigvalsh(q.conj().T @ H @ q)
    assert np.max(np.abs(np.sort(r.values) - want)) <= 1e-12 * np.max(np.abs(want))
