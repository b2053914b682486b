"""GPU parity at the BASELINE.json configs' own sizes (VERDICT r1
"Next round" 1): the sm_100a path through the C ABI against the UNMODIFIED
compiled reference (oracle/_ref, OpenMP on all host cores).

* C2 (configs[1]): TI 64^3 slab, V = 0.5, seed 1, n_b = 32, N_p = 100, start block
  = the reference's BlockVector::randomize(7) -- apply_filter (filter.hpp:73-116)
  X bit for bit, moments within 1e-12 of the column norm.
* C4 (configs[3]) one-GPU sub-lattice: TI 512 x 512 x 8, n_b = 64, N_p = 12
  (12 Chebyshev steps: the start-up pair and ten fused steps) -- X bit for bit.
* C5 (configs[4]): graphene 2048 x 2048, V = 1.0, fused step (kernels.hpp:74-118)
  for n_b in {1, 4, 8, 16, 32, 64} -- W and X bit for bit, Kahan dots 1e-12.

W and X are row-local, so the reference's bits do not depend on its thread count;
only dot / moment reductions change summation order (tolerances below).
Also: bitwise run-to-run repeatability of the device path (the counterpart of
test_core_linalg.cpp:244-254), moments and Gram included.
"""
import os

import numpy as np
import pytest

import paper_1510_04895_b200 as cf

pytestmark = [pytest.mark.gpu, pytest.mark.slow]


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture(scope="module")
def ref_mt():
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref/libchebfd_ref.so not built here")
    return oracle.Ref(threads=os.cpu_count() or 1)


def test_c2_apply_filter_bitexact_vs_reference(ctx, ref_mt):
    spec = cf.LatticeSpec(64, 64, 64, disorder=0.5, seed=1)
    A = cf.SparseMatrix.topological_insulator(ctx, spec)
    m = ref_mt.topological_insulator(64, 64, 64, disorder=0.5, seed=1)
    assert (A.dim(), A.nnz()) == (m.dim, m.nnz) == (1048576, 11517952)
    x0 = ref_mt.randomize(m.dim, 32, 7, True)
    X = cf.BlockVector(A, 32).randomize(7)  # the library's parallel stream of the same seed
    assert bits_equal(X.to_numpy(), x0)
    p = cf.make_filter((-0.28, 0.28), (-5.6, 5.6), 100, "lanczos2")
    ring0 = ctx.ring_launches
    mom = cf.apply_filter(A, X, p, want_moments=True)
    # steps 3 .. 100 -- the V_n-only steps with their doubling moment sums and the X-update
    # steps -- ran on the site-ring kernel (default from 8 MB planes and a dozen waves of CTAs)
    assert ctx.ring_launches - ring0 == 98
    xr, mr = ref_mt.apply_filter(m, x0, p.combined, p.alpha, p.beta, want_moments=True)
    assert bits_equal(X.to_numpy(), xr)
    assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
    # the north star's bar, stated for the record: ||Y_gpu - Y_ref|| / ||Y_ref|| <= 1e-10
    assert np.linalg.norm(X.to_numpy() - xr) <= 1e-10 * np.linalg.norm(xr)


def test_c4_sublattice_apply_filter_bitexact_vs_reference(ctx, ref_mt):
    spec = cf.LatticeSpec(512, 512, 8, disorder=0.5, seed=1)
    A = cf.SparseMatrix.topological_insulator(ctx, spec)
    m = ref_mt.topological_insulator(512, 512, 8, disorder=0.5, seed=1)
    assert (A.dim(), A.nnz()) == (m.dim, m.nnz) == (8388608, 91226112)
    x0 = cf.host_randomize(m.dim, 64, 3, True)  # = BlockVector::randomize(3), parallel
    X = cf.BlockVector(A, 64).upload(x0)
    p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), 12, "jackson")
    ring0 = ctx.ring_launches
    cf.apply_filter(A, X, p)
    assert ctx.ring_launches - ring0 == 10  # the fused loop ran on the site-ring kernel (default)
    got = X.to_numpy()
    del X
    xr, _ = ref_mt.apply_filter(m, x0, p.combined, p.alpha, p.beta)
    assert bits_equal(got, xr)


def test_c5_fused_step_bitexact_vs_reference(ctx, ref_mt):
    spec = cf.LatticeSpec(2048, 2048, disorder=1.0, seed=1)
    A = cf.SparseMatrix.graphene(ctx, spec)
    m = ref_mt.graphene(2048, 2048, disorder=1.0, seed=1)
    assert (A.dim(), A.nnz()) == (m.dim, m.nnz) == (8388608, 33554432)
    alpha, beta, coeff = 2.0 / 7.2, 0.0, 0.37
    for nb in (1, 4, 8, 16, 32, 64):
        u, w, x = (cf.host_randomize(m.dim, nb, s, False) for s in (1, 2, 3))
        U, W, X = (cf.BlockVector(A, nb).upload(h) for h in (u, w, x))
        d = cf.spmmvm_fused(A, U, W, X, alpha, beta, coeff, dots=True)
        dref = ref_mt.spmmvm_fused(m, u, w, x, alpha, beta, coeff, want_dots=True)
        assert bits_equal(W.to_numpy(), w), nb
        assert bits_equal(X.to_numpy(), x), nb
        assert np.allclose(d, dref, rtol=1e-12, atol=1e-12 * np.max(np.abs(dref))), nb
        del U, W, X


def test_device_path_bitwise_repeatable(ctx):
    """Same inputs, same bits, twice: apply_filter X and moments (fixed-order grid
    reductions), fused dots, Gram (test_core_linalg.cpp:244-254 asks the reference's
    gram to repeat bitwise)."""
    spec = cf.LatticeSpec(64, 64, 64, disorder=0.5, seed=1)
    A = cf.SparseMatrix.topological_insulator(ctx, spec)
    p = cf.make_filter((-0.28, 0.28), (-5.6, 5.6), 60, "lanczos2")
    runs = []
    for _ in range(2):
        X = cf.BlockVector(A, 32).randomize(7)
        mom = cf.apply_filter(A, X, p, want_moments=True)
        U = cf.BlockVector(A, 32).randomize(1)
        W = cf.BlockVector(A, 32).randomize(2)
        d = cf.spmmvm_fused(A, U, W, X, p.alpha, p.beta, 0.5, dots=True)
        g = cf.gram(X, W)
        runs.append((X.to_numpy(), mom.m.copy(), d, g))
    for a, b in zip(runs[0], runs[1]):
        assert bits_equal(a, b)
