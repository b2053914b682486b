"""GPU Rayleigh-Ritz / SVQB / spectral probes / full solve against the
reference's known answers (test_solver.cpp, test_spectral.cpp) and dense
numpy eigenvalues.  Tolerances are the reference tests' own."""
import json
import os

import numpy as np
import pytest

import paper_1510_04895_b200 as cf

pytestmark = pytest.mark.gpu

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def random_symmetric(d, seed):
    rng = np.random.default_rng(seed)
    a = rng.uniform(-1, 1, (d, d)) / np.sqrt(d)
    a = np.triu(a)
    a = a + np.triu(a, 1).T
    return a


def dense_to_matrix(ctx, a):
    d = a.shape[0]
    offs = np.arange(0, d * d + 1, d)
    cols = np.tile(np.arange(d), d)
    return cf.SparseMatrix.from_csr(ctx, d, offs, cols, a.reshape(-1))


def orthonormality_defect(q):
    g = q.conj().T @ q
    return np.max(np.abs(g - np.eye(q.shape[1])))


def test_svqb_preserves_orthonormal_block(ctx, orc):
    """test_solver.cpp:60-73"""
    A = dense_to_matrix(ctx, random_symmetric(128, 1))
    Y = cf.BlockVector(A, 6).randomize(3)
    first = cf.svqb_orthonormalize(Y)
    assert first.rank == 6
    second = cf.svqb_orthonormalize(first.q)
    assert second.rank == 6
    q1, q2 = first.q.to_numpy(), second.q.to_numpy()
    assert orthonormality_defect(q2) <= 1e-12
    assert np.max(np.abs(q1 @ q1.T - q2 @ q2.T)) <= 1e-12


def test_svqb_drops_duplicate_column(ctx, orc):
    """test_solver.cpp:75-82"""
    A = dense_to_matrix(ctx, random_symmetric(64, 2))
    y = orc.randomize(64, 4, 5)
    y[:, 3] = y[:, 1]
    r = cf.svqb_orthonormalize(cf.BlockVector(A, 4).upload(y))
    assert r.rank == 3
    assert orthonormality_defect(r.q.to_numpy()[:, :3]) <= 1e-12


def test_svqb_matches_qr_projector(ctx, orc):
    """test_solver.cpp:84-96"""
    A = dense_to_matrix(ctx, random_symmetric(500, 3))
    y = orc.randomize(500, 40, 11)
    r = cf.svqb_orthonormalize(cf.BlockVector(A, 40).upload(y))
    assert r.rank == 40
    q = r.q.to_numpy()
    qd, _ = np.linalg.qr(y)
    assert np.max(np.abs(q @ q.T - qd @ qd.T)) <= 1e-10


def test_svqb_rejects_zero_block(ctx):
    """test_solver.cpp:98-101"""
    A = dense_to_matrix(ctx, random_symmetric(32, 4))
    with pytest.raises(cf.NumericalError):
        cf.svqb_orthonormalize(cf.BlockVector(A, 2))


def test_rayleigh_ritz_invariant_subspace(ctx):
    """test_solver.cpp:103-116"""
    lam = np.array([-0.9, -0.5, -0.1, 0.2, 0.6, 1.0])
    A = cf.SparseMatrix.from_csr(ctx, 6, np.arange(7), np.arange(6), lam)
    q = np.zeros((6, 3))
    q[1, 0] = q[3, 1] = q[4, 2] = 1.0
    r = cf.rayleigh_ritz(A, cf.BlockVector(A, 3).upload(q))
    assert np.allclose(r.values, [-0.5, 0.2, 0.6], rtol=1e-13)
    assert np.all(r.residual_norms <= 1e-13)


def test_rayleigh_ritz_interlacing(ctx, orc):
    """test_solver.cpp:130-145"""
    a = random_symmetric(200, 31)
    A = dense_to_matrix(ctx, a)
    q = cf.svqb_orthonormalize(cf.BlockVector(A, 12).randomize(32)).q
    r = cf.rayleigh_ritz(A, q)
    ev = np.linalg.eigvalsh(a)
    for k in range(12):
        assert ev[k] - 1e-10 <= r.values[k] <= ev[k + 200 - 12] + 1e-10
    assert np.all(np.diff(r.values) >= 0)


def test_rayleigh_ritz_complex_residuals(ctx, orc):
    c = orc.topological_insulator(4, 4, 4, disorder=0.5)
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(4, 4, 4, disorder=0.5))
    q = cf.svqb_orthonormalize(cf.BlockVector(A, 10).randomize(3)).q
    r = cf.rayleigh_ritz(A, q)
    v = r.vectors.to_numpy()
    h = c.to_dense()
    res = np.linalg.norm(h @ v - v * r.values[None, :], axis=0)
    assert np.allclose(r.residual_norms, res, rtol=1e-9, atol=1e-13)


def test_lanczos_bounds_contain_spectrum(ctx, orc):
    """test_spectral.cpp:20-27 (flat spectrum) and the graphene bound test."""
    d = 2000
    lam = -1.0 + 2.0 * np.arange(1, d + 1) / (d + 1)
    A = cf.SparseMatrix.from_csr(ctx, d, np.arange(d + 1), np.arange(d), lam)
    b = cf.lanczos_bounds(A, 30, 1)
    assert b.lo <= lam[0] and b.hi >= lam[-1] and b.width() <= 1.05 * 2.0
    G = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(16, 16, boundary="periodic_all"))
    g = cf.lanczos_bounds(G, 40, 6)
    assert -3.07 <= g.lo <= -2.9 and 2.9 <= g.hi <= 3.07


def test_kpm_flat_dos(ctx):
    """test_spectral.cpp:56-65: interior 0.2-windows hold D*0.1."""
    d = 1000
    lam = -1.0 + 2.0 * np.arange(1, d + 1) / (d + 1)
    A = cf.SparseMatrix.from_csr(ctx, d, np.arange(d + 1), np.arange(d), lam)
    dos = cf.kpm_dos(A, (-1.05, 1.05), 2000, 32, 4)
    for lo in np.arange(-0.8, 0.75, 0.2):
        n = dos.count(lo, lo + 0.2)
        # doctest::Approx(100).epsilon(0.05): |a-b| < eps*(1 + max(|a|,|b|))
        assert abs(n - 100.0) < 0.05 * (1.0 + max(abs(n), 100.0))
    # the same probe stream as the reference: its window count is 105.05979586060153
    assert abs(dos.count(-0.2, 0.0) - 105.05979586060153) <= 1e-9
    with pytest.raises(cf.NumericalError):  # test_spectral.cpp:108-111
        B = cf.SparseMatrix.from_csr(ctx, 200, np.arange(201), np.arange(200),
                                     -2.0 + 4.0 * np.arange(1, 201) / 201)
        cf.kpm_dos(B, (-1.0, 1.0), 2000, 4, 8)


@pytest.mark.parametrize("mode", ["doubling", "direct"])
def test_kpm_matches_reference_moments(ctx, orc, mode):
    """Same probe stream as the reference -> moments agree to rounding, whether each
    moment is a <z, T_n z> dot (spectral.cpp:186-195) or comes from the doubling
    identities over half the recurrence steps."""
    path = os.path.join(GOLDEN, "kpm_ti4.json")
    g = json.load(open(path))
    ctx.set_option("moments", mode)
    try:
        A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(4, 4, 4, disorder=0.5, seed=3))
        dos = cf.kpm_dos(A, g["bounds"], g["order"], g["samples"], g["seed"])
    finally:
        ctx.set_option("moments", "doubling")
    mu = np.array(g["mu"])
    assert np.max(np.abs(dos.moments - mu)) <= 1e-9 * mu[0]


@pytest.mark.parametrize("order", [2, 3, 40, 41, 257])
def test_kpm_doubling_equals_direct(ctx, order):
    """kpm_dos moments from the doubling identities (order/2 + 1 recurrence steps) equal the
    direct <z, T_n z> moments (spectral.cpp:186-195) to rounding, odd and even orders."""
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(5, 4, 6, disorder=0.5, seed=2))
    b = (-6.0, 6.0)
    out = {}
    for mode in ("direct", "doubling"):
        ctx.set_option("moments", mode)
        out[mode] = cf.kpm_dos(A, b, order, 8, 3).moments
    ctx.set_option("moments", "doubling")
    assert out["direct"].shape == out["doubling"].shape == (order + 1,)
    assert np.max(np.abs(out["direct"] - out["doubling"])) <= 1e-11 * A.dim()


def test_solve_random_matrix_interior(ctx):
    """test_solver.cpp:147-192"""
    d = 200
    a = random_symmetric(d, 41)
    ev = np.linalg.eigvalsh(a)
    norm2 = max(abs(ev[0]), abs(ev[-1]))
    mid = d // 2
    lo, hi = 0.5 * (ev[mid - 5] + ev[mid - 6]), 0.5 * (ev[mid + 4] + ev[mid + 5])
    A = dense_to_matrix(ctx, a)
    rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(lo, hi), epsilon=1e-10, seed=5,
                                       dos_moments=400, dos_samples=16, degree=60))
    assert rep.converged
    acc = np.sort(rep.ritz.values[rep.ritz.accepted])
    want = ev[(ev >= lo) & (ev <= hi)]
    assert len(want) == 10 and len(acc) == 10
    assert np.max(np.abs(acc - want)) <= 1e-10 * norm2
    assert rep.total_spmvms == rep.iterations * rep.n_search * rep.degree


def test_solve_empty_target(ctx):
    """test_solver.cpp:224-235"""
    d = 500
    lam = -1.0 + 2.0 * np.arange(1, d + 1) / (d + 1)
    A = cf.SparseMatrix.from_csr(ctx, d, np.arange(d + 1), np.arange(d), lam)
    rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(2.5, 2.6), bounds=cf.Interval(-1.1, 3.0),
                                       dos_moments=300, dos_samples=8, degree=20))
    assert rep.converged and len(rep.ritz.values) == 0 and rep.n_target_estimate < 0.5


def test_solve_config1_matches_reference(ctx):
    """BASELINE config 1: graphene 64x64, V=0.1, N_S=40, N_p=500, Lanczos-2,
    window [-0.13, 0.13] (24 eigenvalues).  Golden values from
    the compiled reference (tests/golden/make_golden.py)."""
    g = json.load(open(os.path.join(GOLDEN, "c1_solve.json")))
    A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(64, 64, disorder=0.1, seed=1))
    rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(-0.13, 0.13), n_search=40, degree=500,
                                       seed=1))
    assert rep.converged
    assert rep.iterations == g["iterations"]
    assert abs(rep.n_target_estimate - g["n_target_estimate"]) <= 1e-8 * g["n_target_estimate"]
    acc = np.sort(rep.ritz.values[rep.ritz.accepted])
    want = np.sort(np.array(g["accepted_values"]))
    assert len(acc) == len(want) == 24
    assert np.max(np.abs(acc - want)) <= 1e-10  # north_star: Ritz values within 1e-10
    assert np.all(rep.ritz.residual_norms[rep.ritz.accepted] <= 1e-10)
    assert abs(rep.weight_integral - 40.0) <= 0.4  # test_solver.cpp:256: integral = N_S (1%)


def test_solve_automatic_degree_matches_reference(ctx):
    """solve with degree = 0: the reference's degree rule (choose_parameters,
    solver.cpp:130-136) on a TI slab; golden from the compiled reference."""
    g = json.load(open(os.path.join(GOLDEN, "ti6_auto_solve.json")))
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(6, 6, 6, disorder=0.5, seed=4))
    rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(-0.45, 0.45), degree=0, seed=3,
                                       dos_moments=600, dos_samples=16))
    assert rep.converged and rep.degree == g["degree"] and rep.n_search == g["n_search"]
    assert rep.iterations == g["iterations"]
    assert abs(rep.sigma - g["sigma"]) <= 1e-9 * g["sigma"]
    acc = np.sort(rep.ritz.values[rep.ritz.accepted])
    assert np.max(np.abs(acc - np.array(g["accepted_values"]))) <= 1e-10
    assert set(rep.timings) == {"bounds", "dos", "design", "filter", "ortho", "rr", "start"}


def test_async_start_block_equals_synchronous(ctx):
    """With N_S given, solve() generates the start block on a helper thread while the
    device runs the bounds and the KPM DOS (CHEBFD_OPT_ASYNC_START, default above 2^26
    entries).  Lowered to every size, it must give the synchronous path's bits: the same
    Ritz values, residuals and iteration count."""
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(6, 6, 6, disorder=0.5, seed=4))
    opts = cf.SolverOptions(target=cf.Interval(-0.45, 0.45), n_search=16, degree=60, seed=3,
                            dos_moments=300, dos_samples=8)
    ctx.set_option("async_start", 0)
    try:
        sync = cf.solve(A, opts)
        ctx.set_option("async_start", 1)  # every start block on the helper thread
        asyn = cf.solve(A, opts)
    finally:
        ctx.set_option("async_start", 1 << 26)
    assert asyn.iterations == sync.iterations and asyn.converged == sync.converged
    assert np.array_equal(asyn.ritz.values, sync.ritz.values)
    assert np.array_equal(asyn.ritz.residual_norms, sync.ritz.residual_norms)
    # the empty-target early return joins the helper cleanly
    ctx.set_option("async_start", 1)
    try:
        rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(9.0, 9.5), n_search=16, degree=60,
                                           bounds=cf.Interval(-10.0, 10.0)))
        assert rep.converged and rep.iterations == 0
    finally:
        ctx.set_option("async_start", 1 << 26)
