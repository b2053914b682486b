"""ChebFD solve at the C3 scale (BASELINE.json configs[2]) -- solve() (solver.cpp:93-214)
through the C ABI on the device.

* The scaled C3 protocol against the compiled reference's own solve
  (tests/golden/c3s_solve.json, tests/golden/make_c3s_golden.py): TI 64x64x32, N_S = 64,
  window +-h with ~24 eigenvalues, automatic degree, Lanczos-2 and Jackson -- the same
  degree, N_S, iteration count, N_T estimate and accepted Ritz values within 1e-10.
* C3 itself (TI 128x128x64, D = 4,194,304, N_S = 256, ~100 eigenvalues, Lanczos-2): the
  reference's solve does not fit this host in time or memory, so every accepted pair is
  verified independently on the CPU with the reference's own kernels (oracle/_ref):
  ||H v - lambda v|| <= epsilon by the reference spmmvm, and V^H V = I by its gram.
"""
import json
import os

import numpy as np
import pytest

import paper_1510_04895_b200 as cf

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "c3s_solve.json")


@pytest.mark.parametrize("kernel", ["lanczos2", "jackson"])
def test_scaled_c3_solve_matches_reference(ctx, kernel):
    if not os.path.exists(GOLDEN):
        pytest.skip("tests/golden/c3s_solve.json not generated")
    g = json.load(open(GOLDEN))
    want = g["runs"][kernel]
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(*g["lattice"], disorder=g["disorder"],
                                                                  seed=g["seed"]))
    h = g["h"]
    rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(-h, h), n_search=g["n_search"], degree=0,
                                       kernel=cf.Kernel.parse(kernel), seed=1,
                                       bounds=cf.Interval(*g["bounds"])))
    assert rep.converged == want["converged"]
    assert rep.degree == want["degree"] and rep.n_search == want["n_search"]
    assert abs(rep.n_target_estimate - want["n_target_estimate"]) <= 1e-8 * want["n_target_estimate"]
    assert rep.iterations == want["iterations"]
    acc = np.sort(rep.ritz.values[rep.ritz.accepted])
    assert len(acc) == len(want["accepted_values"])
    assert np.max(np.abs(acc - np.array(want["accepted_values"]))) <= 1e-10
    assert np.all(rep.ritz.residual_norms[rep.ritz.accepted] <= 1e-10)


def test_c3_solve_pairs_verified_by_reference_kernels(ctx):
    import oracle
    if not oracle.ref_available():
        pytest.skip("oracle/_ref not built here")
    spec = cf.LatticeSpec(128, 128, 64, disorder=0.5, seed=1)
    A = cf.SparseMatrix.topological_insulator(ctx, spec)
    b = cf.lanczos_bounds(A, 30, 1)
    dos = cf.kpm_dos(A, b, 2000, 32, 2)
    lo, hi = 0.0, 0.999 * min(-b.lo, b.hi)
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        f = dos.count(-mid, mid) - 100.0
        if abs(f) <= 1e-4:
            lo = hi = mid
            break
        lo, hi = (mid, hi) if f < 0 else (lo, mid)
    h = 0.5 * (lo + hi)
    eps = 1e-10
    rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(-h, h), n_search=256, degree=0,
                                       kernel=cf.Kernel.parse("lanczos2"), seed=1, bounds=b,
                                       epsilon=eps))
    assert rep.converged
    acc = np.flatnonzero(rep.ritz.accepted)
    assert len(acc) >= int(np.ceil(rep.n_target_estimate - 3 * np.sqrt(rep.n_target_estimate)))
    lam = rep.ritz.values[acc]
    assert np.all(np.abs(lam) <= h)
    V = rep.ritz.vectors.to_numpy()[:, acc].copy()
    r = oracle.Ref(threads=len(os.sched_getaffinity(0)))
    m = r.topological_insulator(128, 128, 64, disorder=0.5, seed=1)
    HV = r.spmmvm(m, V, 1.0, 0.0)  # the reference's spmmvm (kernels.hpp:46-69)
    res = np.linalg.norm(HV - V * lam[None, :], axis=0)
    assert np.all(res <= eps), res.max()
    # the device's residuals agree with the reference-kernel residuals
    assert np.allclose(rep.ritz.residual_norms[acc], res, rtol=1e-2, atol=1e-12)
    G = r.gram(V, V)  # the reference's Kahan gram (kernels.hpp:165-192)
    assert np.max(np.abs(G - np.eye(len(acc)))) <= 1e-12
