"""CPU: pin the solver restatement (oracle/solver.py) to the reference.

C1 (graphene 64^2, N_S = 40, N_p = 500, window [-0.13, 0.13]) must reproduce
the reference's iteration count, N_T estimate and accepted Ritz values
(tests/golden/c1_solve.json, written from the compiled reference); the
spectral probes must agree with the compiled reference where it is built.
"""
import json
import os

import numpy as np
import pytest

from oracle import solver as osolve

GOLD = os.path.join(os.path.dirname(__file__), "golden")


@pytest.mark.slow
def test_oracle_solve_reproduces_reference_c1(orc):
    g = json.load(open(os.path.join(GOLD, "c1_solve.json")))
    a = orc.graphene(64, 64, disorder=0.1, seed=1)
    rep = osolve.solve(orc, a, (-0.13, 0.13), 500, n_search=40, seed=1,
                       bounds=tuple(g["bounds"]))
    assert rep["converged"] and rep["iterations"] == g["iterations"]
    assert abs(rep["n_target_estimate"] - g["n_target_estimate"]) <= 1e-9 * g["n_target_estimate"]
    acc = np.sort(rep["values"][rep["accepted"]])
    assert len(acc) == 24
    assert np.max(np.abs(acc - np.array(g["accepted_values"]))) <= 1e-10


def test_spectral_probes_match_reference(orc, ref):
    a = orc.topological_insulator(4, 4, 4, disorder=0.5, seed=3)
    m = ref.from_csr(a)
    lo, hi = osolve.lanczos_bounds(orc, a, 30, 2)
    rlo, rhi = ref.lanczos_bounds(m, 30, 2)
    assert abs(lo - rlo) <= 1e-9 and abs(hi - rhi) <= 1e-9
    mu = osolve.kpm_dos(orc, a, (-5.6, 5.6), 300, 8, 11)
    rmu = ref.kpm_dos(m, (-5.6, 5.6), 300, 8, 11)
    assert np.max(np.abs(mu - rmu)) <= 1e-9 * mu[0]
    for lo_, hi_ in ((-1.0, 1.0), (-5.6, 0.3)):
        assert abs(osolve.dos_count(orc, mu, (-5.6, 5.6), lo_, hi_)
                   - ref.dos_count(rmu, (-5.6, 5.6), lo_, hi_)) <= 1e-9


def test_svqb_and_rr_match_reference(orc, ref):
    a = orc.graphene(8, 8, disorder=0.3, seed=2)
    m = ref.from_csr(a)
    y = orc.randomize(a.dim, 10, 4)
    q, r = osolve.svqb(orc, y)
    rq, rr = ref.svqb(y)
    assert r == rr == 10
    assert np.max(np.abs(q @ q.T - rq @ rq.T)) <= 1e-12  # same span, rotation-free
    vals, v, res = osolve.rayleigh_ritz(orc, a, q)
    rvals, rv, rres = ref.rayleigh_ritz(m, rq)
    assert np.max(np.abs(vals - rvals)) <= 1e-12
    assert np.max(np.abs(res - rres)) <= 1e-10
    y[:, 9] = y[:, 2]
    assert osolve.svqb(orc, y)[1] == 9  # test_solver.cpp:75-82
    with pytest.raises(RuntimeError):
        osolve.svqb(orc, np.zeros((32, 2)))
