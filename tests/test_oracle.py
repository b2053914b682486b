"""CPU: pin the oracle (oracle/chebfd_oracle.c) against the reference.

(a) golden fixtures written from the compiled reference by
    tests/golden/make_golden.py (always available, committed);
(b) the reference's own known-answer tests (test_filter.cpp,
    test_core_linalg.cpp, test_models.cpp, test_bench.cpp);
(c) the compiled reference itself (oracle/_ref) where it was built.
Integer / generator / RNG / row-local results are compared bit for bit.
"""
import math
import os

import numpy as np
import pytest

GOLD = np.load(os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz"))


def bits(a, b):
    a, b = np.ascontiguousarray(a), np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


MODELS = {
    "g_8x8_per": ("graphene", (8, 8), dict(disorder=0.1, seed=1, boundary="periodic_xy_open_z")),
    "g_4x3_open": ("graphene", (4, 3), dict(disorder=1.5, seed=12, boundary="open_all")),
    "g_1x2_per": ("graphene", (1, 2), dict(disorder=0.5, seed=5, boundary="periodic_all")),
    "ti_3x3x3_slab": ("ti", (3, 3, 3), dict(disorder=2.0, seed=9, boundary="periodic_xy_open_z")),
    "ti_4x4x4_per": ("ti", (4, 4, 4), dict(disorder=1.0, seed=1, boundary="periodic_all")),
    "ti_2x2x2_per": ("ti", (2, 2, 2), dict(disorder=0.5, seed=3, boundary="periodic_all")),
    "ti_3x2x2_open": ("ti", (3, 2, 2), dict(disorder=0.5, seed=4, boundary="open_all")),
}


@pytest.mark.parametrize("name", sorted(MODELS))
def test_models_match_golden(orc, name):
    kind, l, kw = MODELS[name]
    c = orc.graphene(*l, **kw) if kind == "graphene" else orc.topological_insulator(*l, **kw)
    assert np.array_equal(c.offs, GOLD[f"model_{name}_offs"])
    assert np.array_equal(c.cols, GOLD[f"model_{name}_cols"])
    assert bits(c.vals, GOLD[f"model_{name}_vals"])


def test_rng_streams_match_golden(orc):
    assert bits(orc.randomize(50, 7, 3, False), GOLD["rng_real_50x7_s3"])
    assert bits(orc.randomize(20, 5, 9, True), GOLD["rng_cplx_20x5_s9"])


def test_mt19937_64_known_answer(orc):
    # std::mt19937_64 default seed 5489: 10000th output (C++11 [rand.predef])
    st = orc.mt19937_64(5489, 10000)
    assert int(st[-1]) == 9981545732273789042


@pytest.mark.parametrize("k", ["none", "fejer", "jackson", "lanczos2", "lanczos3"])
def test_filters_match_golden(orc, k):
    comb, a, b = orc.make_filter((-0.13, 0.21), (-3.05, 3.1), 64, k)
    assert bits(np.concatenate([[a, b], comb]), GOLD[f"filter_{k}"])


def test_apply_filter_matches_golden(orc):
    for tag, model in (("g", ("graphene", (8, 8), dict(disorder=0.1, seed=1))),
                       ("t", ("ti", (3, 3, 3), dict(disorder=0.5, seed=2)))):
        kind, l, kw = model
        c = orc.graphene(*l, **kw) if kind == "graphene" else orc.topological_insulator(*l, **kw)
        f = GOLD[f"apply_{tag}_filter"]
        y, mom = orc.apply_filter(c, GOLD[f"apply_{tag}_x0"], f[2:], f[0], f[1], want_moments=True)
        assert bits(y, GOLD[f"apply_{tag}_y"])
        assert bits(mom, GOLD[f"apply_{tag}_mom"])  # one-chunk sums = 1-thread reference


def test_fused_and_gram_match_golden(orc):
    c = orc.topological_insulator(3, 3, 3, disorder=0.5, seed=2)
    u, w, x = (GOLD[f"fused_t_{s}"].copy() for s in "uwx")
    d = orc.spmmvm_fused(c, u, w, x, 0.37, -0.21, 0.83, want_dots=True)
    assert bits(w, GOLD["fused_t_w_out"]) and bits(x, GOLD["fused_t_x_out"])
    assert bits(d, GOLD["fused_t_dots"])
    assert bits(orc.gram(GOLD["fused_t_u"], GOLD["fused_t_w_out"]), GOLD["gram_t"])  # w after the step


# ---- the reference's own known answers ---------------------------------------
def test_window_closed_forms(orc):
    """test_filter.cpp:28-52"""
    c = orc.window_coeffs((-1.0, 1.0), (-1.0, 1.0), 8)
    assert abs(c[0] - 1.0) <= 1e-14 and np.all(np.abs(c[1:]) <= 1e-14)
    c = orc.window_coeffs((-0.5, 0.5), (-1.0, 1.0), 4)
    assert abs(c[0] - 1 / 3) <= 1e-14 * (1 + 1 / 3)
    assert abs(c[1]) <= 1e-14
    assert abs(c[2] + math.sqrt(3) / math.pi) <= 1e-14 * (1 + math.sqrt(3) / math.pi)
    assert np.all(np.abs(orc.window_coeffs((-0.123, 0.123), (-1, 1), 31)[1::2]) <= 1e-14)
    assert np.all(np.abs(orc.window_coeffs((1.7, 2.3), (1.0, 3.0), 31)[1::2]) <= 1e-13)
    assert orc.window_coeffs((-0.001, 0.001), (-1, 1), 3)[0] > 0


def test_kernel_known_values(orc):
    """test_filter.cpp:54-75"""
    for k in ("none", "fejer", "jackson", "lanczos2"):
        assert abs(orc.kernel_coeffs(k, 5)[0] - 1.0) <= 1e-14
    assert abs(orc.kernel_coeffs("fejer", 3)[2] - 0.5) <= 1e-15
    assert abs(orc.kernel_coeffs("lanczos2", 1)[1] - 4 / math.pi ** 2) <= 1e-14
    assert np.all(orc.kernel_coeffs("none", 7) == 1.0)
    g = orc.kernel_coeffs("jackson", 50)
    assert np.all(np.diff(g) <= 1e-14) and np.all(g >= -1e-14) and g[50] <= 1e-2


def test_eval_scalar_known_answers(orc):
    """test_filter.cpp:83-140"""
    comb, a, b = orc.make_filter((-2.0, 4.0), (-2.0, 4.0), 16, "none")
    for x in (-2.0, -1.0, 0.3, 2.5, 4.0):
        assert abs(orc.eval_scalar(comb, a, b, x) - 1.0) <= 1e-12
    comb, a, b = orc.make_filter((-0.01, 0.01), (-1.0, 1.0), 200, "lanczos2")
    for x in (0.0, 0.005, -0.3, 0.77, 0.999):
        t = math.acos(a * x + b)
        ref = sum(float(np.longdouble(comb[n]) * np.cos(np.longdouble(n * t))) for n in range(201))
        assert abs(orc.eval_scalar(comb, a, b, x) - ref) <= 1e-12 * max(1.0, abs(ref))
    comb, a, b = orc.make_filter((-0.001, 0.001), (-1.0, 1.0), 64926, "lanczos2")
    for x in (-1.0, -0.5, 0.0, 0.0005, 0.7, 1.0):
        v = orc.eval_scalar(comb, a, b, x)
        assert math.isfinite(v) and abs(v) <= 2.0


def _diag(v):
    import oracle
    n = len(v)
    return oracle.CSR(np.arange(n + 1), np.arange(n), np.asarray(v, dtype=np.float64))


def test_apply_filter_diagonal_known_answer(orc):
    """test_filter.cpp:142-154"""
    lam = [-0.8, -0.3, 0.0, 0.25, 0.6, 0.95]
    comb, a, b = orc.make_filter((-0.1, 0.3), (-1.0, 1.0), 40, "lanczos2")
    y, _ = orc.apply_filter(_diag(lam), 2.0 * np.eye(6), comb, a, b)
    want = np.diag([2.0 * orc.eval_scalar(comb, a, b, l) for l in lam])
    assert np.max(np.abs(y - want)) <= 1e-12


def test_degree2_filter_explicit_polynomial(orc):
    """test_filter.cpp:156-198 (random symmetric 8x8, degree 2, Jackson)."""
    rng = np.random.default_rng(3)
    d = 8
    h = np.triu(rng.uniform(-0.1, 0.1, (d, d)))
    A = h + np.triu(h, 1).T
    import oracle
    csr = oracle.CSR(np.arange(0, d * d + 1, d), np.tile(np.arange(d), d), A.reshape(-1))
    comb, a, b = orc.make_filter((-0.2, 0.2), (-1.0, 1.0), 2, "jackson")
    hm = a * A + b * np.eye(d)
    pa = comb[0] * np.eye(d) + comb[1] * hm + comb[2] * (2 * hm @ hm - np.eye(d))
    x = orc.randomize(d, 3, 4)
    y, _ = orc.apply_filter(csr, x, comb, a, b)
    assert np.max(np.abs(y - pa @ x)) <= 1e-13


def test_moments_known_answer(orc):
    """test_filter.cpp:200-224: diagonal A, <x, T_n(h) x> in long double."""
    lam = np.array([-0.95 + 1.9 * i / 95.0 for i in range(96)])
    comb, a, b = orc.make_filter((-0.3, 0.1), (-1.0, 1.0), 25, "lanczos2")
    x = orc.randomize(96, 3, 77)
    _, mom = orc.apply_filter(_diag(lam), x, comb, a, b, want_moments=True)
    t = np.arccos(np.longdouble(a) * lam.astype(np.longdouble) + np.longdouble(b))
    for n in range(26):
        ref = (np.cos(n * t)[:, None] * x.astype(np.longdouble) ** 2).sum(axis=0)
        assert np.all(np.abs(mom[n] - ref.astype(np.float64)) <= 1e-10 * np.maximum(1, abs(ref)))


def test_fused_equals_unfused(orc):
    """test_core_linalg.cpp:131-155"""
    rng = np.random.default_rng(23)
    d = 64
    h = np.triu(0.1 * rng.uniform(-1, 1, (d, d)))
    A = h + np.triu(h, 1).T
    import oracle
    csr = oracle.CSR(np.arange(0, d * d + 1, d), np.tile(np.arange(d), d), A.reshape(-1))
    u, w, x = (orc.randomize(d, 4, s) for s in (1, 2, 3))
    alpha, beta, coeff = 0.37, -0.21, 0.83
    w_ref = orc.spmmvm(csr, u, 2 * alpha, 2 * beta)
    orc.block_axpy_scal(w_ref, w, w, 1.0, -1.0, 0.0)
    x_ref = x.copy()
    orc.block_axpy_scal(x_ref, w_ref, w_ref, 1.0, coeff, 0.0)
    dots_ref = orc.column_dots(x, w_ref)
    dots = orc.spmmvm_fused(csr, u, w, x, alpha, beta, coeff, want_dots=True)
    scale = lambda a: np.max(np.abs(a))  # noqa: E731
    assert np.max(np.abs(w - w_ref)) <= 1e-13 * scale(w_ref)
    assert np.max(np.abs(x - x_ref)) <= 1e-13 * scale(x_ref)
    assert np.allclose(dots, dots_ref, rtol=1e-12)


def test_fused_rejects_aliasing(orc):
    c = orc.graphene(2, 2)
    u = orc.randomize(c.dim, 2, 1)
    w = orc.randomize(c.dim, 2, 2)
    with pytest.raises(ValueError):
        orc.spmmvm_fused(c, u, w, w, 1.0, 0.0, 0.5)


def test_model_structure_known_answers(orc):
    """test_models.cpp:94-121,177-208"""
    p = orc.topological_insulator(4, 4, 4, disorder=1.0, boundary="periodic_all")
    assert p.nnz / p.dim == 11.0
    s = orc.topological_insulator(4, 4, 4, disorder=1.0, boundary="periodic_xy_open_z")
    assert s.nnz == p.nnz - 2 * 4 * 4 * 2
    for c in (p, s, orc.graphene(8, 8, disorder=1.5, seed=12)):
        d = c.to_dense()
        assert np.array_equal(d, d.conj().T)  # exactly Hermitian
    g = orc.graphene(16, 16, boundary="periodic_all")
    assert g.nnz / g.dim == 4.0
    gd = orc.graphene(8, 8, disorder=1.5, seed=12).to_dense()
    assert np.all(np.abs(np.diag(gd)) <= 0.75)


def test_clean_ti_bulk_gap(orc):
    """test_models.cpp:123-148: clean periodic 4^3 bulk gap = 1, slab gap smaller."""
    ev = np.linalg.eigvalsh(orc.topological_insulator(4, 4, 4, boundary="periodic_all").to_dense())
    assert np.allclose(ev, -ev[::-1], atol=1e-9)
    assert abs(np.min(np.abs(ev)) - 1.0) <= 1e-9
    evs = np.linalg.eigvalsh(orc.topological_insulator(4, 4, 4).to_dense())
    assert np.min(np.abs(evs)) < 1.0


def test_intensity_model_known_values(orc):
    """test_bench.cpp:11-36 (bench.cpp:28-42 conventions)."""
    def intensity(n_nzr, s_d, s_i, f_a, f_m, nb):
        return orc.per_row_flops(n_nzr, f_a, f_m) / orc.per_row_bytes(n_nzr, s_d, s_i, nb)
    assert abs(intensity(13, 16, 4, 2, 6, 1) - 146 / 340) <= 1e-12
    assert abs(intensity(13, 16, 4, 2, 6, 1 << 20) - 146 / 80) <= 1e-4 * 146 / 80
    assert abs(intensity(4, 8, 4, 1, 1, 16) - 19 / 43) <= 1e-12
    assert abs(intensity(7, 8, 4, 1, 1, 2) - 25 / 82) <= 1e-12


# ---- against the compiled reference, when it is present --------------------------
def test_oracle_matches_compiled_reference(orc, ref):
    for l in [(3, 3, 3), (2, 5, 3)]:
        c = orc.topological_insulator(*l, disorder=0.5, seed=5)
        m = ref.topological_insulator(*l, disorder=0.5, seed=5)
        rc = m.csr()
        assert np.array_equal(c.cols, rc.cols) and bits(c.vals, rc.vals)
        x = orc.randomize(c.dim, 5, 9, True)
        comb, a, b = orc.make_filter((-0.1, 0.1), (-5.6, 5.6), 30, "lanczos2")
        y1, m1 = orc.apply_filter(c, x, comb, a, b, True)
        y2, m2 = ref.apply_filter(m, x, comb, a, b, True)
        assert bits(y1, y2) and bits(m1, m2)
    assert bits(orc.randomize(33, 4, 2, True), ref.randomize(33, 4, 2, True))
