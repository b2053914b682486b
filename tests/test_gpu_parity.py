"""GPU parity: the sm_100a path through the C ABI against the CPU oracle.

Row-local results (spmmvm, fused step W/X, apply_filter X) are compared
BIT-FOR-BIT: the kernels evaluate each entry with the reference's exact
operation order (no FMA contraction), see kernels.cu header.  Reductions
(dots, moments, Gram) differ only in summation order and are compared with a
relative tolerance written in each test.
"""
import numpy as np
import pytest

import paper_1510_04895_b200 as cf

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def rel(a, b):
    return np.max(np.abs(a - b)) / max(np.max(np.abs(b)), 1e-300)


def graphene(ctx, orc, lx, ly, disorder=0.1, seed=1, boundary="periodic_xy_open_z"):
    A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(lx, ly, disorder=disorder, seed=seed,
                                                     boundary=boundary))
    return A, orc.graphene(lx, ly, disorder=disorder, seed=seed, boundary=boundary)


def ti(ctx, orc, l, disorder=0.5, seed=1, boundary="periodic_xy_open_z"):
    A = cf.SparseMatrix.topological_insulator(
        ctx, cf.LatticeSpec(*l, disorder=disorder, seed=seed, boundary=boundary))
    return A, orc.topological_insulator(*l, disorder=disorder, seed=seed, boundary=boundary)


def block(A, host):
    return cf.BlockVector(A, host.shape[1]).upload(host)


CASES = [
    ("graphene", (8, 8), 5), ("graphene", (16, 16), 40), ("graphene", (13, 7), 1),
    ("graphene", (16, 16), 3), ("ti", (4, 4, 4), 5), ("ti", (3, 5, 4), 32), ("ti", (4, 4, 4), 1),
]


def make_case(ctx, orc, name, l):
    return graphene(ctx, orc, *l) if name == "graphene" else ti(ctx, orc, l)


@pytest.mark.parametrize("name,l,nb", CASES)
def test_spmmvm_bitexact(ctx, orc, name, l, nb):
    A, c = make_case(ctx, orc, name, l)
    x = orc.randomize(c.dim, nb, 11, name == "ti")
    for alpha, beta in ((1.0, 0.0), (0.37, -0.21)):
        y = cf.spmmvm(A, block(A, x), alpha, beta).to_numpy()
        assert bits_equal(y, orc.spmmvm(c, x, alpha, beta))


@pytest.mark.parametrize("name,l,nb", CASES)
def test_fused_bitexact_and_dots(ctx, orc, name, l, nb):
    A, c = make_case(ctx, orc, name, l)
    cx = name == "ti"
    u, w, x = (orc.randomize(c.dim, nb, s, cx) for s in (1, 2, 3))
    U, W, X = block(A, u), block(A, w), block(A, x)
    d = cf.spmmvm_fused(A, U, W, X, 0.37, -0.21, 0.83, dots=True)
    dref = orc.spmmvm_fused(c, u, w, x, 0.37, -0.21, 0.83, want_dots=True)
    assert bits_equal(W.to_numpy(), w)
    assert bits_equal(X.to_numpy(), x)
    # Kahan dots vs Kahan dots, different summation order: 1e-12 relative
    # (test_core_linalg.cpp:152 uses 1e-12 against the unfused dots)
    assert np.allclose(d, dref, rtol=1e-12, atol=1e-12 * np.max(np.abs(dref)))


@pytest.mark.parametrize("name,l,nb", CASES[:5])
def test_recurrence_step_bitexact(ctx, orc, name, l, nb):
    A, c = make_case(ctx, orc, name, l)
    cx = name == "ti"
    u, w = (orc.randomize(c.dim, nb, s, cx) for s in (4, 5))
    U, W = block(A, u), block(A, w)
    cf.recurrence_step(A, U, W, 0.6, 0.1)
    orc.recurrence_step(c, u, w, 0.6, 0.1)
    assert bits_equal(W.to_numpy(), w)


def test_axpy_bitexact(ctx, orc):
    A, c = ti(ctx, orc, (3, 3, 3))
    x, u, w = (orc.randomize(c.dim, 4, s, True) for s in (1, 2, 3))
    X, U, W = block(A, x), block(A, u), block(A, w)
    cf.block_axpy_scal(X, U, W, 0.2, -1.3, 0.7)
    orc.block_axpy_scal(x, u, w, 0.2, -1.3, 0.7)
    assert bits_equal(X.to_numpy(), x)


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("name,l,nb,deg", [
    ("graphene", (16, 16), 40, 50), ("graphene", (8, 8), 3, 7), ("ti", (4, 4, 4), 32, 40),
    ("ti", (3, 3, 2), 5, 2), ("graphene", (8, 8), 1, 3)])
def test_apply_filter_bitexact_with_moments(ctx, orc, name, l, nb, deg, graphs):
    ctx.set_option("graphs", graphs)
    try:
        A, c = make_case(ctx, orc, name, l)
        bounds = (-3.2, 3.3) if name == "graphene" else (-5.6, 5.6)
        p = cf.make_filter((-0.2, 0.3), bounds, deg, "lanczos2")
        x0 = orc.randomize(c.dim, nb, 9, name == "ti")
        X = block(A, x0)
        mom = cf.apply_filter(A, X, p, want_moments=True)
        xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=True)
        assert bits_equal(X.to_numpy(), xr)
        # moments: plain sums in a different order; 1e-12 of the column norm
        scale = np.max(np.abs(mr[0]))
        assert np.max(np.abs(mom.m - mr)) <= 1e-12 * scale
        # second call (graph replay / cache hit) with new coefficients
        p2 = cf.make_filter((-0.1, 0.4), bounds, deg, "jackson")
        X.upload(x0)
        cf.apply_filter(A, X, p2)
        xr2, _ = orc.apply_filter(c, x0, p2.combined, p2.alpha, p2.beta)
        assert bits_equal(X.to_numpy(), xr2)
    finally:
        ctx.set_option("graphs", True)


PAIR_CASES = [
    ("ti", (4, 4, 4), 5, 9, {}), ("ti", (6, 5, 8), 32, 12, {"pair_tile_rows": 32}),
    ("ti", (6, 6, 6), 16, 11, {"pair_slab": 5}), ("ti", (5, 6, 7), 8, 10, {"pair_extra": 0}),
    ("graphene", (16, 16), 40, 10, {"pair_threads": 256}), ("graphene", (13, 7), 1, 7, {}),
    ("graphene", (16, 16), 3, 8, {"pair_hints": 0}),
]


@pytest.mark.parametrize("name,l,nb,deg,knobs", PAIR_CASES)
def test_apply_filter_pair_kernel_bitexact(ctx, orc, name, l, nb, deg, knobs):
    """Two fused steps per launch (pair.cu, option pair=2): X bit-identical to the
    oracle's apply_filter (filter.hpp:73-116), moments (direct <x0, w> mode, which the
    pair kernel carries through both steps) within 1e-12.  Opt-in variant: only in an
    EXPERIMENTAL=1 build (elsewhere the option must be refused)."""
    if not cf.experimental_build():
        with pytest.raises(cf.Unsupported):
            ctx.set_option("pair", 2)
        pytest.skip("pair kernel not in this build (make EXPERIMENTAL=1)")
    ctx.set_option("pair", 2)
    ctx.set_option("moments", "direct")
    for k, v in knobs.items():
        ctx.set_option(k, v)
    try:
        A, c = make_case(ctx, orc, name, l)
        bounds = (-3.2, 3.3) if name == "graphene" else (-5.6, 5.6)
        p = cf.make_filter((-0.2, 0.3), bounds, deg, "lanczos2")
        x0 = orc.randomize(c.dim, nb, 19, name == "ti")
        X = block(A, x0)
        before = ctx.launch_count
        mom = cf.apply_filter(A, X, p, want_moments=True)
        launched = ctx.launch_count - before
        xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=True)
        assert bits_equal(X.to_numpy(), xr)
        assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
        # start-up steps + ceil((deg - 2) / 2) launches per column slab
        if "pair_slab" not in knobs:
            assert launched == 2 + (deg - 2 + 1) // 2
    finally:
        ctx.set_option("pair", 0)
        ctx.set_option("moments", "doubling")
        for k in knobs:
            ctx.set_option(k, -1 if k == "pair_extra" else (1 if k == "pair_hints" else 0))


MOMENT_CASES = [("ti", (4, 4, 4), 5), ("ti", (3, 5, 4), 32), ("graphene", (16, 16), 40),
                ("graphene", (13, 7), 1), ("graphene", (16, 16), 3)]


@pytest.mark.parametrize("name,l,nb", MOMENT_CASES)
@pytest.mark.parametrize("deg", [2, 3, 4, 5, 30, 101])
@pytest.mark.parametrize("mode", ["doubling", "direct"])
def test_apply_filter_moments_both_modes(ctx, orc, name, l, nb, deg, mode):
    """MomentTable (filter.hpp:61-68, 86-113) by direct <x0, T_n x0> dots and by the
    Chebyshev doubling identities (Hermitian lattices): within 1e-12 of the column norm
    of the oracle's direct sums; X stays bit-exact."""
    ctx.set_option("moments", mode)
    try:
        A, c = make_case(ctx, orc, name, l)
        bounds = (-3.2, 3.3) if name == "graphene" else (-5.6, 5.6)
        p = cf.make_filter((-0.25, 0.2), bounds, deg, "jackson")
        x0 = orc.randomize(c.dim, nb, 31, name == "ti")
        X = block(A, x0)
        mom = cf.apply_filter(A, X, p, want_moments=True)
        xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=True)
        assert bits_equal(X.to_numpy(), xr)
        assert mom.m.shape == mr.shape
        assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
    finally:
        ctx.set_option("moments", "doubling")


@pytest.mark.parametrize("group", [0, 2, 3])
@pytest.mark.parametrize("deg", [2, 3, 4, 5, 6, 7, 8, 31])
@pytest.mark.parametrize("mode", ["doubling", "direct"])
def test_apply_filter_delayed_x_groups(ctx, orc, group, deg, mode):
    """X updated once per G steps (V_n-only steps, then one step adding the group's terms in
    the reference's order): X bit-identical to the oracle's per-step update, moments within
    1e-12, for every tail length (degree - 2 mod G)."""
    ctx.set_option("delayed_x", group)
    ctx.set_option("moments", mode)
    try:
        A, c = ti(ctx, orc, (4, 5, 4))
        p = cf.make_filter((-0.25, 0.2), (-5.6, 5.6), deg, "lanczos2")
        x0 = orc.randomize(c.dim, 6, 17, True)
        X = block(A, x0)
        mom = cf.apply_filter(A, X, p, want_moments=True)
        xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=True)
        assert bits_equal(X.to_numpy(), xr)
        assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
    finally:
        ctx.set_option("delayed_x", 3)
        ctx.set_option("moments", "doubling")


def test_moments_non_hermitian_operator_uses_direct_dots(ctx, orc):
    """A from_csr operator that is not bitwise Hermitian must not use the doubling
    identities (they would give wrong moments): moments equal the oracle's direct sums."""
    rng = np.random.default_rng(3)
    d = 40
    dense = np.where(rng.random((d, d)) < 0.15, rng.uniform(-1, 1, (d, d)), 0.0)
    np.fill_diagonal(dense, rng.uniform(-1, 1, d))
    offs = np.concatenate([[0], np.cumsum((dense != 0).sum(1))]).astype(np.int64)
    cols = np.nonzero(dense)[1].astype(np.int64)
    vals = dense[dense != 0]
    A = cf.SparseMatrix.from_csr(ctx, d, offs, cols, vals)
    import oracle
    c = oracle.CSR(offs, cols, vals)
    p = cf.make_filter((-0.2, 0.2), (-4.0, 4.0), 12, "lanczos2")
    x0 = orc.randomize(d, 3, 2)
    X = block(A, x0)
    mom = cf.apply_filter(A, X, p, want_moments=True)
    xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=True)
    assert bits_equal(X.to_numpy(), xr)
    assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
    # and the symmetric part of it is detected as Hermitian (doubling within tolerance)
    sym = np.triu(dense) + np.triu(dense, 1).T
    offs = np.concatenate([[0], np.cumsum((sym != 0).sum(1))]).astype(np.int64)
    cols = np.nonzero(sym)[1].astype(np.int64)
    vals = sym[sym != 0]
    B = cf.SparseMatrix.from_csr(ctx, d, offs, cols, vals)
    XB = block(B, x0)
    momb = cf.apply_filter(B, XB, p, want_moments=True)
    xr, mr = orc.apply_filter(oracle.CSR(offs, cols, vals), x0, p.combined, p.alpha, p.beta,
                              want_moments=True)
    assert bits_equal(XB.to_numpy(), xr)
    assert np.max(np.abs(momb.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))


def test_apply_filter_host_e2e(ctx, orc):
    A, c = ti(ctx, orc, (4, 4, 3))
    p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), 30, "lanczos2")
    x = orc.randomize(c.dim, 8, 3, True)
    y = x.copy()
    cf.apply_filter_host(A, y, p)
    xr, _ = orc.apply_filter(c, x, p.combined, p.alpha, p.beta)
    assert bits_equal(y, xr)


def test_filter_pipe_streams_bitexact(ctx, orc):
    """chebfd_filter_pipe: five jobs in flight over two device slots (pinned and
    pageable host blocks, in place and out of place) equal the oracle's filter."""
    A, c = ti(ctx, orc, (5, 4, 6))
    nb = 6
    pipe = cf.FilterPipe(A, nb)
    try:
        ps = [cf.make_filter((-0.3, 0.2 + 0.05 * k), (-5.6, 5.6), 20 + 3 * k, "lanczos2")
              for k in range(5)]
        xs = [orc.randomize(c.dim, nb, 40 + k, True) for k in range(5)]
        ins, outs = [], []
        for k in range(5):
            xin = cf.host_array(xs[k].shape, np.complex128) if k % 2 == 0 else xs[k].copy()
            xin[:] = xs[k]
            xout = xin if k < 3 else np.empty_like(xs[k])
            pipe.submit(xin, ps[k], xout)
            ins.append(xin)
            outs.append(xout)
        pipe.wait()
        for k in range(5):
            xr, _ = orc.apply_filter(c, xs[k], ps[k].combined, ps[k].alpha, ps[k].beta)
            assert bits_equal(outs[k], xr), k
    finally:
        pipe.close()


def test_block_equals_independent_columns(ctx, orc):
    """test_core_linalg.cpp:87-99 for the whole filter: columns never mix."""
    A, c = ti(ctx, orc, (6, 6, 6))
    p = cf.make_filter((-0.2, 0.2), (-5.6, 5.6), 60, "lanczos2")
    x = orc.randomize(c.dim, 6, 21, True)
    X = block(A, x)
    cf.apply_filter(A, X, p)
    full = X.to_numpy()
    for k in (0, 3, 5):
        Xk = block(A, np.ascontiguousarray(x[:, k:k + 1]))
        cf.apply_filter(A, Xk, p)
        assert bits_equal(Xk.to_numpy()[:, 0], full[:, k])


def test_diagonal_filter_known_answer(ctx):
    """test_filter.cpp:142-154: apply_filter on a diagonal = eval_scalar."""
    lam = np.array([-0.8, -0.3, 0.0, 0.25, 0.6, 0.95])
    A = cf.SparseMatrix.from_csr(ctx, 6, np.arange(7), np.arange(6), lam)
    p = cf.make_filter((-0.1, 0.3), (-1.0, 1.0), 40, "lanczos2")
    X = cf.BlockVector(A, 6).upload(2.0 * np.eye(6))
    cf.apply_filter(A, X, p)
    want = np.diag([2.0 * cf.eval_scalar(p, v) for v in lam])
    assert np.max(np.abs(X.to_numpy() - want)) <= 1e-12


def test_fused_coeff0_is_T2(ctx):
    """test_core_linalg.cpp:101-116"""
    d = np.array([-0.9, -0.3, 0.2, 0.8])
    A = cf.SparseMatrix.from_csr(ctx, 4, np.arange(5), np.arange(4), d)
    U = cf.BlockVector(A, 1).upload(d[:, None])
    W = cf.BlockVector(A, 1).upload(np.ones((4, 1)))
    X = cf.BlockVector(A, 1).upload(np.full((4, 1), 0.5))
    cf.spmmvm_fused(A, U, W, X, 1.0, 0.0, 0.0)
    assert np.allclose(W.to_numpy()[:, 0], 2 * d * d - 1, rtol=1e-15)
    assert np.array_equal(X.to_numpy(), np.full((4, 1), 0.5))


def test_fused_rejects_aliasing(ctx, orc):
    """test_core_linalg.cpp:157-164"""
    A, c = graphene(ctx, orc, 4, 4)
    U = cf.BlockVector(A, 2).randomize(1)
    W = cf.BlockVector(A, 2).randomize(2)
    with pytest.raises(cf.InvalidArgument):
        cf.spmmvm_fused(A, U, W, W, 1.0, 0.0, 0.5)
    with pytest.raises(cf.InvalidArgument):
        cf.spmmvm_fused(A, U, U, W, 1.0, 0.0, 0.5)


def test_apply_filter_rejects_degree_below_2(ctx):
    """test_filter.cpp:226-235"""
    A = cf.SparseMatrix.from_csr(ctx, 2, np.arange(3), np.arange(2), np.array([0.0, 0.5]))
    p = cf.make_filter((-0.5, 0.5), (-1.0, 1.0), 4, "none")
    p.degree = 1
    p.combined = p.combined[:2]
    X = cf.BlockVector(A, 1).randomize(1)
    with pytest.raises(cf.InvalidArgument):
        cf.apply_filter(A, X, p)


def test_randomize_matches_reference_stream(ctx, orc):
    A, c = ti(ctx, orc, (3, 3, 3))
    X = cf.BlockVector(A, 7).randomize(42)
    assert bits_equal(X.to_numpy(), orc.randomize(c.dim, 7, 42, True))
    B, cg = graphene(ctx, orc, 5, 5)
    Y = cf.BlockVector(B, 3).randomize(5)
    assert bits_equal(Y.to_numpy(), orc.randomize(cg.dim, 3, 5, False))


@pytest.mark.parametrize("cx", [False, True])
def test_reductions(ctx, orc, cx):
    A, c = (ti(ctx, orc, (4, 4, 4)) if cx else graphene(ctx, orc, 16, 16))
    x = orc.randomize(c.dim, 6, 1, cx)
    y = orc.randomize(c.dim, 6, 2, cx)
    X, Y = block(A, x), block(A, y)
    assert rel(cf.column_dots(X, Y), orc.column_dots(x, y)) <= 1e-13
    assert rel(cf.column_norms(X), orc.column_norms(x)) <= 1e-14
    assert rel(cf.gram(X, Y), orc.gram(x, y)) <= 1e-13
    b = orc.randomize(6, 4, 3, cx)
    assert rel(cf.block_mult_small(X, b).to_numpy(), orc.block_mult_small(x, b)) <= 1e-13


def test_gram_kahan_exact_count(ctx):
    """test_core_linalg.cpp:399-403: gram of ones counts the dimension."""
    n = 1000
    A = cf.SparseMatrix.from_csr(ctx, n, np.arange(n + 1), np.arange(n), np.ones(n))
    X = cf.BlockVector(A, 1).upload(np.ones((n, 1)))
    assert cf.gram(X, X)[0, 0] == 1000.0


def test_cpp_dropin_layer_on_device(lib_built, tmp_path):
    """include/chebfd_b200.hpp used from C++ against the device (tests/cpp)."""
    import os
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = tmp_path / "use"
    r = subprocess.run(["/usr/bin/g++", "-std=c++20", "-O1", f"-I{root}/include",
                        os.path.join(root, "tests", "cpp", "use_wrapper.cpp"), "-o", str(out),
                        f"-L{os.path.dirname(lib_built)}", "-lchebfd_b200",
                        f"-Wl,-rpath,{os.path.dirname(lib_built)}"], capture_output=True, text=True)
    assert r.returncode == 0, r.stderr[-2000:]
    run = subprocess.run([str(out), "--device", str(tmp_path)], capture_output=True, text=True,
                         timeout=120)
    assert run.returncode == 0, run.stdout + run.stderr


def test_set_option_invalidates_captured_filters(ctx, orc):
    """Options change which kernels a filter launches; a graph captured before
    the change must not be replayed after it (results stay bit-exact)."""
    A, c = ti(ctx, orc, (4, 4, 6))
    p = cf.make_filter((-0.2, 0.3), (-5.6, 5.6), 12, "lanczos2")
    x0 = orc.randomize(c.dim, 8, 4, True)
    xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=False)
    X = block(A, x0)

    def run():
        X.upload(x0)
        before = ctx.launch_count
        cf.apply_filter(A, X, p)
        assert bits_equal(X.to_numpy(), xr)
        return ctx.launch_count - before

    d0 = run()
    assert run() == d0  # replay of the captured graph
    try:
        ctx.set_option("slab_units", 2)  # 8 complex columns -> 4 column slabs per step
        assert run() > d0
        ctx.set_option("kernel", "gather")
        run()
    finally:
        ctx.set_option("slab_units", 0)
        ctx.set_option("kernel", "tma")
    assert run() == d0


@pytest.mark.parametrize("cplx", [False, True])
def test_streamed_randomize_matches_reference_stream(ctx, cplx):
    """Blocks above 4 M entries are randomized in pieces through pinned
    buffers (NormalStream); every piece continues the reference's stream."""
    if cplx:
        A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(16, 16, 64, disorder=0.5))
        nb = 81  # 65536 x 81 = 5.3 M entries: two pieces
    else:
        A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(512, 256, disorder=0.5))
        nb = 19  # 262144 x 19 = 4.98 M entries: one full piece + a ragged tail
    X = cf.BlockVector(A, nb).randomize(11)
    want = cf.host_randomize(A.dim(), nb, 11, cplx)
    assert bits_equal(X.to_numpy(), want)


STAGE_CASES = [("ti", (4, 4, 4), 32, "periodic_xy_open_z", "stage"),
               ("ti", (3, 5, 4), 32, "open_all", "stage"),
               ("graphene", (16, 16), 64, "periodic_xy_open_z", "tma2"),
               ("graphene", (13, 7), 64, "open_all", "tma2"),
               ("graphene", (16, 8), 32, "open_all", "tma2"),
               ("graphene", (16, 8), 32, "periodic_all", "tma")]


@pytest.mark.parametrize("name,l,nb,boundary,kernel", STAGE_CASES)
def test_staged_kernel_bitexact(ctx, orc, name, l, nb, boundary, kernel):
    """Kernel variants 2 (gathered rows staged in shared memory by TMA, per-chunk
    plan; rows of >= 8 entries) and 3 / default for short rows (two units per
    thread, 256-bit accesses, W/X staged by TMA): apply_filter X bit-exact with
    moments, fused W/X bit-exact with dots, on full, padded (open boundaries)
    and partial chunks."""
    cx = name == "ti"
    if cx:
        A, c = ti(ctx, orc, l, boundary=boundary)
    else:
        A, c = graphene(ctx, orc, *l, boundary=boundary)
    if kernel == "stage" and not cf.experimental_build():
        with pytest.raises(cf.Unsupported):
            ctx.set_option("kernel", kernel)
        pytest.skip("staged-gather kernel not in this build (make EXPERIMENTAL=1)")
    if kernel == "stage":
        assert A.info["stage_rows"] > 0
    ctx.set_option("kernel", kernel)
    try:
        bounds = (-5.6, 5.6) if cx else (-3.2, 3.3)
        p = cf.make_filter((-0.2, 0.3), bounds, 24, "lanczos2")
        x0 = orc.randomize(c.dim, nb, 9, cx)
        X = block(A, x0)
        mom = cf.apply_filter(A, X, p, want_moments=True)
        xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=True)
        assert bits_equal(X.to_numpy(), xr)
        assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
        u, w, x = (orc.randomize(c.dim, nb, s, cx) for s in (1, 2, 3))
        U, W, Xb = block(A, u), block(A, w), block(A, x)
        d = cf.spmmvm_fused(A, U, W, Xb, p.alpha, p.beta, 0.83, dots=True)
        dref = orc.spmmvm_fused(c, u, w, x, p.alpha, p.beta, 0.83, want_dots=True)
        assert bits_equal(W.to_numpy(), w) and bits_equal(Xb.to_numpy(), x)
        assert np.allclose(d, dref, rtol=1e-12, atol=1e-12 * np.max(np.abs(dref)))
    finally:
        ctx.set_option("kernel", "tma")


@pytest.mark.parametrize("name,l,nb", [("ti", (24, 24, 17), 32), ("ti", (24, 24, 17), 7),
                                       ("graphene", (160, 128), 4), ("graphene", (160, 128), 1),
                                       ("graphene", (160, 128), 9)])
def test_large_operator_cta_shapes_bitexact(ctx, orc, name, l, nb):
    """Operators above 4 x SMs 64-row tiles take the large-problem CTA shapes
    (128-thread CTAs with 64-row tiles; 64-thread CTAs for rows of <= 4 units)
    -- fused W/X bit-exact with dots, apply_filter X bit-exact with moments."""
    A, c = make_case(ctx, orc, name, l)
    assert c.dim // 64 >= 4 * 148
    cx = name == "ti"
    u, w, x = (orc.randomize(c.dim, nb, s, cx) for s in (1, 2, 3))
    U, W, X = block(A, u), block(A, w), block(A, x)
    bounds = (-5.6, 5.6) if cx else (-3.2, 3.3)
    p = cf.make_filter((-0.2, 0.3), bounds, 6, "lanczos2")
    cf.apply_filter(A, block(A, x), p)  # creates the pre-scaled values the TMA path uses
    d = cf.spmmvm_fused(A, U, W, X, p.alpha, p.beta, 0.83, dots=True)
    dref = orc.spmmvm_fused(c, u, w, x, p.alpha, p.beta, 0.83, want_dots=True)
    assert bits_equal(W.to_numpy(), w) and bits_equal(X.to_numpy(), x)
    assert np.allclose(d, dref, rtol=1e-12, atol=1e-12 * np.max(np.abs(dref)))
    x0 = orc.randomize(c.dim, nb, 9, cx)
    Xf = block(A, x0)
    mom = cf.apply_filter(A, Xf, p, want_moments=True)
    xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=True)
    assert bits_equal(Xf.to_numpy(), xr)
    assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
