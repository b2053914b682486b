"""The row-group step kernel (step_group.cuh; grouped matrix form, group.cu).

Rows 4g .. 4g+3 share one merged list of gathered columns; every row still meets its
entries in CSR order, so W / X must equal the oracle (kernels.hpp:46-145,
filter.hpp:73-116) bit for bit exactly like the SELL kernels.  Option "grouped" = 2
forces the kernel onto small operators (the default takes it from 4 x SMs 64-row tiles);
Context.group_launches proves it ran.  Covered: TI / graphene / irregular from_csr
operators (row counts not multiples of 4 or 64, rows of 0..13 entries, unsorted rows),
every step kind through apply_filter (with / without moments, direct and doubling, every
delayed-X tail), fused Kahan dots, block widths below / at / above a warp, and the
multi-rank split launches of a virtual group.
"""
import numpy as np
import pytest

import paper_1510_04895_b200 as cf

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


@pytest.fixture()
def gctx(ctx):
    ctx.set_option("grouped", 2)
    yield ctx
    ctx.set_option("grouped", 1)


def ti(ctx, orc, l, boundary="periodic_xy_open_z"):
    A = cf.SparseMatrix.topological_insulator(
        ctx, cf.LatticeSpec(*l, disorder=0.5, seed=1, boundary=boundary))
    return A, orc.topological_insulator(*l, disorder=0.5, seed=1, boundary=boundary)


def graphene(ctx, orc, l, boundary="periodic_xy_open_z"):
    A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(*l, disorder=0.4, seed=2, boundary=boundary))
    return A, orc.graphene(*l, disorder=0.4, seed=2, boundary=boundary)


def block(A, host):
    return cf.BlockVector(A, host.shape[1]).upload(host)


CASES = [("ti", (4, 4, 4), 4), ("ti", (5, 3, 4), 32), ("ti", (3, 5, 7), 64), ("ti", (6, 6, 5), 9),
         ("ti", (4, 4, 3), 96), ("graphene", (16, 16), 8), ("graphene", (13, 7), 16),
         ("graphene", (9, 11), 5), ("graphene", (16, 16), 64)]


def make(ctx, orc, name, l):
    return ti(ctx, orc, l) if name == "ti" else graphene(ctx, orc, l)


@pytest.mark.parametrize("name,l,nb", CASES)
def test_group_spmmvm_and_fused_bitexact(gctx, orc, name, l, nb):
    A, c = make(gctx, orc, name, l)
    cx = name == "ti"
    before = gctx.group_launches
    x = orc.randomize(c.dim, nb, 11, cx)
    y = cf.spmmvm(A, block(A, x), 0.37, -0.21).to_numpy()
    assert bits_equal(y, orc.spmmvm(c, x, 0.37, -0.21))
    u, w, xx = (orc.randomize(c.dim, nb, s, cx) for s in (1, 2, 3))
    U, W, X = block(A, u), block(A, w), block(A, xx)
    d = cf.spmmvm_fused(A, U, W, X, 0.37, -0.21, 0.83, dots=True)
    dref = orc.spmmvm_fused(c, u, w, xx, 0.37, -0.21, 0.83, want_dots=True)
    assert bits_equal(W.to_numpy(), w)
    assert bits_equal(X.to_numpy(), xx)
    assert np.allclose(d, dref, rtol=1e-12, atol=1e-12 * np.max(np.abs(dref)))
    u, w = (orc.randomize(c.dim, nb, s, cx) for s in (4, 5))
    U, W = block(A, u), block(A, w)
    cf.recurrence_step(A, U, W, 0.6, 0.1)
    orc.recurrence_step(c, u, w, 0.6, 0.1)
    assert bits_equal(W.to_numpy(), w)
    assert gctx.group_launches >= before + 3


@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("moments", ["doubling", "direct"])
@pytest.mark.parametrize("name,l,nb,deg", [
    ("ti", (4, 4, 4), 32, 40), ("ti", (5, 4, 3), 8, 7), ("ti", (3, 3, 5), 64, 11),
    ("graphene", (16, 16), 40, 21), ("graphene", (13, 7), 4, 6)])
def test_group_apply_filter_bitexact_with_moments(gctx, orc, name, l, nb, deg, graphs, moments):
    gctx.set_option("graphs", graphs)
    gctx.set_option("moments", moments)
    try:
        A, c = make(gctx, orc, name, l)
        bounds = (-3.4, 3.4) if name == "graphene" else (-5.6, 5.6)
        p = cf.make_filter((-0.2, 0.3), bounds, deg, "lanczos2")
        x0 = orc.randomize(c.dim, nb, 9, name == "ti")
        before = gctx.group_launches
        for want in (True, False):
            X = block(A, x0)
            mom = cf.apply_filter(A, X, p, want_moments=want)
            xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=want)
            assert bits_equal(X.to_numpy(), xr)
            if want:
                assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
        if not graphs:
            assert gctx.group_launches >= before + 2 * deg
    finally:
        gctx.set_option("graphs", True)
        gctx.set_option("moments", "doubling")


@pytest.mark.parametrize("deg", [2, 3, 4, 5, 6, 7, 8])
@pytest.mark.parametrize("group", [1, 2, 3])
def test_group_delayed_x_tails(gctx, orc, deg, group):
    gctx.set_option("delayed_x", group)
    try:
        A, c = ti(gctx, orc, (4, 3, 4))
        p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), deg, "jackson")
        x0 = orc.randomize(c.dim, 16, 5, True)
        X = block(A, x0)
        cf.apply_filter(A, X, p)
        xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta)
        assert bits_equal(X.to_numpy(), xr)
    finally:
        gctx.set_option("delayed_x", 3)


def random_csr(rng, dim, complex_, sort_rows=True, max_len=13):
    offs = [0]
    cols, vals = [], []
    for r in range(dim):
        n = int(rng.integers(0, max_len + 1))
        cs = rng.choice(dim, size=min(n, dim), replace=False)
        # neighbouring rows share columns, as lattice rows do
        if r % 4 and len(cols) and n:
            prev = np.array(cols[offs[-2]:offs[-1]], dtype=np.int64)
            if len(prev):
                k = min(len(prev), len(cs) // 2)
                cs[:k] = rng.choice(prev, size=k, replace=False)
                cs = np.unique(cs)
        cs = np.sort(cs) if sort_rows else rng.permutation(cs)
        cols.extend(int(v) for v in cs)
        for _ in cs:
            vals.append(complex(rng.normal(), rng.normal()) if complex_ else float(rng.normal()))
        offs.append(len(cols))
    return (np.array(offs, dtype=np.int64), np.array(cols, dtype=np.int64),
            np.array(vals, dtype=np.complex128 if complex_ else np.float64))


@pytest.mark.parametrize("dim,complex_,nb,sort_rows", [
    (257, True, 8, True), (130, False, 6, True), (203, True, 32, False), (64, False, 5, True),
    (1031, True, 16, True)])
def test_group_irregular_from_csr(gctx, orc, dim, complex_, nb, sort_rows):
    """Row counts that are no multiple of 4 / 64, empty rows, rows of up to 13 entries,
    unsorted rows (the merge falls back to unshared entries where orders disagree)."""
    import oracle
    rng = np.random.default_rng(dim)
    offs, cols, vals = random_csr(rng, dim, complex_, sort_rows)
    A = cf.SparseMatrix.from_csr(gctx, dim, offs, cols, vals)
    c = oracle.CSR(offs, cols, vals)
    x = orc.randomize(dim, nb, 3, complex_)
    before = gctx.group_launches
    y = cf.spmmvm(A, block(A, x), 0.9, 0.3).to_numpy()
    assert gctx.group_launches > before
    assert bits_equal(y, orc.spmmvm(c, x, 0.9, 0.3))
    u, w, xx = (orc.randomize(dim, nb, s, complex_) for s in (1, 2, 3))
    U, W, X = block(A, u), block(A, w), block(A, xx)
    cf.spmmvm_fused(A, U, W, X, 0.37, -0.21, 0.83)
    orc.spmmvm_fused(c, u, w, xx, 0.37, -0.21, 0.83)
    assert bits_equal(W.to_numpy(), w)
    assert bits_equal(X.to_numpy(), xx)


def test_group_off_equals_on(ctx, orc):
    """The SELL kernels and the row-group kernel give the same bits, dots included to 1e-13."""
    A, c = ti(ctx, orc, (6, 6, 6))
    p = cf.make_filter((-0.2, 0.3), (-5.6, 5.6), 31, "lanczos2")
    x0 = orc.randomize(c.dim, 32, 9, True)
    out = {}
    for g in (0, 2):
        ctx.set_option("grouped", g)
        X = block(A, x0)
        before = ctx.group_launches
        mom = cf.apply_filter(A, X, p, want_moments=True)
        out[g] = (X.to_numpy(), mom.m.copy(), ctx.group_launches - before)
    ctx.set_option("grouped", 1)
    assert out[0][2] == 0 and out[2][2] > 0
    assert bits_equal(out[0][0], out[2][0])
    assert np.max(np.abs(out[0][1] - out[2][1])) <= 1e-13 * np.max(np.abs(out[0][1][0]))


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,l,boundary", [
    ("ti", (4, 4, 8), "periodic_all"), ("ti", (4, 4, 9), "periodic_xy_open_z"),
    ("graphene", (16, 12), "periodic_all")])
def test_group_virtual_ranks(orc, world, name, l, boundary):
    """Split launches (interior + boundary rows) and halo-extended column indices; a ring's
    wrapped halo puts extended indices out of global column order."""
    cx = name == "ti"
    spec = cf.LatticeSpec(*l, disorder=0.5, seed=3, boundary=boundary)
    csr = (orc.topological_insulator(*l, disorder=0.5, seed=3, boundary=boundary) if cx
           else orc.graphene(*l, disorder=0.5, seed=3, boundary=boundary))
    g = cf.VirtualGroup(world)
    try:
        g.set_option("grouped", 2)
        As = g.topological_insulator(spec) if cx else g.graphene(spec)
        rows, r0 = [], 0
        for A in As:
            rows.append((r0, r0 + A.local_rows))
            r0 += A.local_rows
        nb = 8
        x0 = orc.randomize(csr.dim, nb, 9, cx)
        Xs = [cf.BlockVector(A, nb).upload(x0[a:b]) for A, (a, b) in zip(As, rows)]
        bounds = (-5.6, 5.6) if cx else (-3.4, 3.4)
        p = cf.make_filter((-0.3, 0.2), bounds, 17, "lanczos2")
        mom = g.apply_filter(As, Xs, p, want_moments=True)
        xr, mr = orc.apply_filter(csr, x0, p.combined, p.alpha, p.beta, want_moments=True)
        got = np.concatenate([X.to_numpy() for X in Xs])
        assert bits_equal(got, xr)
        assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
    finally:
        g.close()


@pytest.mark.parametrize("lines", [1, 2, 4])
def test_group_default_takes_the_band_launches(orc, lines):
    """Default mode ("grouped" = 1): dot-free steps that run in the band tile order take the
    row-group kernel (forced on a small lattice by a tiny slice budget, as
    test_band_order_keeps_the_bits does), everything else the SELL kernels; tiles of 1, 2
    or 4 lattice lines give the same bits.  Static TI patterns (interior sites of the three
    slab regions) and the generic path (x / y wrap sites) both run here."""
    l = (8, 32, 6)
    nb = 8
    g = cf.VirtualGroup(1)
    try:
        ctx1 = g.ranks[0]
        ctx1.set_option("group_lines", lines)
        # slices of 2 lattice lines (64 rows), 4 for 4-line tiles
        ctx1.set_option("band_bytes", 32 * max(lines, 2) * nb * 16)
        spec = cf.LatticeSpec(*l, disorder=0.5, seed=2)
        csr = orc.topological_insulator(*l, disorder=0.5, seed=2)
        A = g.topological_insulator(spec)[0]
        x0 = orc.randomize(csr.dim, nb, 5, True)
        p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 17, "lanczos2")
        xr, _ = orc.apply_filter(csr, x0, p.combined, p.alpha, p.beta)
        X = cf.BlockVector(A, nb).upload(x0)
        b0, g0 = ctx1.band_launches, ctx1.group_launches
        g.apply_filter([A], [X], p)
        assert ctx1.band_launches > b0 and ctx1.group_launches - g0 == ctx1.band_launches - b0
        assert bits_equal(X.to_numpy(), xr)
    finally:
        g.close()


def test_group_sparse_block_with_exact_zeros(gctx, orc):
    """Unit-vector columns: most products are exact zeros.  The two-multiply products of the
    static TI patterns drop the 0 * u terms of purely real / imaginary entries, which only
    matters for the sign of an exact zero when a whole product is zero; sums start from +0 and
    round to nearest, so the filtered block still equals the oracle's bits here."""
    l = (6, 6, 5)
    A, c = ti(gctx, orc, l)
    nb = 8
    x0 = np.zeros((c.dim, nb), dtype=np.complex128)
    for k in range(nb):
        x0[(37 * k + 5) % c.dim, k] = 1.0 if k % 2 == 0 else -1.0j
    p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 9, "lanczos2")
    X = block(A, x0)
    before = gctx.group_launches
    cf.apply_filter(A, X, p)
    assert gctx.group_launches > before
    xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta)
    assert bits_equal(X.to_numpy(), xr)
