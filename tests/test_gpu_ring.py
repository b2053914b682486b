"""The site-ring step kernel (step_ring.cuh): producer warp + TMA-fed shared-memory rings.

A strip of four lattice lines marches along x; every gathered operand is read from shared
memory (x / y neighbours from neighbouring ring slots, z neighbours and matrix values from
the column's stage).  Each row still meets its entries in CSR order with the reference's
roundings, so apply_filter (filter.hpp:73-116) and spmmvm_fused / recurrence_step
(kernels.hpp:74-145) must equal the oracle bit for bit.  Option "ring" = 2 forces the kernel
onto small lattices; Context.ring_launches proves it ran.  Covered: the three slab patterns
(bottom / interior / top plane), generic sites (x / y wrap, open edges), periodic z, x
segments with aprons, shallow rings, 32- and 64-unit slabs, multi-slab widths, virtual rank
groups (halo rows behind the z -+ 1 indices, compact and full).
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
def rctx(ctx):
    ctx.set_option("ring", 2)
    yield ctx
    for k in ("ring_segx", "ring_no", "ring_nz", "ring_rows", "ring_unit"):
        ctx.set_option(k, 0)
    ctx.set_option("ring_order", 3)
    ctx.set_option("ring", 1)
    ctx.set_option("ring_consts", 1)
    ctx.set_option("ring_tmap", 1)
    ctx.set_option("ring_dots", 1)
    ctx.set_option("slab_units", 0)
    ctx.set_option("delayed_x", 3)


def ti(ctx, orc, l, boundary="periodic_xy_open_z"):
    A = cf.SparseMatrix.topological_insulator(
        ctx, cf.LatticeSpec(*l, disorder=0.5, seed=1, boundary=boundary))
    return A, orc.topological_insulator(*l, disorder=0.5, seed=1, boundary=boundary)


def block(A, host):
    return cf.BlockVector(A, host.shape[1]).upload(host)


@pytest.mark.parametrize("l,nb,boundary", [
    ((8, 8, 5), 64, "periodic_xy_open_z"),
    ((8, 8, 5), 32, "periodic_xy_open_z"),
    ((7, 4, 3), 64, "periodic_xy_open_z"),
    ((8, 12, 4), 32, "periodic_all"),
    ((6, 8, 4), 64, "open_all"),
    ((8, 8, 3), 96, "periodic_xy_open_z"),    # three 32-unit slabs (row copies, not site copies)
    ((8, 4, 3), 128, "periodic_xy_open_z"),   # one 128-unit slab on two-line strips
])
@pytest.mark.parametrize("tmap", [1, 2, 0])
def test_ring_filter_bitexact(rctx, orc, l, nb, boundary, tmap):
    """tmap: tensor-map TMA box copies (UTMALDG) for column slabs only (default), always, or
    never (1D bulk copies, UBLKCP: per row where a slab is narrower than the row)."""
    rctx.set_option("ring_tmap", tmap)
    A, c = ti(rctx, orc, l, boundary)
    x0 = orc.randomize(c.dim, nb, 5, True)
    p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 17, "lanczos2")
    xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta)
    X = block(A, x0)
    before = rctx.ring_launches
    cf.apply_filter(A, X, p)
    assert rctx.ring_launches > before
    assert bits_equal(X.to_numpy(), xr)


@pytest.mark.parametrize("nb,slab,consts,boundary", [
    (256, 0, 1, "periodic_xy_open_z"),    # two 128-unit slabs on two-line strips (the default from 128 columns)
    (128, 128, 1, "periodic_xy_open_z"),  # one whole-row 128-unit slab (1D bulk copies)
    (384, 128, 0, "periodic_all"),        # three 128-unit slabs, values from memory
    (256, 64, 1, "open_all"),             # four 64-unit slabs on four-line strips
])
def test_ring_wide_blocks(rctx, orc, nb, slab, consts, boundary):
    """Blocks wider than a slab: 128-unit slabs run strips of two lattice lines (tensor-map
    box copies of 4 / 2 / 1 rows x 2 KB), 64-unit slabs strips of four."""
    rctx.set_option("slab_units", slab)
    rctx.set_option("ring_consts", consts)
    A, c = ti(rctx, orc, (8, 8, 3), boundary)
    x0 = orc.randomize(c.dim, nb, 4, True)
    p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 9, "lanczos2")
    xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta)
    X = block(A, x0)
    before = rctx.ring_launches
    cf.apply_filter(A, X, p)
    assert rctx.ring_launches > before
    assert bits_equal(X.to_numpy(), xr)


@pytest.mark.parametrize("segx,no,nz", [(3, 4, 2), (1, 5, 3), (5, 6, 3), (64, 4, 2)])
def test_ring_segments_and_depths(rctx, orc, segx, no, nz):
    """x segments shorter than a line (apron columns on both sides, ragged last segment) and
    the shallowest / deepest rings give the same bits."""
    l, nb = (8, 8, 4), 64
    rctx.set_option("ring_segx", segx)
    rctx.set_option("ring_no", no)
    rctx.set_option("ring_nz", nz)
    A, c = ti(rctx, orc, l)
    x0 = orc.randomize(c.dim, nb, 6, True)
    p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 11, "jackson")
    xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta)
    X = block(A, x0)
    before = rctx.ring_launches
    cf.apply_filter(A, X, p)
    assert rctx.ring_launches > before
    assert bits_equal(X.to_numpy(), xr)


@pytest.mark.parametrize("order,unit", [(1, 0), (1, 4), (1, 9), (0, 0), (2, 0)])
def test_ring_cta_order_x_segments_slowest(rctx, orc, order, unit):
    """CTA order 1: (x segment, band of strips, plane, strip) with bands of `unit` / planes
    strips; order 2: (x segment, strip, plane) -- only which CTA computes which rows changes."""
    l, nb = (8, 16, 3), 64
    rctx.set_option("ring_order", order)
    rctx.set_option("ring_unit", unit)
    rctx.set_option("ring_segx", 3)
    A, c = ti(rctx, orc, l)
    x0 = orc.randomize(c.dim, nb, 9, True)
    p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 10, "lanczos2")
    xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta)
    X = block(A, x0)
    before = rctx.ring_launches
    cf.apply_filter(A, X, p)
    assert rctx.ring_launches > before
    assert bits_equal(X.to_numpy(), xr)


@pytest.mark.parametrize("consts", [1, 0])
@pytest.mark.parametrize("rows", [4, 2, 1])
@pytest.mark.parametrize("l,nb,boundary", [((8, 8, 4), 64, "periodic_xy_open_z"),
                                           ((8, 8, 4), 32, "periodic_all"),
                                           ((6, 4, 3), 32, "open_all")])
def test_ring_rows_per_thread(rctx, orc, rows, l, nb, boundary, consts):
    """4, 2 or 1 rows of a site per consumer thread (1, 2 or 4 consumer groups sharing the
    staged operands; 64-unit slabs run at most 2 groups): static and generic sites.  With
    and without the hopping values as kernel-parameter constants (the builder found every
    static site of a pattern to hold the same off-diagonal values)."""
    rctx.set_option("ring_rows", rows)
    rctx.set_option("ring_consts", consts)
    A, c = ti(rctx, orc, l, boundary)
    x0 = orc.randomize(c.dim, nb, 8, True)
    p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 13, "lanczos2")
    xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta)
    X = block(A, x0)
    before = rctx.ring_launches
    cf.apply_filter(A, X, p)
    assert rctx.ring_launches > before
    assert bits_equal(X.to_numpy(), xr)


@pytest.mark.parametrize("delayed", [3, 2])
@pytest.mark.parametrize("l,nb,boundary,segx", [
    ((8, 8, 5), 64, "periodic_xy_open_z", 0),
    ((8, 12, 4), 32, "periodic_all", 3),        # two CTAs per SM, x segments with aprons
    ((6, 8, 3), 64, "open_all", 4),             # generic sites on every edge
    ((8, 4, 3), 256, "periodic_xy_open_z", 0),  # two 128-unit slabs: one reduction per slab
    ((8, 8, 3), 128, "periodic_xy_open_z", 5),
])
def test_ring_moment_steps(rctx, orc, l, nb, boundary, segx, delayed):
    """V_n-only steps that carry the doubling moment sums (DMODE 5 / 6 of a triple, 4 / 6 of a
    pair) on the site-ring kernel (CHEBFD_OPT_RING_DOTS): X bit-exact, the MomentTable
    (filter.hpp:61-68, 86-113) within 1e-12 of the oracle's direct sums, bitwise equal between
    two runs (per-CTA partials reduced in CTA index order), and more ring launches than with
    the option off."""
    rctx.set_option("ring_segx", segx)
    rctx.set_option("delayed_x", delayed)
    A, c = ti(rctx, orc, l, boundary)
    x0 = orc.randomize(c.dim, nb, 21, True)
    for deg in (12, 31):
        p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), deg, "jackson")
        xr, mr = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta, want_moments=True)
        runs = []
        for dots in (0, 1, 1):
            rctx.set_option("ring_dots", dots)
            X = block(A, x0)
            before = rctx.ring_launches
            mom = cf.apply_filter(A, X, p, want_moments=True)
            runs.append((rctx.ring_launches - before, mom.m.copy()))
            assert bits_equal(X.to_numpy(), xr)
            assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0])), (deg, dots)
        assert runs[1][0] > runs[0][0], "moment steps did not run the ring kernel"
        assert bits_equal(runs[1][1], runs[2][1])


def test_ring_kpm_dos(rctx, orc):
    """kpm_dos (spectral.cpp:156-205) with its doubling steps (DMODE 4) on the ring kernel
    agrees with the row-group / SELL kernels' moments to rounding."""
    A, c = ti(rctx, orc, (8, 8, 4))
    mus = []
    for dots in (0, 1):
        rctx.set_option("ring_dots", dots)
        before = rctx.ring_launches
        mus.append((cf.kpm_dos(A, (-5.6, 5.6), 64, 32, seed=3).moments.copy(), rctx.ring_launches - before))
    assert mus[1][1] > mus[0][1]
    assert np.max(np.abs(mus[1][0] - mus[0][0])) <= 1e-12 * abs(mus[0][0][0])


@pytest.mark.parametrize("delayed", [0, 2, 3])
def test_ring_step_kinds(rctx, orc, delayed):
    """Every dot-free kind of the fused loop: kStepFused (delayed_x off), kStepRecur +
    kStepFusedX2 / X3, and the public single steps."""
    l, nb = (8, 8, 4), 32
    A, c = ti(rctx, orc, l)
    rctx.set_option("delayed_x", delayed)
    x0 = orc.randomize(c.dim, nb, 7, True)
    for deg in (9, 10, 11):
        p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), deg, "lanczos2")
        xr, _ = orc.apply_filter(c, x0, p.combined, p.alpha, p.beta)
        X = block(A, x0)
        before = rctx.ring_launches
        cf.apply_filter(A, X, p)
        assert rctx.ring_launches > before
        assert bits_equal(X.to_numpy(), xr), deg
    u, w, xx = (orc.randomize(c.dim, nb, s, True) for s in (1, 2, 3))
    U, W, X = block(A, u), block(A, w), block(A, xx)
    before = rctx.ring_launches
    cf.spmmvm_fused(A, U, W, X, 0.37, -0.21, 0.83, dots=False)
    orc.spmmvm_fused(c, u, w, xx, 0.37, -0.21, 0.83, want_dots=False)
    assert rctx.ring_launches > before
    assert bits_equal(W.to_numpy(), w)
    assert bits_equal(X.to_numpy(), xx)
    u, w = (orc.randomize(c.dim, nb, s, True) for s in (4, 5))
    U, W = block(A, u), block(A, w)
    cf.recurrence_step(A, U, W, 0.6, 0.1)
    orc.recurrence_step(c, u, w, 0.6, 0.1)
    assert bits_equal(W.to_numpy(), w)


@pytest.mark.parametrize("world,compact", [(2, 1), (3, 1), (2, 0)])
def test_ring_virtual_ranks(orc, world, compact):
    """Rank partitions by z-planes: the z -+ 1 indices of a rank's outer planes point into its
    halo regions (compact halos renumber them); interior / boundary launches of whole
    planes."""
    l, nb = (8, 8, 6), 64
    spec = cf.LatticeSpec(*l, disorder=0.5, seed=2)
    csr = orc.topological_insulator(*l, disorder=0.5, seed=2)
    x0 = orc.randomize(csr.dim, nb, 5, True)
    p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 14, "lanczos2")
    xr, _ = orc.apply_filter(csr, x0, p.combined, p.alpha, p.beta)
    g = cf.VirtualGroup(world)
    try:
        g.set_option("compact_halo", compact)
        g.set_option("ring", 2)
        As = g.topological_insulator(spec)
        rows, a = [], 0
        for A in As:
            rows.append((a, a + A.local_rows))
            a += A.local_rows
        Xs = [cf.BlockVector(A, nb).upload(x0[a:b]) for A, (a, b) in zip(As, rows)]
        before = sum(c.ring_launches for c in g.ranks)
        g.apply_filter(As, Xs, p)
        assert sum(c.ring_launches for c in g.ranks) > before
        assert bits_equal(np.concatenate([X.to_numpy() for X in Xs]), xr)
    finally:
        g.close()
