"""The multi-rank device path on one GPU (virtual rank groups, vgroup.cu).

Every rank owns a z-plane (TI) / y-row (graphene) slab of the operator with halo rows;
each step runs capi.cu's launch_split (interior rows while the halo arrives, then the
boundary rows, cross-launch dot reduction) with the halo rows pulled from the
neighbours' blocks.  The gathered result must equal the single-rank oracle's
apply_filter (filter.hpp:73-116) / spmmvm_fused (kernels.hpp:74-118) bit for bit (row-
local arithmetic); moments, dots and Gram matrices (reduction order differs) within
the tolerances written below.  Also: the compact halo moves half a plane per side for
TI (orbitals {0,3} below, {1,2} above), and the band tile order keeps the bits.
"""
import numpy as np
import pytest

import paper_1510_04895_b200 as cf

pytestmark = pytest.mark.gpu


def bits_equal(a, b):
    a = np.ascontiguousarray(a)
    b = np.ascontiguousarray(b)
    return a.shape == b.shape and np.array_equal(a.view(np.uint64), b.view(np.uint64))


def split_rows(As):
    out, r0 = [], 0
    for A in As:
        out.append((r0, r0 + A.local_rows))
        r0 += A.local_rows
    return out


CASES = [("ti", (5, 4, 9), "periodic_xy_open_z"), ("ti", (4, 4, 8), "periodic_all"),
         ("ti", (3, 5, 6), "open_all"), ("graphene", (16, 12), "periodic_xy_open_z"),
         ("graphene", (12, 9), "periodic_all")]


@pytest.mark.parametrize("world", [2, 3])
@pytest.mark.parametrize("name,l,boundary", CASES)
@pytest.mark.parametrize("graphs", [True, False])
@pytest.mark.parametrize("compact", [True, False])
def test_vgroup_apply_filter_matches_single_rank(orc, world, name, l, boundary, graphs, compact):
    cx = name == "ti"
    spec = cf.LatticeSpec(*l, disorder=0.5, seed=3, boundary=boundary)
    csr = (orc.topological_insulator(*l, disorder=0.5, seed=3, boundary=boundary) if cx
           else orc.graphene(*l, disorder=0.5, seed=3, boundary=boundary))
    g = cf.VirtualGroup(world)
    try:
        g.set_option("graphs", graphs)
        g.set_option("compact_halo", compact)
        As = g.topological_insulator(spec) if cx else g.graphene(spec)
        rows = split_rows(As)
        assert rows[-1][1] == csr.dim
        nb = 6
        x0 = orc.randomize(csr.dim, nb, 9, cx)
        Xs = [cf.BlockVector(A, nb).upload(x0[a:b]) for A, (a, b) in zip(As, rows)]
        bounds = (-5.6, 5.6) if cx else (-3.4, 3.4)
        p = cf.make_filter((-0.3, 0.2), bounds, 23, "lanczos2")
        mom = g.apply_filter(As, Xs, p, want_moments=True)
        xr, mr = orc.apply_filter(csr, x0, p.combined, p.alpha, p.beta, want_moments=True)
        got = np.concatenate([X.to_numpy() for X in Xs])
        assert bits_equal(got, xr)
        assert np.max(np.abs(mom.m - mr)) <= 1e-12 * np.max(np.abs(mr[0]))
        # replay (graph cache hit) with new coefficients, no moments
        p2 = cf.make_filter((-0.1, 0.4), bounds, 23, "jackson")
        for X, (a, b) in zip(Xs, rows):
            X.upload(x0[a:b])
        g.apply_filter(As, Xs, p2)
        xr2, _ = orc.apply_filter(csr, x0, p2.combined, p2.alpha, p2.beta)
        assert bits_equal(np.concatenate([X.to_numpy() for X in Xs]), xr2)
        # fused step with Kahan dots, and the Gram, summed over ranks
        u, w, x = (orc.randomize(csr.dim, nb, s, cx) for s in (1, 2, 3))
        Us = [cf.BlockVector(A, nb).upload(u[a:b]) for A, (a, b) in zip(As, rows)]
        Ws = [cf.BlockVector(A, nb).upload(w[a:b]) for A, (a, b) in zip(As, rows)]
        Xf = [cf.BlockVector(A, nb).upload(x[a:b]) for A, (a, b) in zip(As, rows)]
        d = g.spmmvm_fused(As, Us, Ws, Xf, p.alpha, p.beta, 0.7, dots=True)
        dref = orc.spmmvm_fused(csr, u, w, x, p.alpha, p.beta, 0.7, want_dots=True)
        assert bits_equal(np.concatenate([W.to_numpy() for W in Ws]), w)
        assert bits_equal(np.concatenate([X.to_numpy() for X in Xf]), x)
        assert np.allclose(d, dref, rtol=1e-12, atol=1e-12 * np.max(np.abs(dref)))
        G = g.gram(Xf, Ws)
        Gref = orc.gram(x, w)
        assert np.max(np.abs(G - Gref)) <= 1e-13 * np.max(np.abs(Gref))
    finally:
        g.close()


@pytest.mark.parametrize("world", [2, 3])
def test_compact_halo_is_half_a_ti_plane(world):
    """TI rows read orbitals {0,3} of the plane below and {1,2} of the plane above
    (models.cpp:121-137): the compact halo holds 2 Lx Ly rows per side instead of the
    4 Lx Ly of a whole plane, and what a rank sends equals what its neighbour receives."""
    lx, ly, lz = 6, 5, 3 * world
    spec = cf.LatticeSpec(lx, ly, lz, disorder=0.5, seed=1, boundary="periodic_all")
    full = {}
    for compact in (True, False):
        g = cf.VirtualGroup(world)
        try:
            g.set_option("compact_halo", compact)
            As = g.topological_insulator(spec)
            h = [cf.VirtualGroup.halo_rows(A) for A in As]
            full[compact] = h
            for r in range(world):
                hi = (r + 1) % world
                assert h[r]["send_hi"] == h[hi]["halo_lo"]
                assert h[r]["send_lo"] == h[(r - 1) % world]["halo_hi"]
        finally:
            g.close()
    for r in range(world):
        # compact: exactly half a plane; contiguous: the span from the first to the last
        # referenced row of the plane (4 Lx Ly - 1 above: the top site's orbital 3 unread)
        assert full[True][r]["halo_lo"] == full[True][r]["halo_hi"] == 2 * lx * ly
        assert full[False][r]["halo_lo"] >= 4 * lx * ly - 3
        assert full[False][r]["halo_hi"] >= 4 * lx * ly - 3


@pytest.mark.parametrize("world", [1, 2, 3])
def test_band_order_keeps_the_bits(orc, world):
    """The band (2.5D) tile order of dot-free steps (CHEBFD_OPT_BAND_BYTES; forced here on
    a small lattice by a tiny slice budget: 4 x 32 lines of 16 rows, slices of 4 lines)
    changes only which CTA computes which rows: X bit-exact, every tiles_per_cta."""
    l = (4, 32, 6)
    spec = cf.LatticeSpec(*l, disorder=0.5, seed=2)
    csr = orc.topological_insulator(*l, disorder=0.5, seed=2)
    nb = 4
    x0 = orc.randomize(csr.dim, nb, 5, True)
    p = cf.make_filter((-0.3, 0.2), (-5.6, 5.6), 17, "lanczos2")
    xr, _ = orc.apply_filter(csr, x0, p.combined, p.alpha, p.beta)
    g = cf.VirtualGroup(world)
    try:
        g.set_option("band_bytes", 64 * nb * 16)  # 64-row slices = 4 lattice lines
        for tpc in (1, 2, 3):
            g.set_option("tiles_per_cta", tpc)
            As = g.topological_insulator(spec)
            rows = split_rows(As)
            Xs = [cf.BlockVector(A, nb).upload(x0[a:b]) for A, (a, b) in zip(As, rows)]
            before = sum(c.band_launches for c in g.ranks)
            g.apply_filter(As, Xs, p)
            assert sum(c.band_launches for c in g.ranks) > before  # the band order ran
            assert bits_equal(np.concatenate([X.to_numpy() for X in Xs]), xr), tpc
            for X in Xs:
                X.close()
            for A in As:
                A.close()
    finally:
        g.close()


def test_nccl_bootstrap_and_one_rank_distributed_context():
    """The process-per-GPU entry (chebfd_ctx_create_dist, what `bench.py --gpus N` calls):
    the library's own NCCL hands out a unique id on this box, and a one-rank distributed
    context filters to the same bits as a plain context (no communicator, no halos)."""
    uid = cf.Context.nccl_unique_id()
    assert len(uid) == 128 and any(uid)
    assert cf.Context.nccl_unique_id() != uid
    spec = cf.LatticeSpec(5, 4, 6, disorder=0.5, seed=3)
    p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), 17, "lanczos2")
    out = []
    for make in (lambda: cf.Context(0), lambda: cf.Context.distributed(0, 0, 1, uid)):
        ctx = make()
        try:
            A = cf.SparseMatrix.topological_insulator(ctx, spec)
            assert A.local_rows == A.dim()
            X = cf.BlockVector(A, 8).randomize(5)
            mom = cf.apply_filter(A, X, p, want_moments=True)
            out.append((X.to_numpy(), np.asarray(mom.m)))
        finally:
            ctx.close()
    assert bits_equal(out[0][0], out[1][0])
    assert bits_equal(out[0][1], out[1][1])
    with pytest.raises(cf.ChebfdError):
        cf.Context.distributed(0, 2, 2, uid)  # rank outside the group
