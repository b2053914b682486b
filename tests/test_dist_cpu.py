"""CPU, multi-process (gloo): the distributed filter's host logic.

Each rank plans its plane partition with the library
(chebfd_plan_partition / chebfd_plan_sends / chebfd_plan_map_column --
the same code the NCCL device path runs), all-gathers the halo descriptors
over gloo, exchanges halos every Chebyshev step in the device path's message
order (send A to hi, send B to lo, recv A from lo, recv B from hi), applies
the step to its extended local rows in numpy, and all-reduces the moments.
The gathered result must equal the single-process oracle apply_filter.
"""
import os
import socket

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _local_matrix(cf, spec, model, plan):
    import scipy.sparse as sp
    r0, r1 = plan.row_begin, plan.row_begin + plan.local_rows
    gen = cf.csr_topological_insulator if model == "ti" else cf.csr_graphene
    offs, cols, vals = gen(spec, r0, r1)
    ext = np.array([cf.plan_map_column(plan, g) for g in cols], dtype=np.int64)
    assert np.all(ext >= 0), "column outside own rows + halos"
    n_ext = plan.halo_lo + plan.local_rows + plan.halo_hi
    return sp.csr_matrix((vals, ext, offs), shape=(plan.local_rows, n_ext))


def _exchange(dist, plan, U):
    """Fill U's halo rows (U has ext rows) -- device-path message order."""
    lo, n, hi = plan.halo_lo, plan.local_rows, plan.halo_hi
    own = U[lo:lo + n]
    reqs, keep = [], []
    if plan.hi_rank >= 0 and plan.send_hi_n > 0:  # A: my last rows -> hi's lo halo
        keep.append(_t(own[plan.send_hi_begin:plan.send_hi_begin + plan.send_hi_n]))
        reqs.append(dist.isend(keep[-1], plan.hi_rank))
    if plan.lo_rank >= 0 and plan.send_lo_n > 0:  # B: my first rows -> lo's hi halo
        keep.append(_t(own[plan.send_lo_begin:plan.send_lo_begin + plan.send_lo_n]))
        reqs.append(dist.isend(keep[-1], plan.lo_rank))
    bufs = []
    if plan.lo_rank >= 0 and lo > 0:
        b = _t(np.zeros_like(U[:lo]))
        reqs.append(dist.irecv(b, plan.lo_rank))
        bufs.append((slice(0, lo), b))
    if plan.hi_rank >= 0 and hi > 0:
        b = _t(np.zeros_like(U[lo + n:]))
        reqs.append(dist.irecv(b, plan.hi_rank))
        bufs.append((slice(lo + n, lo + n + hi), b))
    for r in reqs:
        r.wait()
    for sl, b in bufs:
        U[sl] = b.numpy().view(U.dtype).reshape(U[sl].shape)


def _t(a):
    import torch
    a = np.ascontiguousarray(a)
    return torch.from_numpy(a.view(np.float64).reshape(-1).copy())


def _worker(rank, world, port, model, lattice, boundary, nb, degree, q):
    try:
        os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
        import sys
        sys.path.insert(0, ROOT)
        import torch.distributed as dist
        import paper_1510_04895_b200 as cf
        import oracle
        dist.init_process_group("gloo", rank=rank, world_size=world)
        spec = cf.LatticeSpec(*lattice, disorder=0.5, boundary=boundary, seed=3)
        plan = cf.plan_partition(spec, model, rank, world)
        mine = np.array(cf.plan_all4(plan), dtype=np.int64)
        allv = [None] * world
        dist.all_gather_object(allv, mine.tolist())
        cf.plan_sends(plan, rank, [v for a in allv for v in a])
        A = _local_matrix(cf, spec, model, plan)
        orc = oracle.Oracle()
        cplx = model == "ti"
        dim = 4 * int(np.prod(lattice)) if cplx else 2 * lattice[0] * lattice[1]
        xg = orc.randomize(dim, nb, 9, cplx)
        r0, n, lo = plan.row_begin, plan.local_rows, plan.halo_lo
        x = xg[r0:r0 + n].copy()
        bounds = (-5.6, 5.6) if cplx else (-3.6, 3.6)
        p = cf.make_filter((-0.3, 0.2), bounds, degree, "lanczos2")
        a, b, cmb = p.alpha, p.beta, p.combined
        ext = lambda own: np.concatenate([np.zeros((lo, nb), own.dtype), own,  # noqa: E731
                                          np.zeros((plan.halo_hi, nb), own.dtype)])
        mom = np.zeros((degree + 1, nb))
        dot = lambda u, v: np.real(np.sum(np.conj(u) * v, axis=0))  # noqa: E731
        X = ext(x)
        _exchange(dist, plan, X)
        u = a * (A @ X) + b * x                       # filter.hpp:92
        mom[0], mom[1] = dot(x, x), dot(x, u)
        U = ext(u)
        _exchange(dist, plan, U)
        w = 2 * a * (A @ U) + 2 * b * u - x           # filter.hpp:93-94
        mom[2] = dot(x, w)
        xf = cmb[0] * x + cmb[1] * u + cmb[2] * w     # filter.hpp:103
        uo, wo = u, w
        for k in range(3, degree + 1):                # filter.hpp:107-114
            uo, wo = wo, uo
            U = ext(uo)
            _exchange(dist, plan, U)
            wo = 2 * a * (A @ U) + 2 * b * uo - wo
            xf = xf + cmb[k] * wo
            mom[k] = dot(x, wo)
        import torch
        tm = torch.from_numpy(mom)
        dist.all_reduce(tm)
        parts = [None] * world
        dist.all_gather_object(parts, xf)
        if rank == 0:
            full = np.concatenate(parts)
            c = orc.graphene(*lattice, disorder=0.5, boundary=boundary, seed=3) if not cplx else \
                orc.topological_insulator(*lattice, disorder=0.5, boundary=boundary, seed=3)
            yref, mref = orc.apply_filter(c, xg, cmb, a, b, want_moments=True)
            q.put(("ok", float(np.max(np.abs(full - yref)) / np.max(np.abs(yref))),
                   float(np.max(np.abs(tm.numpy() - mref)) / np.max(np.abs(mref[0]))),
                   dict(halo_lo=plan.halo_lo, halo_hi=plan.halo_hi)))
        dist.barrier()
        dist.destroy_process_group()
    except Exception as e:  # pragma: no cover - surfaced by the parent
        import traceback
        q.put(("err", repr(e) + traceback.format_exc(), 0, {}))


@pytest.mark.parametrize("model,lattice,boundary,world", [
    ("ti", (4, 4, 8), "periodic_xy_open_z", 2),
    ("ti", (4, 4, 8), "periodic_all", 2),   # 2-rank ring: lo and hi neighbour coincide
    ("ti", (3, 4, 9), "periodic_all", 3),
    ("graphene", (6, 8), "periodic_xy_open_z", 2),
])
def test_distributed_filter_matches_oracle(model, lattice, boundary, world):
    import multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, model, lattice, boundary, 3, 25, q))
             for r in range(world)]
    for p in procs:
        p.start()
    res = q.get(timeout=240)
    for p in procs:
        p.join(timeout=60)
    assert res[0] == "ok", res[1]
    _, ex, em, info = res
    assert ex <= 1e-12, ex   # numpy sums vs oracle's sequential sums
    assert em <= 1e-12, em
