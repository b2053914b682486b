"""Measurement sweeps for the BASELINE.json configs other than the bench line.

    python tools/sweeps.py c5     graphene 2048^2, n_b in {1,4,8,16,32,64}: fused step vs the
                                  unfused spmmvm + block_axpy_scal + column_dots sequence
                                  (test_core_linalg.cpp:139-147)
    python tools/sweeps.py c1     graphene 64^2, n_b=40, N_p=500: apply_filter + full solve
    python tools/sweeps.py c4     TI 512x512x8 sub-lattice (one GPU's share of C4), n_b=64,
                                  200 fused steps + one Gram
Prints one JSON object per measurement (CUDA events on the library stream).
"""
import ctypes as C
import json
import math
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1510_04895_b200 as cf  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0


def model(dim, nnz, nb, cplx):
    n_nzr = nnz / dim
    f_a, f_m, s_d = (2, 6, 16) if cplx else (1, 1, 8)
    flops = (n_nzr * (f_a + f_m) + math.ceil(9 * f_a / 2) + math.ceil(11 * f_m / 2)) * dim * nb
    return flops, nnz * (s_d + 4) + 5 * dim * nb * s_d


def timed(ctx, fn, reps):
    fn()
    ctx.synchronize()
    ctx.record(0)
    for _ in range(reps):
        fn()
    ctx.record(1)
    return ctx.elapsed_ms(0, 1) / reps


def c5(ctx):
    A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(2048, 2048, disorder=1.0, seed=1))
    D, nnz = A.dim(), A.nnz()
    lib = cf.load()
    p = cf.make_filter((-0.15, 0.15), (-3.6, 3.6), 2, "lanczos2")  # builds alpha / 2alpha copies
    for nb in (1, 4, 8, 16, 32, 64):
        U, W, X = (cf.BlockVector(A, nb).randomize_device(s) for s in (1, 2, 3))
        Y = cf.BlockVector(A, nb)
        cf.apply_filter(A, X, p)
        flops, b = model(D, nnz, nb, False)
        state = {"u": U, "w": W}

        def fused():
            cf.spmmvm_fused(A, state["u"], state["w"], X, p.alpha, p.beta, 0.3)
            state["u"], state["w"] = state["w"], state["u"]

        d = np.empty(nb)

        def unfused():  # w_ref = spmmvm(2a,2b); w_ref -= w; x += c w_ref; dots(x, w_ref)
            lib.chebfd_spmmvm(A._h, state["u"]._h, Y._h, 2 * p.alpha, 2 * p.beta)
            lib.chebfd_block_axpy_scal(Y._h, state["w"]._h, state["w"]._h, 1.0, -1.0, 0.0)
            lib.chebfd_block_axpy_scal(X._h, Y._h, Y._h, 1.0, 0.3, 0.0)
            lib.chebfd_column_dots(X._h, Y._h, d.ctypes.data_as(C.c_void_p))

        def fused_dots():
            cf.spmmvm_fused(A, state["u"], state["w"], X, p.alpha, p.beta, 0.3, dots=True)

        reps = 20 if nb >= 16 else 40
        tf = timed(ctx, fused, reps)
        tfd = timed(ctx, fused_dots, reps)
        tu = timed(ctx, unfused, reps)
        print(json.dumps({"config": "C5 graphene 2048x2048 V=1.0", "n_b": nb, "D": D, "nnz": nnz,
                          "fused_ms": round(tf, 4), "fused_dots_ms": round(tfd, 4),
                          "unfused_ms": round(tu, 4),
                          "fused_gbs": round(b / tf / 1e6, 1),
                          "fused_frac": round(b / tf / 1e6 / PEAK, 4),
                          "fused_gflops": round(flops / tf / 1e6, 1),
                          "unfused_gbs_same_model": round(b / tu / 1e6, 1),
                          "speedup_fused_vs_unfused": round(tu / tfd, 2)}), flush=True)
        for blk in (U, W, X, Y):
            blk.close()


def c1(ctx):
    A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(64, 64, disorder=0.1, seed=1))
    D, nnz = A.dim(), A.nnz()
    b = cf.lanczos_bounds(A, 30, 1)
    p = cf.make_filter((-0.13, 0.13), (b.lo, b.hi), 500, "lanczos2")
    X = cf.BlockVector(A, 40).randomize(3)
    for graphs in (True, False):
        ctx.set_option("graphs", graphs)
        t = timed(ctx, lambda: cf.apply_filter(A, X, p), 10)
        flops, by = model(D, nnz, 40, False)
        print(json.dumps({"config": "C1 graphene 64x64 V=0.1, n_b=40, N_p=500", "cuda_graphs": graphs,
                          "apply_filter_ms": round(t, 4), "us_per_step": round(1e3 * t / 500, 3),
                          "gflops": round(flops * 500 / t / 1e6, 1)}), flush=True)
    ctx.set_option("graphs", True)
    t0 = time.perf_counter()
    rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(-0.13, 0.13), n_search=40, degree=500,
                                       seed=1))
    dt = time.perf_counter() - t0
    print(json.dumps({"config": "C1 full ChebFD solve", "converged": rep.converged,
                      "iterations": rep.iterations, "accepted": int(rep.ritz.accepted.sum()),
                      "n_target_estimate": rep.n_target_estimate, "wall_s": round(dt, 3),
                      "solver_seconds": round(rep.seconds, 3)}), flush=True)


def c4(ctx):
    spec = cf.LatticeSpec(512, 512, 8, disorder=0.5, seed=1)
    A = cf.SparseMatrix.topological_insulator(ctx, spec)
    D, nnz = A.dim(), A.nnz()
    nb = 64
    p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), 200, "lanczos2")
    X = cf.BlockVector(A, nb).randomize_device(5)
    t = timed(ctx, lambda: cf.apply_filter(A, X, p), 2)
    flops, b = model(D, nnz, nb, True)
    tg = timed(ctx, lambda: cf.gram(X, X), 3)
    print(json.dumps({"config": "C4 one-GPU share: TI 512x512x8 slab, n_b=64, 200 steps + Gram",
                      "D": D, "nnz": nnz, "apply_filter_ms": round(t, 2),
                      "ms_per_step": round(t / 200, 4), "gbs": round(200 * b / t / 1e6, 1),
                      "frac": round(200 * b / t / 1e6 / PEAK, 4),
                      "gflops": round(200 * flops / t / 1e6, 1), "gram_ms": round(tg, 3),
                      "gram_tflops": round(8 * D * nb * nb / tg / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    ctx = cf.Context(0)
    for what in sys.argv[1:] or ["c5", "c1", "c4"]:
        {"c5": c5, "c1": c1, "c4": c4}[what](ctx)
    ctx.close()
