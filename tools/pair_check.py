"""Pair (two-steps-per-launch) kernel: bit-exactness against single steps and
a timing sweep of its knobs on the C2 workload.

    python tools/pair_check.py [--sweep] [--np 100]
Prints one JSON line per case.
"""
import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402


def run_filter(ctx, A, nb, p, seed, pair, moments, **knobs):
    ctx.set_option("pair", pair)
    for k, v in knobs.items():
        ctx.set_option(k, v)
    X = cf.BlockVector(A, nb).randomize_device(seed)
    mom = cf.apply_filter(A, X, p, want_moments=moments)
    got = X.to_numpy()
    X.close()
    return got, (mom.m if mom is not None else None)


def check(ctx, name, A, nb, degree, moments, **knobs):
    p = cf.make_filter((-0.2, 0.25), (-7.0, 7.0), degree, "lanczos2")
    ref, mref = run_filter(ctx, A, nb, p, 5, 0, moments)
    got, mgot = run_filter(ctx, A, nb, p, 5, 2, moments, **knobs)
    exact = bool(np.array_equal(ref.view(np.uint64), got.view(np.uint64)))
    merr = None
    if moments:
        merr = float(np.max(np.abs(mgot - mref)) / np.max(np.abs(mref[0])))
    rec = {"case": name, "nb": nb, "degree": degree, "moments": moments, "bit_exact": exact,
           "moment_rel": merr, "knobs": knobs}
    print(json.dumps(rec), flush=True)
    return exact and (merr is None or merr < 1e-12)


def time_c2(ctx, A, nb, degree, reps, pair, **knobs):
    ctx.set_option("pair", pair)
    for k, v in knobs.items():
        ctx.set_option(k, v)
    p = cf.make_filter((-0.1, 0.1), (-6.0, 6.0), degree, "lanczos2")
    X = cf.BlockVector(A, nb).randomize_device(7)
    cf.apply_filter(A, X, p)
    cf.apply_filter(A, X, p)
    ctx.synchronize()
    ctx.record(0)
    for _ in range(reps):
        cf.apply_filter(A, X, p)
    ctx.record(1)
    ms = ctx.elapsed_ms(0, 1) / reps
    X.close()
    D, nnz = A.dim(), A.nnz()
    s_d = 16 if A.kind else 8
    b = nnz * (s_d + 4) + 5 * D * nb * s_d
    step_ms = ms / degree
    rec = {"pair": pair, "knobs": knobs, "ms_filter": round(ms, 4), "ms_step": round(step_ms, 5),
           "model_gbs": round(b / step_ms / 1e6, 1), "frac_measured": round(b / step_ms / 1e6 / 6547.2, 4)}
    print(json.dumps(rec), flush=True)
    return ms


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--sweep", action="store_true")
    ap.add_argument("--np", type=int, default=100)
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--skip-check", action="store_true")
    args = ap.parse_args()
    ctx = cf.Context(0)
    ok = True
    if not args.skip_check:
        ti8 = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(8, 8, 8, disorder=0.5, seed=3))
        gr = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(24, 20, disorder=0.3, seed=2))
        ti24 = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(24, 20, 16, disorder=0.5, seed=4))
        for deg in (2, 3, 4, 7, 12):
            ok &= check(ctx, "ti8", ti8, 4, deg, True)
        for nb in (1, 2, 3, 8, 32):
            ok &= check(ctx, "ti8", ti8, nb, 9, nb % 2 == 0)
        for nb in (1, 3, 4, 10, 40):
            ok &= check(ctx, "graphene24x20", gr, nb, 10, nb != 3)
        for knobs in ({}, {"pair_tile_rows": 32}, {"pair_threads": 256}, {"pair_extra": 0},
                      {"pair_extra": 3}, {"pair_slab": 4}, {"pair_slab": 5}, {"pair_slab": 1}):
            ok &= check(ctx, "ti24x20x16", ti24, 16, 11, True, **knobs)
            ctx.set_option("pair_tile_rows", 0)
            ctx.set_option("pair_threads", 0)
            ctx.set_option("pair_extra", -1)
            ctx.set_option("pair_slab", 0)
        print(json.dumps({"all_ok": bool(ok)}), flush=True)
    c1 = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(64, 64, disorder=0.1, seed=1))
    for pair in (0, 1):
        time_c2(ctx, c1, 40, 500, 20, pair)
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(64, 64, 64, disorder=0.5, seed=1))
    if not args.skip_check:
        ok2 = check(ctx, "ti64 (C2)", A, 32, 10, True)
        print(json.dumps({"c2_ok": bool(ok2)}), flush=True)
    time_c2(ctx, A, 32, args.np, args.reps, 0)
    time_c2(ctx, A, 32, args.np, args.reps, 1)
    if args.sweep:
        for slab in (8, 16, 4, 32):
            for tr, th in ((32, 128), (64, 128), (32, 256)):
                for hints in (1, 0):
                    time_c2(ctx, A, 32, args.np, args.reps, 2, pair_slab=slab, pair_tile_rows=tr,
                            pair_threads=th, pair_hints=hints)
    ctx.close()


if __name__ == "__main__":
    main()
