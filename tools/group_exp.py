"""A/B of the row-group step kernel (CHEBFD_OPT_GROUPED) against the SELL kernels.

    python tools/group_exp.py [--deg 30] [--cases c2,c4,c3_32,c3_256,c5_32] [--modes 0,1]

One JSON line per (case, grouped): apply_filter ms per Chebyshev step, the single V_n-only
step (recurrence_step) and the single fused step (spmmvm_fused) timed alone, with each
kernel's algorithmic-bytes rate as a fraction of the measured copy bandwidth."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
CASES = {"c4": ("ti", (512, 512, 8), 64), "c3_256": ("ti", (128, 128, 64), 256),
         "c3_32": ("ti", (128, 128, 64), 32), "c2": ("ti", (64, 64, 64), 32),
         "c2_64": ("ti", (64, 64, 64), 64), "c2_16": ("ti", (64, 64, 64), 16),
         "c5_32": ("graphene", (2048, 2048), 32), "c5_64": ("graphene", (2048, 2048), 64),
         "c5_8": ("graphene", (2048, 2048), 8)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--deg", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cases", default="c2,c4")
    ap.add_argument("--modes", default="0,1")
    args = ap.parse_args()
    ctx = cf.Context(0)
    for name in args.cases.split(","):
        model, l, nb = CASES[name]
        ti = model == "ti"
        spec = cf.LatticeSpec(*l, disorder=0.5 if ti else 1.0, seed=1)
        A = (cf.SparseMatrix.topological_insulator if ti else cf.SparseMatrix.graphene)(ctx, spec)
        D, nnz = A.dim(), A.nnz()
        sd = 16 if ti else 8
        bounds = (-5.6, 5.6) if ti else (-3.6, 3.6)
        p = cf.make_filter((-0.3, 0.3), bounds, args.deg, "lanczos2")
        X = cf.BlockVector(A, nb).randomize_device(7)
        U = cf.BlockVector(A, nb).randomize_device(8)
        W = cf.BlockVector(A, nb).randomize_device(9)
        sched = cf.filter_schedule_bytes(D, nnz, nb, ti, args.deg)
        b_recur = nnz * (sd + 4) + 3 * D * nb * sd
        b_fused = nnz * (sd + 4) + 5 * D * nb * sd
        for mode in [int(m) for m in args.modes.split(",")]:
            ctx.set_option("grouped", mode)
            g0 = ctx.group_launches
            cf.apply_filter(A, X, p)
            ctx.synchronize()
            ctx.record(0)
            for _ in range(args.reps):
                cf.apply_filter(A, X, p)
            ctx.record(1)
            ctx.synchronize()
            ms = ctx.elapsed_ms(0, 1) / args.reps
            cf.recurrence_step(A, U, W, 0.35, 0.01)
            ctx.record(2)
            for _ in range(10):
                cf.recurrence_step(A, U, W, 0.35, 0.01)
            ctx.record(3)
            ctx.synchronize()
            ms_r = ctx.elapsed_ms(2, 3) / 10
            cf.spmmvm_fused(A, U, W, X, 0.35, 0.01, 1e-3)
            ctx.record(4)
            for _ in range(10):
                cf.spmmvm_fused(A, U, W, X, 0.35, 0.01, 1e-3)
            ctx.record(5)
            ctx.synchronize()
            ms_f = ctx.elapsed_ms(4, 5) / 10
            print(json.dumps({"case": name, "lattice": list(l), "nb": nb, "grouped": mode,
                              "group_launches": ctx.group_launches - g0,
                              "filter_ms_per_step": round(ms / args.deg, 4),
                              "filter_sched_frac": round(sched / (ms * 1e-3) / 1e9 / PEAK, 4),
                              "recur_ms": round(ms_r, 4),
                              "recur_frac": round(b_recur / (ms_r * 1e-3) / 1e9 / PEAK, 4),
                              "fused_ms": round(ms_f, 4),
                              "fused_frac": round(b_fused / (ms_f * 1e-3) / 1e9 / PEAK, 4)}),
                  flush=True)
        del X, U, W, A
    ctx.set_option("grouped", 1)
    ctx.close()


if __name__ == "__main__":
    main()
