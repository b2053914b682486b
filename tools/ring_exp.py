"""A/B of the site-ring step kernel (CHEBFD_OPT_RING) against the row-group / SELL kernels.

    python tools/ring_exp.py [--deg 30] [--cases c4,c2_64] [--sets "ring=0;ring=1;ring=1,ring_segx=128"]

One JSON line per (case, option set): apply_filter ms per Chebyshev step, the single V_n-only
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
CASES = {"c4": ((512, 512, 8), 64), "c3_256": ((128, 128, 64), 256), "c3_64": ((128, 128, 64), 64),
         "c3_32": ((128, 128, 64), 32), "c2": ((64, 64, 64), 32), "c2_64": ((64, 64, 64), 64),
         "c4_32": ((512, 512, 8), 32), "c4_128": ((512, 512, 4), 128),
         "c4_256": ((512, 512, 2), 256), "t32_64": ((32, 32, 32), 64), "t48_32": ((48, 48, 48), 32),
         "t96_32": ((96, 96, 32), 32), "t96_64": ((96, 96, 32), 64), "t32_32": ((32, 32, 32), 32)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--deg", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cases", default="c4")
    ap.add_argument("--sets", default="ring=0;ring=1")
    args = ap.parse_args()
    ctx = cf.Context(0)
    for name in args.cases.split(","):
        l, nb = CASES[name]
        A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(*l, disorder=0.5, seed=1))
        D, nnz = A.dim(), A.nnz()
        p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), args.deg, "lanczos2")
        X = cf.BlockVector(A, nb).randomize_device(7)
        U = cf.BlockVector(A, nb).randomize_device(8)
        W = cf.BlockVector(A, nb).randomize_device(9)
        sched = cf.filter_schedule_bytes(D, nnz, nb, True, args.deg)
        b_recur = nnz * 20 + 3 * D * nb * 16
        b_fused = nnz * 20 + 5 * D * nb * 16
        for s in args.sets.split(";"):
            opts = dict(kv.split("=") for kv in s.split(",") if kv)
            defaults = {"ring": 1, "ring_segx": 0, "ring_no": 0, "ring_nz": 0, "ring_rows": 0,
                        "ring_consts": 1, "ring_tmap": 1, "ring_order": 3, "ring_unit": 0, "slab_units": 0, "band_bytes": 16 << 20}
            for k, d in defaults.items():
                ctx.set_option(k, int(opts.get(k, d)))
            for k, v in opts.items():
                if k not in defaults:
                    ctx.set_option(k, int(v))
            r0, g0 = ctx.ring_launches, ctx.group_launches
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
            print(json.dumps({"case": name, "lattice": list(l), "nb": nb, "options": s,
                              "ring_launches": ctx.ring_launches - r0,
                              "group_launches": ctx.group_launches - g0,
                              "filter_ms_per_step": round(ms / args.deg, 4),
                              "filter_sched_frac": round(sched / (ms * 1e-3) / 1e9 / PEAK, 4),
                              "recur_ms": round(ms_r, 4),
                              "recur_frac": round(b_recur / (ms_r * 1e-3) / 1e9 / PEAK, 4),
                              "fused_ms": round(ms_f, 4),
                              "fused_frac": round(b_fused / (ms_f * 1e-3) / 1e9 / PEAK, 4)}),
                  flush=True)
        del X, U, W, A
    ctx.close()


if __name__ == "__main__":
    main()
