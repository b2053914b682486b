"""A/B of the moment-carrying V_n-only steps on the site-ring kernel (CHEBFD_OPT_RING_DOTS).

    python tools/ring_dots_exp.py [--deg 60] [--cases c4,c3_256]

One JSON line per (case, ring_dots): apply_filter with the MomentTable, ms per Chebyshev step,
and a kpm_dos of 32 samples; the moments of the two settings compared."""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1510_04895_b200 as cf  # noqa: E402

CASES = {"c4": ((512, 512, 8), 64), "c3_256": ((128, 128, 64), 256), "c3_64": ((128, 128, 64), 64)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--deg", type=int, default=60)
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--cases", default="c4,c3_256")
    ap.add_argument("--kpm", type=int, default=400)
    args = ap.parse_args()
    ctx = cf.Context(0)
    for name in args.cases.split(","):
        l, nb = CASES[name]
        A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(*l, disorder=0.5, seed=1))
        p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), args.deg, "lanczos2")
        ref = {}
        for dots in (0, 1, 0, 1):
            ctx.set_option("ring_dots", dots)
            X = cf.BlockVector(A, nb).randomize_device(7)
            r0 = ctx.ring_launches
            mom = cf.apply_filter(A, X, p, want_moments=True)
            launches = ctx.ring_launches - r0
            ctx.synchronize()
            ctx.record(0)
            for _ in range(args.reps):
                cf.apply_filter(A, X, p, want_moments=True)
            ctx.record(1)
            ctx.synchronize()
            ms = ctx.elapsed_ms(0, 1) / args.reps
            t0 = time.perf_counter()
            dos = cf.kpm_dos(A, (-5.6, 5.6), args.kpm, 32, seed=3)
            t_kpm = time.perf_counter() - t0
            rec = {"case": name, "lattice": list(l), "nb": nb, "ring_dots": dots, "deg": args.deg,
                   "ring_launches_per_filter": launches,
                   "filter_with_moments_ms_per_step": round(ms / args.deg, 4),
                   "kpm_order": args.kpm, "kpm_s": round(t_kpm, 3)}
            if dots in ref:
                pass
            elif ref:
                m0, d0 = ref[0]
                rec["moments_rel_diff_vs_dots0"] = float(np.max(np.abs(mom.m - m0)) / np.max(np.abs(m0[0])))
                rec["kpm_rel_diff_vs_dots0"] = float(np.max(np.abs(dos.moments - d0)) / abs(d0[0]))
            ref.setdefault(dots, (mom.m.copy(), dos.moments.copy()))
            print(json.dumps(rec), flush=True)
            del X
        del A
    ctx.close()


if __name__ == "__main__":
    main()
