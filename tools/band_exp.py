"""A/B of the band (2.5D) tile order (CHEBFD_OPT_BAND_BYTES) on the TI lattices.

    python tools/band_exp.py [--deg 30] [--cases c4,c3_256,c3_32,c2] [--bytes 0,4,8,16,32]

Prints one JSON line per (case, band_bytes): apply_filter ms per Chebyshev step,
the reference-model bytes rate and the minimal-schedule bytes rate (fractions of
the measured copy bandwidth)."""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402

PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json")))["hbm_gbs"] \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6650.0
CASES = {"c4": ((512, 512, 8), 64), "c3_256": ((128, 128, 64), 256), "c3_32": ((128, 128, 64), 32),
         "c2": ((64, 64, 64), 32), "c4x2": ((512, 512, 16), 64)}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--deg", type=int, default=30)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--cases", default="c4,c3_256,c3_32,c2")
    ap.add_argument("--bytes", default="0,4,8,16,32,64")
    ap.add_argument("--dyn", default="-1", help="tiles per CTA of dot-free launches, comma list (0: persistent; -1: default)")
    args = ap.parse_args()
    ctx = cf.Context(0)
    for name in args.cases.split(","):
        (lx, ly, lz), nb = CASES[name]
        A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(lx, ly, lz, disorder=0.5, seed=1))
        D, nnz = A.dim(), A.nnz()
        p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), args.deg, "lanczos2")
        X = cf.BlockVector(A, nb).randomize_device(7)
        model = (nnz * 20 + 5 * D * nb * 16) * args.deg
        sched = cf.filter_schedule_bytes(D, nnz, nb, True, args.deg)
        for dyn, mb in [(int(d), int(x)) for d in args.dyn.split(",") for x in args.bytes.split(",")]:
            if mb >= 0:  # -1: leave the library default (older builds lack the option)
                ctx.set_option("band_bytes", mb << 20)
            if dyn >= 0:
                ctx.set_option("tiles_per_cta", dyn)
            cf.apply_filter(A, X, p)
            ctx.synchronize()
            ctx.record(0)
            for _ in range(args.reps):
                cf.apply_filter(A, X, p)
            ctx.record(1)
            ms = ctx.elapsed_ms(0, 1) / args.reps
            print(json.dumps({"case": name, "lattice": [lx, ly, lz], "nb": nb, "band_mb": mb, "dyn": dyn,
                              "ms_per_step": round(ms / args.deg, 4),
                              "model_frac": round(model / (ms * 1e-3) / 1e9 / PEAK, 4),
                              "sched_frac": round(sched / (ms * 1e-3) / 1e9 / PEAK, 4)}), flush=True)
        del X, A
    ctx.close()


if __name__ == "__main__":
    main()
