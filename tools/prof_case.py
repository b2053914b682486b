"""One apply_filter on a TI lattice for ncu captures (no timing).

    python tools/prof_case.py --lattice 512 512 8 --nb 64 --deg 8 [--band MB] [--reps 1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", type=int, nargs=3, default=[512, 512, 8])
    ap.add_argument("--nb", type=int, default=64)
    ap.add_argument("--deg", type=int, default=8)
    ap.add_argument("--band", type=int, default=-1, help="band slice MB (-1: library default)")
    ap.add_argument("--reps", type=int, default=1)
    ap.add_argument("--graphs", type=int, default=0)
    ap.add_argument("--dyn", type=int, default=-1)
    args = ap.parse_args()
    ctx = cf.Context(0)
    ctx.set_option("graphs", args.graphs)
    if args.band >= 0:
        ctx.set_option("band_bytes", args.band << 20)
    if args.dyn >= 0:
        ctx.set_option("tiles_per_cta", args.dyn)
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(*args.lattice, disorder=0.5, seed=1))
    p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), args.deg, "lanczos2")
    X = cf.BlockVector(A, args.nb).randomize_device(7)
    for _ in range(args.reps):
        cf.apply_filter(A, X, p)
    ctx.synchronize()
    ctx.close()


if __name__ == "__main__":
    main()
