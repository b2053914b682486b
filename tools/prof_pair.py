"""One C2 apply_filter (N_p = 6) with the pair kernel forced on or off, for ncu.

    python tools/prof_pair.py --pair 2 [--tile-rows 32 --threads 128 --extra -1]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--pair", type=int, default=2)
ap.add_argument("--tile-rows", type=int, default=0)
ap.add_argument("--threads", type=int, default=0)
ap.add_argument("--extra", type=int, default=-1)
ap.add_argument("--np", type=int, default=6)
ap.add_argument("--lattice", type=int, default=64)
ap.add_argument("--nb", type=int, default=32)
args = ap.parse_args()
ctx = cf.Context(0)
ctx.set_option("graphs", 0)
ctx.set_option("pair", args.pair)
ctx.set_option("pair_tile_rows", args.tile_rows)
ctx.set_option("pair_threads", args.threads)
ctx.set_option("pair_extra", args.extra)
L = args.lattice
A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(L, L, L, disorder=0.5, seed=1))
X = cf.BlockVector(A, args.nb).randomize_device(7)
p = cf.make_filter((-0.1, 0.1), (-6.0, 6.0), args.np, "lanczos2")
cf.apply_filter(A, X, p)
ctx.synchronize()
print("done")
ctx.close()
