"""One C2 apply_filter (N_p = 100, no moments unless --moments), graphs off, for ncu:
launches 0/1 are the start-up steps, then V_n-only and X-update steps alternate.

    python tools/prof_filter.py [--moments] [--np 100]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--moments", action="store_true")
ap.add_argument("--np", type=int, default=100)
args = ap.parse_args()
ctx = cf.Context(0)
ctx.set_option("graphs", 0)
A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(64, 64, 64, disorder=0.5, seed=1))
X = cf.BlockVector(A, 32).randomize_device(7)
p = cf.make_filter((-0.1, 0.1), (-6.0, 6.0), args.np, "lanczos2")
cf.apply_filter(A, X, p, want_moments=args.moments)
ctx.synchronize()
print("done")
ctx.close()
