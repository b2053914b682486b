"""kpm_dos on the C3 lattice (TI 128x128x64, 32 probes) for an ncu launch list;
also apply_filter on C2 with and without moments (the <x0, w> stream).

    python tools/prof_kpm.py [--order 40]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--order", type=int, default=40)
ap.add_argument("--c2", action="store_true")
args = ap.parse_args()
ctx = cf.Context(0)
if args.c2:
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(64, 64, 64, disorder=0.5, seed=1))
    X = cf.BlockVector(A, 32).randomize_device(7)
    p = cf.make_filter((-0.1, 0.1), (-6.0, 6.0), 100, "lanczos2")
    for mom in (False, True, False, True):
        cf.apply_filter(A, X, p, want_moments=mom)
        ctx.synchronize()
        ctx.record(0)
        for _ in range(3):
            cf.apply_filter(A, X, p, want_moments=mom)
        ctx.record(1)
        print(json.dumps({"c2_moments": mom, "ms_filter": ctx.elapsed_ms(0, 1) / 3}), flush=True)
else:
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(128, 128, 64, disorder=0.5, seed=1))
    t0 = time.perf_counter()
    cf.kpm_dos(A, cf.Interval(-6.0, 6.0), args.order, 32)
    ctx.synchronize()
    print(json.dumps({"kpm_order": args.order, "s": time.perf_counter() - t0}), flush=True)
ctx.close()
