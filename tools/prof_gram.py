"""Rayleigh-Ritz Gram contractions (Y^H Y, Q^H AQ) on the device: time per call
and FP64 rate, for the tensor-pipe ncu capture.

    python tools/prof_gram.py [--lattice 64 --lz 64 --nb 64 --reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--lattice", type=int, default=64)
ap.add_argument("--lz", type=int, default=64)
ap.add_argument("--nb", type=int, default=64)
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
ctx = cf.Context(0)
A = cf.SparseMatrix.topological_insulator(
    ctx, cf.LatticeSpec(args.lattice, args.lattice, args.lz, disorder=0.5, seed=1))
D, nb = A.dim(), args.nb
Y = cf.BlockVector(A, nb).randomize_device(3)
Z = cf.BlockVector(A, nb).randomize_device(4)
cf.gram(Y, Z)
ctx.synchronize()
ctx.record(0)
for _ in range(args.reps):
    cf.gram(Y, Z)
ctx.record(1)
ms = ctx.elapsed_ms(0, 1) / args.reps
flops = 8.0 * D * nb * nb  # complex: 4 real multiply-adds per entry product
print(json.dumps({"D": D, "n_b": nb, "gram_ms": round(ms, 3), "fp64_tflops": round(flops / ms / 1e9, 2),
                  "bytes_gb": round(2 * D * nb * 16 / 1e9, 3)}), flush=True)
ctx.close()
