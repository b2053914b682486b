"""The hand-written DMMA Gram (gram.cu, CHEBFD_OPT_GRAM=1) against cuBLAS (=0): time and
agreement on the bench / solver shapes.

    python tools/gram_exp.py [--reps 5]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1510_04895_b200 as cf  # noqa: E402

CASES = [("C4 share Y^H Y", "ti", (512, 512, 8), 64, True),
         ("C3 Y^H Y", "ti", (128, 128, 64), 256, True),
         ("C3 Q^H AQ", "ti", (128, 128, 64), 256, False),
         ("C2 Y^H Y", "ti", (64, 64, 64), 32, True),
         ("C5 graphene Y^H Y", "graphene", (2048, 2048), 64, True),
         ("C1 graphene", "graphene", (64, 64), 40, True)]


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--reps", type=int, default=5)
    args = ap.parse_args()
    ctx = cf.Context(0)
    for name, model, l, nb, same in CASES:
        spec = cf.LatticeSpec(*l, disorder=0.5, seed=1)
        A = (cf.SparseMatrix.topological_insulator(ctx, spec) if model == "ti"
             else cf.SparseMatrix.graphene(ctx, spec))
        X = cf.BlockVector(A, nb).randomize_device(1)
        Y = X if same else cf.BlockVector(A, nb).randomize_device(2)
        out = {}
        res = {}
        for mode in (0, 1, 2):
            ctx.set_option("gram", mode)
            res[mode] = cf.gram(X, Y)
            ctx.synchronize()
            ctx.record(0)
            for _ in range(args.reps):
                cf.gram(X, Y)
            ctx.record(1)
            out[mode] = ctx.elapsed_ms(0, 1) / args.reps
        D = A.dim()
        flops = (8 if model == "ti" else 2) * D * nb * nb
        diff = float(np.max(np.abs(res[1] - res[0])) / np.max(np.abs(res[0])))
        diff2 = float(np.max(np.abs(res[2] - res[0])) / np.max(np.abs(res[0])))
        print(json.dumps({"case": name, "D": D, "nb": nb, "cublas_ms": round(out[0], 3),
                          "default_ms": round(out[1], 3), "dmma_forced_ms": round(out[2], 3),
                          "cublas_tflops": round(flops / out[0] * 1e-9, 2),
                          "dmma_tflops_equiv": round(flops / out[2] * 1e-9, 2),
                          "speedup_default": round(out[0] / out[1], 3),
                          "speedup_dmma": round(out[0] / out[2], 3), "rel_diff_dmma": diff2}),
              flush=True)
        del X, Y
        A.close()
    ctx.set_option("gram", 1)
    ctx.close()




def tsgemm(reps=3):
    """block_mult_small Y = X B: the DMMA kernel (gram.cu) against cuBLAS ZGEMM."""
    ctx = cf.Context(0)
    for name, l, nb in (("C4 share Y=XB", (512, 512, 8), 64), ("C3 Y=XB", (128, 128, 64), 256),
                        ("C2 Y=XB", (64, 64, 64), 32)):
        A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(*l, disorder=0.5, seed=1))
        X = cf.BlockVector(A, nb).randomize_device(1)
        rng = np.random.default_rng(3)
        B = (rng.standard_normal((nb, nb)) + 1j * rng.standard_normal((nb, nb))).astype(np.complex128)
        out, res = {}, {}
        for mode in (0, 2):
            ctx.set_option("gram", mode)
            Y = cf.block_mult_small(X, B)
            res[mode] = Y.to_numpy()[:4096]
            Y.close()
            ctx.synchronize()
            ctx.record(0)
            for _ in range(reps):
                Y = cf.block_mult_small(X, B)
                Y.close()
            ctx.record(1)
            out[mode] = ctx.elapsed_ms(0, 1) / reps
        flops = 8 * A.dim() * nb * nb
        print(json.dumps({"case": name, "D": A.dim(), "nb": nb, "cublas_ms": round(out[0], 3),
                          "dmma_ms": round(out[2], 3), "cublas_tflops": round(flops / out[0] * 1e-9, 2),
                          "dmma_tflops": round(flops / out[2] * 1e-9, 2),
                          "speedup": round(out[0] / out[2], 3),
                          "rel_diff": float(np.max(np.abs(res[2] - res[0])) / np.max(np.abs(res[0])))}),
              flush=True)
        X.close()
        A.close()
    ctx.set_option("gram", 1)
    ctx.close()


if __name__ == "__main__":
    if "--tsgemm" in sys.argv:
        tsgemm()
    else:
        main()
