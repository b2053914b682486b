"""Run a few fused Chebyshev steps of a bench workload for profiling.

    python tools/prof_step.py --kernel v3 --steps 6 [--lattice 64 --nb 32]
Prints the CUDA-event time per fused step and the model GB/s.
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--kernel", default="tma", choices=["gather", "tma", "stage", "tma2"])
    ap.add_argument("--steps", type=int, default=6)
    ap.add_argument("--lattice", type=int, default=64)
    ap.add_argument("--nb", type=int, default=32)
    ap.add_argument("--model", default="ti", choices=["ti", "graphene"])
    ap.add_argument("--moments", action="store_true")
    ap.add_argument("--lz", type=int, default=0, help="TI z extent (default = lattice)")
    args = ap.parse_args()
    ctx = cf.Context(0)
    ctx.set_option("kernel", args.kernel)
    L = args.lattice
    if args.model == "ti":
        A = cf.SparseMatrix.topological_insulator(
            ctx, cf.LatticeSpec(L, L, args.lz or L, disorder=0.5))
        s_d = 16
    else:
        A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(L, L, disorder=1.0))
        s_d = 8
    D, nnz, nb = A.dim(), A.nnz(), args.nb
    U = cf.BlockVector(A, nb).randomize_device(1)
    W = cf.BlockVector(A, nb).randomize_device(2)
    X = cf.BlockVector(A, nb).randomize_device(3)
    alpha, beta = 0.17, 0.01
    # the apply_filter path pre-scales values; do the same through a degree-2 filter once
    p = cf.make_filter((-0.1, 0.1), (-6.0, 6.0), 2, "lanczos2")
    cf.apply_filter(A, X, p)
    for _ in range(2):
        cf.spmmvm_fused(A, U, W, X, p.alpha, p.beta, 0.3)
    ctx.record(0)
    for _ in range(args.steps):
        cf.spmmvm_fused(A, U, W, X, p.alpha, p.beta, 0.3)
        U, W = W, U
    ctx.record(1)
    ms = ctx.elapsed_ms(0, 1) / args.steps
    b = nnz * (s_d + 4) + 5 * D * nb * s_d
    print(f"{args.kernel}: {ms:.4f} ms/step, {b / ms / 1e6:.1f} GB/s model, D={D} nnz={nnz} nb={nb}")
    ctx.close()


if __name__ == "__main__":
    main()
