"""The bench's dominant kernel alone, for ncu: V_n-only recurrence steps
(chebfd_recurrence_step -> step_tma_kernel<complex, kStepRecur>) on a TI lattice.

    python tools/prof_recur.py [--lattice 512 512 8] [--nb 64] [--launches 3]
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
    ap.add_argument("--launches", type=int, default=3)
    ap.add_argument("--opt", action="append", default=[], help="context option name=value (repeatable)")
    args = ap.parse_args()
    ctx = cf.Context(0)
    for kv in args.opt:
        k, v = kv.split("=")
        ctx.set_option(k, int(v))
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(*args.lattice, disorder=0.5, seed=1))
    p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), 4, "lanczos2")
    cf.apply_filter(A, cf.BlockVector(A, 1).randomize_device(1), p)  # builds the scaled values
    U = cf.BlockVector(A, args.nb).randomize_device(7)
    W = cf.BlockVector(A, args.nb).randomize_device(8)
    for _ in range(args.launches):
        cf.recurrence_step(A, U, W, p.alpha, p.beta)
        U, W = W, U
    ctx.synchronize()
    ctx.close()


if __name__ == "__main__":
    main()
