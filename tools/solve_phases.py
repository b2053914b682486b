"""Time the phases of a ChebFD solve (C1 by default) to find setup costs.

    python tools/solve_phases.py [--lattice 64] [--nb 40] [--degree 500]
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", type=int, default=64)
    ap.add_argument("--nb", type=int, default=40)
    ap.add_argument("--degree", type=int, default=500)
    args = ap.parse_args()
    t = {}
    t0 = time.perf_counter()
    ctx = cf.Context(0)
    t["context"] = time.perf_counter() - t0

    def tick(name, fn):
        s = time.perf_counter()
        r = fn()
        ctx.synchronize()
        t[name] = round(time.perf_counter() - s, 4)
        return r

    A = tick("matrix", lambda: cf.SparseMatrix.graphene(
        ctx, cf.LatticeSpec(args.lattice, args.lattice, disorder=0.1, seed=1)))
    b = tick("lanczos_bounds", lambda: cf.lanczos_bounds(A, 30, 1))
    tick("kpm_dos", lambda: cf.kpm_dos(A, b, 2000, 32, 2))
    p = cf.make_filter((-0.13, 0.13), b, args.degree, "lanczos2")
    X = cf.BlockVector(A, args.nb).randomize(3)
    tick("apply_filter_first", lambda: cf.apply_filter(A, X, p, True))
    tick("apply_filter", lambda: cf.apply_filter(A, X, p, True))
    q = tick("svqb_first", lambda: cf.svqb_orthonormalize(X))
    tick("svqb", lambda: cf.svqb_orthonormalize(X))
    tick("rayleigh_ritz", lambda: cf.rayleigh_ritz(A, q.q))
    rep = tick("solve_total", lambda: cf.solve(A, cf.SolverOptions(
        target=cf.Interval(-0.13, 0.13), n_search=args.nb, degree=args.degree, seed=1)))
    t["solve_iterations"] = rep.iterations
    t["solve_accepted"] = int(rep.ritz.accepted.sum())
    print(json.dumps(t))
    ctx.close()


if __name__ == "__main__":
    main()
