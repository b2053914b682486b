"""BASELINE config C3: full ChebFD on the TI slab 128x128x64 (D = 4,194,304),
complex fp64, N_S = 256, window +-h with KPM count(-h, h) = 100 from a seeded
DOS estimate (bisection as filter_design.cpp:330-354), degree chosen by the
reference's rule (choose_parameters), Jackson vs Lanczos-2.

    python tools/c3.py [--lattice 128 128 64] [--kernels jackson lanczos2]
Prints one JSON line per kernel.
"""
import argparse
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import paper_1510_04895_b200 as cf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--lattice", type=int, nargs=3, default=[128, 128, 64])
    ap.add_argument("--kernels", nargs="+", default=["jackson", "lanczos2"])
    ap.add_argument("--n-search", type=int, default=256)
    ap.add_argument("--target-count", type=float, default=100.0)
    ap.add_argument("--max-iters", type=int, default=40)
    args = ap.parse_args()
    ctx = cf.Context(0)
    t0 = time.perf_counter()
    A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(*args.lattice, disorder=0.5, seed=1))
    t_build = time.perf_counter() - t0
    b = cf.lanczos_bounds(A, 30, 1)          # what solve() computes (solver.cpp:101-102)
    dos = cf.kpm_dos(A, b, 2000, 32, 2)      # solve's DOS: seed + 1 (solver.cpp:105)
    lo, hi = 0.0, 0.999 * min(-b.lo, b.hi)
    for _ in range(200):                     # count(-h, h) = target_count
        mid = 0.5 * (lo + hi)
        f = dos.count(-mid, mid) - args.target_count
        if abs(f) <= 1e-6 * args.target_count:
            lo = hi = mid
            break
        lo, hi = (mid, hi) if f < 0 else (lo, mid)
    h = 0.5 * (lo + hi)
    for kernel in args.kernels:
        t0 = time.perf_counter()
        rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(-h, h), n_search=args.n_search,
                                           degree=0, kernel=cf.Kernel.parse(kernel), seed=1,
                                           max_iters=args.max_iters, bounds=b))
        dt = time.perf_counter() - t0
        acc = rep.ritz.accepted
        vals = rep.ritz.values[acc]
        print(json.dumps({
            "config": f"C3 TI {args.lattice} slab V=0.5, N_S={args.n_search}, window +-h, "
                      f"KPM count {args.target_count}",
            "kernel": kernel, "D": A.dim(), "h": h, "bounds": [b.lo, b.hi],
            "n_target_estimate": rep.n_target_estimate, "degree": rep.degree,
            "sigma": rep.sigma, "eta": rep.eta, "converged": rep.converged,
            "iterations": rep.iterations, "accepted": int(acc.sum()),
            "max_accepted_residual": float(np.max(rep.ritz.residual_norms[acc])) if acc.any() else None,
            "accepted_in_window": bool(np.all(np.abs(vals) <= h)),
            "total_spmvms": rep.total_spmvms, "solve_s": round(dt, 2),
            "matrix_build_s": round(t_build, 2),
            "timings_s": {k: round(v, 3) for k, v in rep.timings.items()},
            "history": rep.history.tolist()}), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
