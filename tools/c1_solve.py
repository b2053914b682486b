"""BASELINE config C1 end to end: graphene 64x64 (V = 0.1, seed 1), N_S = 40,
N_p = 500, Lanczos-2, window [-0.13, 0.13] -- the full ChebFD solve on the
device (twice: cold, i.e. first use of every kernel in the process, and warm)
and, with --reference, the compiled reference's solve on the host cores.

    python tools/c1_solve.py [--reference]
Prints one JSON line per run.
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
    ap.add_argument("--reference", action="store_true")
    args = ap.parse_args()
    t0 = time.perf_counter()
    ctx = cf.Context(0)
    t_ctx = time.perf_counter() - t0
    for run in ("cold", "warm"):
        t0 = time.perf_counter()
        A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(64, 64, disorder=0.1, seed=1))
        rep = cf.solve(A, cf.SolverOptions(target=cf.Interval(-0.13, 0.13), n_search=40,
                                           degree=500, seed=1))
        dt = time.perf_counter() - t0
        acc = rep.ritz.accepted
        print(json.dumps({"config": "C1 graphene 64x64 V=0.1, N_S=40, N_p=500, lanczos2",
                          "run": run, "impl": "b200", "wall_s": round(dt, 4),
                          "context_s": round(t_ctx, 3) if run == "cold" else 0.0,
                          "iterations": rep.iterations, "accepted": int(acc.sum()),
                          "converged": rep.converged,
                          "timings_s": {k: round(v, 4) for k, v in rep.timings.items()}}),
              flush=True)
    ctx.close()
    if args.reference:
        import oracle
        r = oracle.Ref(threads=os.cpu_count())
        m = r.graphene(64, 64, disorder=0.1, seed=1)
        t0 = time.perf_counter()
        rep = r.solve(m, (-0.13, 0.13), n_search=40, degree=500, kernel="lanczos2", seed=1)
        dt = time.perf_counter() - t0
        print(json.dumps({"config": "C1 graphene 64x64 V=0.1, N_S=40, N_p=500, lanczos2",
                          "impl": "reference (oracle/_ref, OpenMP)", "threads": os.cpu_count(),
                          "wall_s": round(dt, 3), "iterations": rep["iterations"],
                          "accepted": int(np.sum(rep["accepted"]))}), flush=True)


if __name__ == "__main__":
    main()
