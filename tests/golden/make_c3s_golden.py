"""Golden for the scaled C3 solve (tests/test_gpu_c3.py), written by the UNMODIFIED
reference (oracle/_ref, OpenMP on all host cores) -- run where oracle/_ref exists:

    python tests/golden/make_c3s_golden.py [--out tests/golden/c3s_solve.json]

C3 (BASELINE.json configs[2]) is the TI slab 128x128x64 (D = 4.19 M) with N_S = 256 and
a window +-h holding ~100 eigenvalues by the seeded KPM DOS.  Its reference solve needs
> 130 GB of host RAM and hours of CPU; this golden is the same protocol on the 1/8-size
slab 64x64x32 (D = 524,288) with N_S = 64 and a window of ~24 eigenvalues: Lanczos
bounds (solver.cpp:101-102), KPM DOS 2000 x 32 with seed + 1 (solver.cpp:105), h by
bisection of the DOS count, then solve() with the automatic degree (choose_parameters),
Jackson and Lanczos-2 kernels.  The GPU test passes the recorded bounds and h."""
import argparse
import json
import os
import sys
import time

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

import numpy as np  # noqa: E402

import oracle  # noqa: E402

LATTICE = (64, 64, 32)
N_SEARCH = 64
TARGET_COUNT = 24.0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=os.path.join(HERE, "c3s_solve.json"))
    args = ap.parse_args()
    cores = len(os.sched_getaffinity(0))
    r = oracle.Ref(threads=cores)
    t0 = time.perf_counter()
    m = r.topological_insulator(*LATTICE, disorder=0.5, seed=1)
    b = r.lanczos_bounds(m, 30, 1)
    mu = r.kpm_dos(m, b, 2000, 32, 2)
    lo, hi = 0.0, 0.999 * min(-b[0], b[1])
    for _ in range(200):
        mid = 0.5 * (lo + hi)
        f = r.dos_count(mu, b, -mid, mid) - TARGET_COUNT
        if abs(f) <= 1e-6 * TARGET_COUNT:
            lo = hi = mid
            break
        lo, hi = (mid, hi) if f < 0 else (lo, mid)
    h = 0.5 * (lo + hi)
    out = {"lattice": LATTICE, "disorder": 0.5, "seed": 1, "n_search": N_SEARCH,
           "target_count": TARGET_COUNT, "bounds": list(b), "h": h, "threads": cores,
           "generator": "tests/golden/make_c3s_golden.py (oracle/_ref)", "runs": {}}
    for kernel in ("lanczos2", "jackson"):
        t1 = time.perf_counter()
        rep = r.solve(m, (-h, h), n_search=N_SEARCH, degree=0, kernel=kernel, seed=1, bounds=b)
        acc = rep["accepted"]
        out["runs"][kernel] = {
            "converged": bool(rep["converged"]), "iterations": int(rep["iterations"]),
            "degree": int(rep["degree"]), "n_search": int(rep["n_search"]),
            "n_target_estimate": rep["n_target_estimate"], "sigma": rep["sigma"],
            "eta": rep["eta"], "weight_integral": rep["weight_integral"],
            "accepted_values": sorted(float(v) for v in rep["values"][acc]),
            "max_accepted_residual": float(np.max(rep["residual_norms"][acc])) if acc.any() else None,
            "seconds": round(time.perf_counter() - t1, 1)}
        print(kernel, json.dumps({k: v for k, v in out["runs"][kernel].items()
                                  if k != "accepted_values"}), flush=True)
    out["seconds_total"] = round(time.perf_counter() - t0, 1)
    json.dump(out, open(args.out, "w"), indent=1)


if __name__ == "__main__":
    main()
