"""Time the step-kernel workloads whose z +- 1 planes exceed the L2 (KPM on the
C3 lattice, C3 fused steps) and C2, for A/B builds of the library
(CHEBFD_B200_LIB selects the .so).

    CHEBFD_B200_LIB=... python tools/l2_exp.py
"""
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402


def step_time(ctx, A, nb, steps, s_d):
    U = cf.BlockVector(A, nb).randomize_device(1)
    W = cf.BlockVector(A, nb).randomize_device(2)
    X = cf.BlockVector(A, nb).randomize_device(3)
    p = cf.make_filter((-0.1, 0.1), (-6.0, 6.0), 2, "lanczos2")
    cf.apply_filter(A, X, p)
    cf.spmmvm_fused(A, U, W, X, p.alpha, p.beta, 0.3)
    ctx.synchronize()
    ctx.record(0)
    for _ in range(steps):
        cf.spmmvm_fused(A, U, W, X, p.alpha, p.beta, 0.3)
        U, W = W, U
    ctx.record(1)
    ms = ctx.elapsed_ms(0, 1) / steps
    for b in (U, W, X):
        b.close()
    D, nnz = A.dim(), A.nnz()
    b = nnz * (s_d + 4) + 5 * D * nb * s_d
    return ms, b / ms / 1e6


def main():
    lib = os.environ.get("CHEBFD_B200_LIB", "default")
    ctx = cf.Context(0)
    out = {"lib": os.path.basename(lib)}
    c3 = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(128, 128, 64, disorder=0.5, seed=1))
    b = cf.Interval(-6.0, 6.0)
    cf.kpm_dos(c3, b, 20, 32)
    ctx.synchronize()
    t0 = time.perf_counter()
    cf.kpm_dos(c3, b, 400, 32)
    ctx.synchronize()
    kpm_s = time.perf_counter() - t0
    D, nnz = c3.dim(), c3.nnz()
    kb = nnz * 20 + 4 * D * 32 * 16
    out["kpm_c3_400_s"] = round(kpm_s, 4)
    out["kpm_c3_model_gbs"] = round(kb * 399 / kpm_s / 1e9, 1)
    for nb in (32, 256):
        ms, gbs = step_time(ctx, c3, nb, 6 if nb == 256 else 20, 16)
        out[f"c3_fused_nb{nb}_ms"] = round(ms, 4)
        out[f"c3_fused_nb{nb}_gbs"] = round(gbs, 1)
    c3.close()
    c2 = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(64, 64, 64, disorder=0.5, seed=1))
    ms, gbs = step_time(ctx, c2, 32, 40, 16)
    out["c2_fused_ms"] = round(ms, 4)
    out["c2_fused_gbs"] = round(gbs, 1)
    print(json.dumps(out), flush=True)
    ctx.close()


if __name__ == "__main__":
    main()
