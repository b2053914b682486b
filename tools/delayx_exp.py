"""apply_filter with the X update every step vs every second step (CHEBFD_OPT_DELAYED_X).

    python tools/delayx_exp.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402

ctx = cf.Context(0)
cases = [("C2 TI 64^3 nb32 Np100", lambda: cf.SparseMatrix.topological_insulator(
             ctx, cf.LatticeSpec(64, 64, 64, disorder=0.5, seed=1)), 32, 100, 5, (-6.0, 6.0)),
         ("C3 lattice TI 128x128x64 nb256 Np20", lambda: cf.SparseMatrix.topological_insulator(
             ctx, cf.LatticeSpec(128, 128, 64, disorder=0.5, seed=1)), 256, 20, 2, (-6.0, 6.0)),
         ("C1 graphene 64^2 nb40 Np500", lambda: cf.SparseMatrix.graphene(
             ctx, cf.LatticeSpec(64, 64, disorder=0.1, seed=1)), 40, 500, 20, (-3.2, 3.2)),
         ("C5 graphene 2048^2 nb32 Np100", lambda: cf.SparseMatrix.graphene(
             ctx, cf.LatticeSpec(2048, 2048, disorder=1.0, seed=1)), 32, 100, 3, (-3.7, 3.7))]
for name, mk, nb, Np, reps, bnd in cases:
    A = mk()
    p = cf.make_filter((-0.1, 0.1), bnd, Np, "lanczos2")
    X = cf.BlockVector(A, nb).randomize_device(7)
    for dx in (0, 2, 3, 0, 2, 3):
        ctx.set_option("delayed_x", dx)
        for mom in (False, True):
            cf.apply_filter(A, X, p, want_moments=mom)
            ctx.synchronize()
            ctx.record(0)
            for _ in range(reps):
                cf.apply_filter(A, X, p, want_moments=mom)
            ctx.record(1)
            ms = ctx.elapsed_ms(0, 1) / reps
            print(json.dumps({"case": name, "delayed_x": dx, "moments": mom, "ms_filter": round(ms, 4),
                              "us_per_step": round(ms / Np * 1e3, 2)}), flush=True)
    X.close()
    A.close()
ctx.set_option("delayed_x", 3)
ctx.close()
