"""C3 lattice (TI 128x128x64), n_b = 256: fused-step time per column-slab width.

    python tools/slab_exp.py
"""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402
from l2_exp import step_time  # noqa: E402

ctx = cf.Context(0)
c3 = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(128, 128, 64, disorder=0.5, seed=1))
for slab in (0, 128, 64, 32, 16):
    ctx.set_option("slab_units", slab)
    ms, gbs = step_time(ctx, c3, 256, 5, 16)
    print(json.dumps({"slab_units": slab, "ms": round(ms, 3), "model_gbs": round(gbs, 1)}), flush=True)
ctx.close()
