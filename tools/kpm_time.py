import sys, time, json
sys.path.insert(0, '/root/repo')
import paper_1510_04895_b200 as cf
ctx = cf.Context(0)
A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(128, 128, 64, disorder=0.5, seed=1))
for ring in (1, 2, 1, 2):
    ctx.set_option("ring", ring)
    dots = ring
    for order in (400, 2000):
        r0, l0 = ctx.ring_launches, ctx.launch_count
        t0 = time.perf_counter(); cf.kpm_dos(A, (-5.6, 5.6), order, 32, seed=3); t = time.perf_counter() - t0
        print(json.dumps({"ring_opt": dots, "order": order, "s": round(t, 3), "ring": ctx.ring_launches - r0, "launches": ctx.launch_count - l0}), flush=True)
