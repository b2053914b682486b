"""Write the golden fixtures in tests/golden/ from the REAL reference.

Runs only in the build container (needs /root/reference, compiled in place
into oracle/_ref/libchebfd_ref.so by oracle/Makefile).  The reference runs
with one OpenMP thread so the chunked reductions are deterministic.  The
fixtures are small and committed; the GPU box never needs the reference.

    python tests/golden/make_golden.py            # everything
    python tests/golden/make_golden.py formats    # only tests/golden/formats/
    python tests/golden/make_golden.py bench      # only bench_filter.json
"""
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

import oracle  # noqa: E402


def formats_golden(r):
    """Matrix Market / .cbfd files written by the reference itself."""
    d = os.path.join(HERE, "formats")
    os.makedirs(d, exist_ok=True)
    g = r.graphene(6, 5, disorder=0.3, seed=2)
    r.write_matrix_market(g, os.path.join(d, "graphene_6x5_symmetric.mtx"), hermitian=True)
    r.write_matrix_market(g, os.path.join(d, "graphene_6x5_general.mtx"), hermitian=False)
    t = r.topological_insulator(2, 2, 3, disorder=0.4, seed=6)
    r.write_matrix_market(t, os.path.join(d, "ti_2x2x3_hermitian.mtx"), hermitian=True)
    r.block_save(r.randomize(30, 4, 5, False), os.path.join(d, "block_real_30x4.cbfd"))
    r.block_save(r.randomize(12, 3, 6, True), os.path.join(d, "block_complex_12x3.cbfd"))


def bench_golden(r):
    """bench_filter's model fields (timing-independent) from the reference."""
    out = {}
    for name, m, sizes in (("graphene_32x32", r.graphene(32, 32, disorder=0.2, seed=3), [1, 3, 8]),
                           ("ti_4x4x4", r.topological_insulator(4, 4, 4, disorder=0.5, seed=2),
                            [1, 4])):
        rows = r.bench_filter(m, sizes, 16, 1000.0)
        out[name] = dict(sizes=sizes, degree=16, bandwidth=1000.0,
                         flops=rows[:, 2].tolist(), intensity=rows[:, 5].tolist(),
                         roofline=rows[:, 6].tolist())
    json.dump(out, open(os.path.join(HERE, "bench_filter.json"), "w"), indent=1)


def main():
    oracle.build()
    r = oracle.Ref(threads=1)
    if sys.argv[1:] == ["formats"]:
        formats_golden(r)
        return
    if sys.argv[1:] == ["bench"]:
        bench_golden(r)
        return
    formats_golden(r)
    bench_golden(r)
    out = {}

    # --- models (models.cpp) ---------------------------------------------
    models = {
        "g_8x8_per": ("graphene", (8, 8), dict(disorder=0.1, seed=1, boundary="periodic_xy_open_z")),
        "g_4x3_open": ("graphene", (4, 3), dict(disorder=1.5, seed=12, boundary="open_all")),
        "g_1x2_per": ("graphene", (1, 2), dict(disorder=0.5, seed=5, boundary="periodic_all")),
        "ti_3x3x3_slab": ("ti", (3, 3, 3), dict(disorder=2.0, seed=9, boundary="periodic_xy_open_z")),
        "ti_4x4x4_per": ("ti", (4, 4, 4), dict(disorder=1.0, seed=1, boundary="periodic_all")),
        "ti_2x2x2_per": ("ti", (2, 2, 2), dict(disorder=0.5, seed=3, boundary="periodic_all")),
        "ti_3x2x2_open": ("ti", (3, 2, 2), dict(disorder=0.5, seed=4, boundary="open_all")),
    }
    for name, (kind, l, kw) in models.items():
        m = r.graphene(*l, **kw) if kind == "graphene" else r.topological_insulator(*l, **kw)
        c = m.csr()
        out[f"model_{name}_offs"] = c.offs
        out[f"model_{name}_cols"] = c.cols
        out[f"model_{name}_vals"] = c.vals

    # --- RNG (block_vector.hpp:42-51) --------------------------------------
    out["rng_real_50x7_s3"] = r.randomize(50, 7, 3, False)
    out["rng_cplx_20x5_s9"] = r.randomize(20, 5, 9, True)

    # --- filter coefficients (filter.cpp) -----------------------------------
    for k in ("none", "fejer", "jackson", "lanczos2", "lanczos3"):
        comb, a, b = r.make_filter((-0.13, 0.21), (-3.05, 3.1), 64, k)
        out[f"filter_{k}"] = np.concatenate([[a, b], comb])
    out["window_half"] = r.window_coeffs((-0.5, 0.5), (-1.0, 1.0), 4)

    # --- kernels and apply_filter (kernels.hpp, filter.hpp) ---------------
    g = r.graphene(8, 8, disorder=0.1, seed=1)
    gc = g.csr()
    x = r.randomize(gc.dim, 3, 7, False)
    comb, a, b = r.make_filter((-0.2, 0.3), (-3.2, 3.3), 20, "lanczos2")
    y, mom = r.apply_filter(g, x, comb, a, b, True)
    out["apply_g_x0"], out["apply_g_y"], out["apply_g_mom"] = x, y, mom
    out["apply_g_filter"] = np.concatenate([[a, b], comb])
    t = r.topological_insulator(3, 3, 3, disorder=0.5, seed=2)
    tc = t.csr()
    xt = r.randomize(tc.dim, 2, 8, True)
    comb, a, b = r.make_filter((-0.4, 0.1), (-5.6, 5.6), 10, "jackson")
    yt, momt = r.apply_filter(t, xt, comb, a, b, True)
    out["apply_t_x0"], out["apply_t_y"], out["apply_t_mom"] = xt, yt, momt
    out["apply_t_filter"] = np.concatenate([[a, b], comb])
    u, w, xx = (r.randomize(tc.dim, 4, s, True) for s in (1, 2, 3))
    out["fused_t_u"], out["fused_t_w"], out["fused_t_x"] = u.copy(), w.copy(), xx.copy()
    d = r.spmmvm_fused(t, u, w, xx, 0.37, -0.21, 0.83, True)
    out["fused_t_w_out"], out["fused_t_x_out"], out["fused_t_dots"] = w, xx, d
    out["gram_t"] = r.gram(u, w)
    np.savez_compressed(os.path.join(HERE, "reference_vectors.npz"), **out)

    # --- spectral probes and full solve (spectral.cpp, solver.cpp) ---------
    t4 = r.topological_insulator(4, 4, 4, disorder=0.5, seed=3)
    kpm = dict(bounds=[-5.6, 5.6], order=200, samples=8, seed=11)
    mu = r.kpm_dos(t4, kpm["bounds"], kpm["order"], kpm["samples"], kpm["seed"])
    json.dump(dict(kpm, mu=mu.tolist()), open(os.path.join(HERE, "kpm_ti4.json"), "w"))

    g16 = r.graphene(16, 16, boundary="periodic_all")
    lo, hi = r.lanczos_bounds(g16, 40, 6)
    json.dump(dict(lx=16, ly=16, iters=40, seed=6, lo=lo, hi=hi),
              open(os.path.join(HERE, "lanczos_g16.json"), "w"))

    # automatic degree (choose_parameters) on a small TI slab
    t6 = r.topological_insulator(6, 6, 6, disorder=0.5, seed=4)
    rep = r.solve(t6, (-0.45, 0.45), degree=0, kernel="lanczos2", seed=3, dos_moments=600,
                  dos_samples=16)
    json.dump(dict(config="TI 6x6x6 slab V=0.5 seed=4, target [-0.45,0.45], N_S auto, degree "
                          "auto (choose_parameters), lanczos2, seed 3, dos 600x16",
                   converged=bool(rep["converged"]), iterations=rep["iterations"],
                   degree=rep["degree"], n_search=rep["n_search"], sigma=rep["sigma"],
                   eta=rep["eta"], n_target_estimate=rep["n_target_estimate"],
                   bounds=[rep["bounds_lo"], rep["bounds_hi"]],
                   accepted_values=sorted(rep["values"][rep["accepted"]].tolist())),
              open(os.path.join(HERE, "ti6_auto_solve.json"), "w"), indent=1)

    r.set_threads(8)  # solve results do not depend on the thread count beyond rounding
    c1 = r.graphene(64, 64, disorder=0.1, seed=1)
    rep = r.solve(c1, (-0.13, 0.13), n_search=40, degree=500, kernel="lanczos2", seed=1)
    acc = rep["values"][rep["accepted"]]
    json.dump(dict(config="graphene 64x64 V=0.1 seed=1, target [-0.13,0.13], N_S=40, N_p=500, "
                          "lanczos2, seed 1 (BASELINE.json configs[0])",
                   converged=bool(rep["converged"]), iterations=rep["iterations"],
                   n_target_estimate=rep["n_target_estimate"],
                   bounds=[rep["bounds_lo"], rep["bounds_hi"]],
                   accepted_values=sorted(acc.tolist()),
                   residual_norms=rep["residual_norms"].tolist(),
                   values=rep["values"].tolist(), history=rep["history"].tolist(),
                   weight_integral=rep["weight_integral"], total_spmvms=rep["total_spmvms"]),
              open(os.path.join(HERE, "c1_solve.json"), "w"), indent=1)
    print("golden fixtures written to", HERE)


if __name__ == "__main__":
    main()
