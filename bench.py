"""Fused Chebyshev-filter benchmark (BASELINE.json metric) on B200.

Default workload = BASELINE.json configs[3] (C4), the configuration the metric's
"1/2/4/8 B200" refers to: the 3D topological-insulator slab Hamiltonian, complex
fp64, disorder V = 0.5, seed 1, block width n_b = 64, 200 Chebyshev steps plus one
Rayleigh-Ritz Gram per step.  Weak scaling (the default at N GPUs): every rank owns
a 512 x 512 x 8 sub-lattice of the 512 x 512 x (8 N) slab (N = 1: the one-GPU share
of C4, D = 8,388,608); z-plane row partition, NCCL halo exchange overlapped with the
interior rows, Gram all-reduced.  --strong (N >= 2) adds the fixed 512 x 512 x 64
lattice split over the N ranks.  --workload c2 keeps the round-1 line (configs[1]:
TI 64^3, n_b = 32, N_p = 100, no Gram).

One "step" = one apply_filter (N_p fused recurrence steps, filter.hpp:73-116) of the
resident block + the Gram X^H X of the result (kernels.hpp:165-192).  Every block
exceeds the 126 MB L2 (C4: 8.6 GB), so no flush is needed between steps.

value = the filter's model flops (bench.cpp:28-30,116 with the generator's actual
nnz/row) per step time; the Gram's time is inside the step, its flops are not
counted.  roofline = the V_n-only step kernel (2 of every 3 filter steps) timed
in its own loop right after the timed region: algorithmic bytes nnz*(16+4) +
3*D*n_b*16 per launch (SURVEY §8d for a step that reads U, reads and writes W).
`schedule` = the whole filter's minimal bytes as the library schedules it (X
streamed once per group of three steps) over the filter's time, beside the
reference's 5-stream model bytes.

  python bench.py [--steps K] [--warmup W] [--gpus N] [--impl ours|reference]
                  [--workload c4|c2] [--strong]
"""
from __future__ import annotations

import os

# the reference CPU path (oracle/_ref, OpenMP) binds its threads to cores: set before
# libgomp is loaded
os.environ.setdefault("OMP_PROC_BIND", "close")
os.environ.setdefault("OMP_PLACES", "cores")

import argparse  # noqa: E402
import json  # noqa: E402
import math  # noqa: E402
import statistics  # noqa: E402
import subprocess  # noqa: E402
import sys  # noqa: E402
import time  # noqa: E402

import numpy as np  # noqa: E402

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "fused Chebyshev-filter SpMMV Gflop/s & HBM GB/s (% roofline) at 1/2/4/8 B200"
UNIT = "Gflop/s"
SPEC_HBM_GBS = 8000.0  # B200 datasheet (north star's "~8 TB/s"), for context only

WORKLOADS = {
    # name: (lx, ly, lz per rank, n_b, N_p, gram, BASELINE config)
    "c4": (512, 512, 8, 64, 200, True, "configs[3]"),
    "c2": (64, 64, 64, 32, 100, False, "configs[1]"),
}
NCU_TRAFFIC = {  # committed ncu captures of the dominant kernel for a workload
    "c4": "profiles/r02e_c4_ring_recur_step.json",
    "c2": "profiles/r02_c2_recur_step.json",
}


def peaks():
    path = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(path):
        p = json.load(open(path))
        return p.get("hbm_gbs", 6650.0), "measured (MEASURED_PEAKS.json hbm_gbs, copy)"
    return 6650.0, "fallback (B200_PROFILING.md)"


def model_flops(dim, nnz, nb, degree, cplx=True):
    """bench.cpp:28-30,116: per row, per vector, per step, with the actual nnz/row."""
    f_a, f_m = (2, 6) if cplx else (1, 1)
    per_row = (nnz / dim) * (f_a + f_m) + math.ceil(9 * f_a / 2) + math.ceil(11 * f_m / 2)
    return per_row * dim * nb * degree


def model_step_bytes(dim, nnz, nb, cplx=True):
    """The reference's model bytes of one fused step (bench.cpp:32-34, S_i = 4):
    X read and written every step (5 block streams)."""
    s_d = 16 if cplx else 8
    return nnz * (s_d + 4) + 5 * dim * nb * s_d


def recur_step_bytes(dim, nnz, nb, cplx=True):
    """Algorithmic bytes of one V_n-only step: matrix once, U gathered once, W read and
    written (3 block streams)."""
    s_d = 16 if cplx else 8
    return nnz * (s_d + 4) + 3 * dim * nb * s_d


def gram_flops(dim, nb, cplx=True):
    return (8 if cplx else 2) * dim * nb * nb


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("clocks.sm,clocks.max.sm,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, device=0):
        self.device = device
        self.proc = None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
        except Exception:
            self.proc = None
        time.sleep(0.25)
        return self

    def __exit__(self, *a):
        self.lines = []
        if self.proc:
            time.sleep(0.15)
            self.proc.terminate()
            try:
                out, _ = self.proc.communicate(timeout=5)
            except Exception:
                self.proc.kill()
                out = ""
            self.lines = [ln for ln in out.splitlines() if ln.strip()]

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in getattr(self, "lines", []):
            f = [x.strip() for x in ln.split(",")]
            try:
                sm.append(float(f[0]))
                mx = float(f[1])
            except (ValueError, IndexError):
                continue
            for n, v in zip(names, f[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sm:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


def dist_env():
    return (int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
            int(os.environ.get("LOCAL_RANK", "0")))


def cpu_model():
    try:
        for ln in open("/proc/cpuinfo"):
            if ln.startswith("model name"):
                return ln.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def ncu_traffic(workload, lattice_per_rank):
    """DRAM bytes (read + write) per launch of the dominant kernel from the committed
    ncu capture of this workload (None when the bench runs another shape)."""
    path = os.path.join(ROOT, NCU_TRAFFIC.get(workload, ""))
    if not os.path.isfile(path):
        return None, None
    try:
        rec = json.load(open(path))
        if tuple(rec["lattice"]) != tuple(lattice_per_rank):
            return None, None
        return float(rec["traffic_bytes"]), NCU_TRAFFIC[workload]
    except (OSError, KeyError, ValueError, TypeError):
        return None, None


class Step:
    """One bench step on the device: apply_filter + (optionally) the Gram of the result."""

    def __init__(self, cf, A, X, p, gram):
        self.cf, self.A, self.X, self.p, self.gram = cf, A, X, p, gram

    def __call__(self):
        self.cf.apply_filter(self.A, self.X, self.p)
        if self.gram:
            return self.cf.gram(self.X, self.X)
        return None


def allreduce_max(dist, vals):
    if not dist:
        return vals
    import torch
    t = torch.tensor(vals, dtype=torch.float64)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return [float(v) for v in t]


def run_ours(args):
    import paper_1510_04895_b200 as cf

    rank, world, local = dist_env()
    dist = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("gloo")
        uid = cf.Context.nccl_unique_id() if rank == 0 else bytes(128)
        obj = [uid]
        dist.broadcast_object_list(obj, src=0)
        ctx = cf.Context.distributed(local, rank, world, obj[0])
    else:
        ctx = cf.Context(local)
    lx, ly, lz_r, nb, Np, do_gram, cfg_name = WORKLOADS[args.workload]
    nb = args.nb or nb
    Np = args.degree or Np
    spec = cf.LatticeSpec(lx, ly, lz_r * world, disorder=0.5, seed=1,
                          boundary="periodic_xy_open_z")
    A = cf.SparseMatrix.topological_insulator(ctx, spec)
    D, nnz = A.dim(), A.nnz()
    Dl, nnz_l = A.local_rows, A.info["local_nnz"]
    # the reference bench's window choice (bench.cpp:83-87): centre +- 5 % of the bounds
    bounds = cf.lanczos_bounds(A, 30, 1)
    hw = bounds.half_width()
    target = (bounds.center() - 0.05 * hw, bounds.center() + 0.05 * hw)
    p = cf.make_filter(target, (bounds.lo, bounds.hi), Np, "lanczos2")
    X = cf.BlockVector(A, nb).randomize_device(7 + rank)
    step = Step(cf, A, X, p, do_gram)
    flops_step = model_flops(D, nnz, nb, Np)  # whole job (global operator)
    # ---- device-resident timed region -------------------------------------------------
    for _ in range(args.warmup):
        step()
    ctx.synchronize()
    if dist:
        dist.barrier()
    launches0 = ctx.launch_count
    gram_ms = 0.0
    with ClockSampler(local) as clk:
        ctx.record(0)
        for _ in range(args.steps):
            cf.apply_filter(A, X, p)
            if do_gram:
                ctx.record(2)
                cf.gram(X, X)  # returns the host Gram (synchronises on the result)
                ctx.record(3)
                gram_ms += ctx.elapsed_ms(2, 3)
        ctx.record(1)
        ms = ctx.elapsed_ms(0, 1)
    ctx.synchronize()
    launches = ctx.launch_count - launches0
    ms, gram_ms = allreduce_max(dist, [ms, gram_ms])
    if dist:
        dist.barrier()
    ms_step = ms / args.steps
    filter_ms = (ms - gram_ms) / args.steps
    value = flops_step / (ms_step * 1e-3) / 1e9
    peak, peak_src = peaks()
    # ---- the dominant kernel on its own: V_n-only steps (recurrence_step), 20 launches ---
    U = X
    W = cf.BlockVector(A, nb).randomize_device(11 + rank)
    for _ in range(3):
        cf.recurrence_step(A, U, W, p.alpha, p.beta)
    ctx.synchronize()
    nrec = 20
    ctx.record(4)
    grp0, ring0 = ctx.group_launches, ctx.ring_launches
    for _ in range(nrec):
        cf.recurrence_step(A, U, W, p.alpha, p.beta)
        U, W = W, U
    ctx.record(5)
    grouped = ctx.group_launches - grp0 >= nrec  # which step kernel the library chose
    ringed = ctx.ring_launches - ring0 >= nrec
    rec_ms = ctx.elapsed_ms(4, 5) / nrec
    # ---- the reference's fused step itself (spmmvm_fused, kernels.hpp:74-118): W <- 2(aH+b)U - W,
    # X += c W every launch (5 block streams), 10 launches, no dots
    Xf = cf.BlockVector(A, nb).randomize_device(13 + rank)
    for _ in range(2):
        cf.spmmvm_fused(A, U, W, Xf, p.alpha, p.beta, 1e-3)
    ctx.synchronize()
    nfus = 10
    ctx.record(6)
    for _ in range(nfus):
        cf.spmmvm_fused(A, U, W, Xf, p.alpha, p.beta, 1e-3)
        U, W = W, U
    ctx.record(7)
    fus_ms = ctx.elapsed_ms(6, 7) / nfus
    fus_bytes = model_step_bytes(Dl, nnz_l, nb)
    fus_gbs = fus_bytes / (fus_ms * 1e-3) / 1e9
    del W, Xf
    rec_bytes = recur_step_bytes(Dl, nnz_l, nb)
    achieved = rec_bytes / (rec_ms * 1e-3) / 1e9
    traffic, traffic_src = ncu_traffic(args.workload, (lx, ly, lz_r))
    sched_bytes = cf.filter_schedule_bytes(Dl, nnz_l, nb, True, Np)
    model_bytes = model_step_bytes(Dl, nnz_l, nb) * Np
    sched_gbs = sched_bytes / (filter_ms * 1e-3) / 1e9
    model_gbs = model_bytes / (filter_ms * 1e-3) / 1e9
    # ---- end to end through the public C ABI: pinned host blocks, streamed ----------------
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(cf, ctx, A, p, nb, Dl, do_gram, flops_step, args, dist, rank)
    strong = None
    if args.strong and world > 1 and args.workload == "c4":
        strong = run_strong(cf, ctx, nb, Np, args, dist)
    out = None
    if rank == 0:
        lat = [lx, ly, lz_r * world]
        out = {
            "metric": METRIC, "value": round(value, 2), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms_step, 4),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "c128",
            "data": "synthetic (seeded TI Hamiltonian, device Gaussian start block)",
            "config": {
                "workload": (f"C4 (BASELINE.json {cfg_name}) weak scaling: TI {lx}x{ly}x{lz_r} "
                             "sub-lattice x4 orbitals per GPU" if args.workload == "c4" else
                             f"C2 fused-filter microbenchmark (BASELINE.json {cfg_name})")
                            + f", complex fp64, V=0.5, n_b={nb}, N_p={Np}"
                            + (" + one Rayleigh-Ritz Gram X^H X per step" if do_gram else ""),
                "lattice": lat, "D": D, "nnz": nnz, "nnz_per_row": round(nnz / D, 4),
                "n_b": nb, "N_p": Np, "gram": do_gram,
                "parallelism": (f"row partition x{world} (z-planes), NCCL halo, allreduce Gram"
                                if world > 1 else "single GPU"),
                "l2": f"no flush: every block ({Dl * nb * 16 / 1e9:.2f} GB per GPU) exceeds "
                      "the 126 MB L2",
                "value_counts": "the filter's model flops (bench.cpp:28-30,116); the Gram's "
                                "time is inside the step, its flops are not counted",
                "filter_ms_per_step": round(filter_ms, 3),
                "gram_ms_per_step": round(gram_ms / args.steps, 3) if do_gram else None,
                "gram_tflops": (round(gram_flops(D, nb) / (gram_ms / args.steps * 1e-3) / 1e12, 2)
                                if do_gram and gram_ms > 0 else None),
            },
            "roofline": {
                "bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic,
                "kernel": ("step_ring_kernel<kStepRecur> (site-ring kernel: producer warps + "
                           "TMA-fed shared-memory rings)" if ringed else
                           "step_group_kernel<complex, kStepRecur> (row-group kernel, band order)"
                           if grouped else "step_tma_kernel<complex, kStepRecur> (SELL kernel)")
                          + ": the V_n-only step, 2 of every 3 filter steps",
                "algorithmic_bytes": rec_bytes,
                "launch_ms": round(rec_ms, 4),
                "note": "algorithmic bytes nnz*(16+4) + 3*D*n_b*16 (matrix, U gathered, W read "
                        "and written) per launch / mean duration of 20 launches timed with CUDA "
                        "events on the library stream right after the timed region",
                "peak_source": peak_src,
                "frac_of_spec_8tbs": round(achieved / SPEC_HBM_GBS, 4),
                "traffic_source": (traffic_src + " (dram__bytes_read.sum + dram__bytes_write.sum "
                                   "per launch, ncu)") if traffic_src else None,
                "fused_step": {
                    "note": "the reference's spmmvm_fused (kernels.hpp:74-118) as one launch: "
                            "algorithmic bytes nnz*(16+4) + 5*D*n_b*16 / mean of 10 launches",
                    "launch_ms": round(fus_ms, 4), "algorithmic_bytes": fus_bytes,
                    "achieved_gbs": round(fus_gbs, 1), "frac": round(fus_gbs / peak, 4),
                    "frac_of_spec_8tbs": round(fus_gbs / SPEC_HBM_GBS, 4),
                    "gflops": round(model_flops(Dl, nnz_l, nb, 1) / (fus_ms * 1e-3) / 1e9, 1),
                },
            },
            "schedule": {
                "note": "whole filter: minimal bytes of the library's schedule (X streamed once "
                        "per group of three steps) and the reference's 5-stream model bytes, "
                        "per filter time",
                "bytes_per_filter": sched_bytes, "achieved_gbs": round(sched_gbs, 1),
                "frac": round(sched_gbs / peak, 4),
                "model_bytes_per_filter": model_bytes, "model_gbs": round(model_gbs, 1),
                "model_frac": round(model_gbs / peak, 4),
                "model_frac_of_spec_8tbs": round(model_gbs / SPEC_HBM_GBS, 4),
            },
            "e2e": e2e,
            "gpu_launches": launches,
            "clocks": clk.summary(),
        }
        if strong:
            out["strong"] = strong
        if not args.no_cpu_baseline and world == 1:  # rank 0 at N = 1 only
            out["cpu_baseline"] = cpu_baseline(args)
    if dist:
        dist.barrier()
        dist.destroy_process_group()
    ctx.close()
    return out


def run_e2e(cf, ctx, A, p, nb, Dl, do_gram, flops_step, args, dist, rank):
    """The same step through the public C ABI from pinned HOST blocks: every step's
    H2D copy of the block and D2H copy of the filtered block (and its Gram) are inside
    the timed region, streamed through chebfd_filter_pipe so the copies of neighbouring
    steps overlap the filter."""
    nbytes = Dl * nb * 16
    xa = cf.host_array((Dl, nb), np.complex128)
    xb = cf.host_array((Dl, nb), np.complex128)
    rng = np.random.default_rng(rank)
    xa.view(np.float64)[:] = rng.standard_normal((Dl, 2 * nb))
    xb[:] = xa
    # pinned: a device -> pageable host copy would block the host until the filter ends
    gram_h = [cf.host_array((nb, nb), np.complex128) for _ in range(2)]
    bufs = (xa, xb)
    pipe = cf.FilterPipe(A, nb)

    def submit(k):
        if do_gram:
            pipe.submit(bufs[k % 2], p, gram_out=gram_h[k % 2])
        else:
            pipe.submit(bufs[k % 2], p)

    for k in range(2):
        submit(k)
    pipe.wait()
    if dist:
        dist.barrier()
    e_steps = max(2, min(args.steps, args.e2e_steps))
    t0 = time.perf_counter()
    for k in range(e_steps):
        submit(k)
    pipe.wait()
    e2e_s = (time.perf_counter() - t0) / e_steps
    pipe.close()
    (e2e_s,) = allreduce_max(dist, [e2e_s])
    del xa, xb, bufs
    gbytes = nb * nb * 16 if do_gram else 0
    return {"value": round(flops_step / e2e_s / 1e9, 2), "unit": UNIT,
            "h2d_bytes_per_step": nbytes, "d2h_bytes_per_step": nbytes + gbytes,
            "ms_per_step": round(e2e_s * 1e3, 3), "steps": e_steps,
            "mode": "streamed: chebfd_filter_pipe_submit_gram, pinned host blocks; every step's "
                    "H2D block copy and D2H copies of the filtered block and its Gram inside the "
                    "timed region (host wall clock, max over ranks), overlapped with the "
                    "neighbouring steps' filters"}


def run_strong(cf, ctx, nb, Np, args, dist):
    """Strong scaling: the full C4 lattice 512 x 512 x 64 split over the ranks."""
    spec = cf.LatticeSpec(512, 512, 64, disorder=0.5, seed=1, boundary="periodic_xy_open_z")
    A = cf.SparseMatrix.topological_insulator(ctx, spec)
    D, nnz = A.dim(), A.nnz()
    bounds = cf.lanczos_bounds(A, 30, 1)
    hw = bounds.half_width()
    p = cf.make_filter((bounds.center() - 0.05 * hw, bounds.center() + 0.05 * hw),
                       (bounds.lo, bounds.hi), Np, "lanczos2")
    X = cf.BlockVector(A, nb).randomize_device(7)
    step = Step(cf, A, X, p, True)
    for _ in range(max(1, args.warmup // 2)):
        step()
    ctx.synchronize()
    if dist:
        dist.barrier()
    k = max(2, min(args.steps, 5))
    ctx.record(6)
    for _ in range(k):
        step()
    ctx.record(7)
    (ms,) = allreduce_max(dist, [ctx.elapsed_ms(6, 7) / k])
    del X, A
    return {"lattice": [512, 512, 64], "D": D, "value": round(model_flops(D, nnz, nb, Np) /
                                                               (ms * 1e-3) / 1e9, 2),
            "unit": UNIT, "ms_per_step": round(ms, 3), "steps": k}


# ---------------------------------------------------------------- CPU reference --
def ref_cpu_run(args, budget_s, reps):
    """The reference's own path (oracle/_ref: the unmodified reference compiled with its
    flags, OpenMP on all host cores) on this GPU's share of the workload, on blocks
    allocated once (oracle.Ref.fused_session): one apply_filter of degree 3 timed around
    the call (its start-up -- two fresh zero-filled blocks and the two start-up steps,
    filter.hpp:90-103 -- plus one fused step), one gram(X, X) (kernels.hpp:165-192), and
    `reps` samples of k consecutive spmmvm_fused steps (kernels.hpp:74-118, the loop of
    filter.hpp:105-114), k sized to budget_s.  The full step = start-up + (N_p - 2)
    fused steps (+ Gram) is assembled from those measured pieces."""
    import oracle
    cores = len(os.sched_getaffinity(0)) if hasattr(os, "sched_getaffinity") else os.cpu_count()
    r = oracle.Ref(threads=cores)
    lx, ly, lz, nb, Np, do_gram, _ = WORKLOADS[args.workload]
    nb = args.nb or nb
    Np = args.degree or Np
    t0 = time.perf_counter()
    m = r.topological_insulator(lx, ly, lz, disorder=0.5, seed=1)
    t_build = time.perf_counter() - t0
    sess = r.fused_session(m, nb)
    one = sess.run(1)  # warm (first touch) and size the samples
    k = int(max(1, min(Np - 2, budget_s / max(one, 1e-4))))
    secs = [sess.run(k) for _ in range(reps)]
    fused_s = statistics.median(secs) / k
    comb, a, b = r.make_filter((-0.3, 0.3), (-5.6, 5.6), 3, "lanczos2")
    t3 = sess.apply_filter(comb, a, b)
    start_s = max(t3 - fused_s, 0.0)  # degree 3 = start-up + one fused step
    gram_s = sess.gram() if do_gram else 0.0
    sess.close()
    step_s = start_s + (Np - 2) * fused_s + gram_s
    value = model_flops(m.dim, m.nnz, nb, Np) / step_s / 1e9
    fused_gflops = model_flops(m.dim, m.nnz, nb, 1) / fused_s / 1e9
    sample = (f"reference on the TI {lx}x{ly}x{lz} n_b={nb} block ({m.dim} rows): "
              f"{reps} x {k} spmmvm_fused steps, median {fused_s:.3f} s per step "
              f"({fused_gflops:.1f} Gflop/s); apply_filter degree 3 = {t3:.2f} s -> start-up "
              f"{start_s:.2f} s" + (f"; gram(X, X) = {gram_s:.2f} s" if do_gram else "")
              + f"; full step (start-up + {Np - 2} fused steps" + (" + Gram" if do_gram else "")
              + f") = {step_s:.1f} s; matrix build {t_build:.1f} s (untimed); OpenMP {cores} "
              f"threads, OMP_PROC_BIND={os.environ.get('OMP_PROC_BIND')}, "
              f"OMP_PLACES={os.environ.get('OMP_PLACES')}, CPU {cpu_model()}")
    return {"value": round(value, 3), "unit": UNIT, "cores": cores, "kind": "reference",
            "sample": sample, "ms_per_step": step_s * 1e3, "secs": secs,
            "fused_gflops": round(fused_gflops, 3)}


def cpu_baseline(args):
    import oracle
    if not oracle.ref_available():
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                "sample": "oracle/_ref not built on this host"}
    res = ref_cpu_run(args, budget_s=3.0, reps=3)
    return {k: res[k] for k in ("value", "unit", "cores", "kind", "sample", "fused_gflops")}


def run_reference(args):
    rank, world, _ = dist_env()
    if rank != 0:
        return None
    import oracle
    if not oracle.ref_available():
        return {"impl": "reference", "unavailable": "oracle/_ref/libchebfd_ref.so not built"}
    # each step: a bounded sample, sized so warm-up + steps stay within ~3 minutes of CPU
    reps_total = args.steps + args.warmup
    res = ref_cpu_run(args, budget_s=max(1.0, 90.0 / reps_total), reps=reps_total)
    lx, ly, lz, nb, Np, do_gram, cfg_name = WORKLOADS[args.workload]
    cb = {k: res[k] for k in ("value", "unit", "cores", "kind", "sample", "fused_gflops")}
    return {
        "impl": "reference", "metric": METRIC, "value": res["value"], "unit": UNIT,
        "n_gpus": 0, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(res["ms_per_step"], 1), "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "c128",
        "data": "synthetic (seeded TI Hamiltonian, Gaussian block)",
        "config": {"workload": f"{args.workload.upper()} (BASELINE.json {cfg_name}) one GPU's "
                               f"share: TI {lx}x{ly}x{lz}, n_b={args.nb or nb}, "
                               f"N_p={args.degree or Np}" + (" + one Gram" if do_gram else "")
                               + "; each timed step = a bounded sample of consecutive "
                                 "spmmvm_fused steps on resident blocks; the full step = the "
                                 "measured apply_filter start-up + (N_p - 2) fused steps (+ the "
                                 "measured Gram)",
                   "lattice": [lx, ly, lz], "n_b": args.nb or nb, "N_p": args.degree or Np},
        "cpu_baseline": cb,
        "e2e": {"value": res["value"], "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--workload", default="c4", choices=sorted(WORKLOADS))
    ap.add_argument("--nb", type=int, default=0, help="block width (0: the workload's)")
    ap.add_argument("--degree", type=int, default=0, help="N_p (0: the workload's)")
    ap.add_argument("--strong", action="store_true",
                    help="N >= 2: also the full 512x512x64 lattice split over the ranks")
    ap.add_argument("--e2e-steps", type=int, default=12)
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    out = run_reference(args) if args.impl == "reference" else run_ours(args)
    if out is not None:
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
