"""The distributed filter's schedule on one GPU: C4's weak-scaled lattice 512 x 512 x (8 P)
split over P virtual ranks (chebfd_vgroup_*), each rank's steps split into interior and
boundary launches with the halo rows pulled from the neighbours -- against P times the
one-rank time.  All ranks share one GPU's HBM, so the ideal is t_P = P t_1; the excess
is the cost of the distributed schedule itself (smaller launches, halo traffic).

    python tools/vgroup_bench.py [--ranks 1,2,4] [--deg 60] [--reps 3] [--nb 64]
"""
import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_1510_04895_b200 as cf  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--ranks", default="1,2,4")
    ap.add_argument("--deg", type=int, default=60)
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--nb", type=int, default=64)
    ap.add_argument("--lz", type=int, default=8)
    ap.add_argument("--compact", type=int, default=1)
    ap.add_argument("--opt", action="append", default=[], help="context option name=value (repeatable)")
    args = ap.parse_args()
    t1 = None
    for P in (int(x) for x in args.ranks.split(",")):
        g = cf.VirtualGroup(P)
        g.set_option("compact_halo", args.compact)
        for kv in args.opt:
            k, v = kv.split("=")
            g.set_option(k, int(v))
        spec = cf.LatticeSpec(512, 512, args.lz * P, disorder=0.5, seed=1)
        As = g.topological_insulator(spec)
        p = cf.make_filter((-0.3, 0.3), (-5.6, 5.6), args.deg, "lanczos2")
        Xs = [cf.BlockVector(A, args.nb).randomize_device(7 + r) for r, A in enumerate(As)]
        g.apply_filter(As, Xs, p)  # capture
        c0 = g.ranks[0]
        c0.synchronize()
        c0.record(0)
        for _ in range(args.reps):
            g.apply_filter(As, Xs, p)
        c0.record(1)
        ms = c0.elapsed_ms(0, 1) / args.reps / args.deg
        halo = [cf.VirtualGroup.halo_rows(A) for A in As]
        halo_bytes = sum(h["halo_lo"] + h["halo_hi"] for h in halo) * args.nb * 16
        if P == 1:
            t1 = ms
        print(json.dumps({"ranks": P, "lattice": [512, 512, args.lz * P], "nb": args.nb,
                          "deg": args.deg, "ms_per_step": round(ms, 4),
                          "ms_per_step_per_rank": round(ms / P, 4),
                          "schedule_efficiency": round(P * t1 / ms, 4) if t1 else None,
                          "halo_bytes_per_step": halo_bytes, "compact": bool(args.compact),
                          "band_launches": sum(c.band_launches for c in g.ranks)}), flush=True)
        for X in Xs:
            X.close()
        g.close()


if __name__ == "__main__":
    main()
