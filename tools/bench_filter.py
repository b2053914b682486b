"""GPU bench front end: the reference CLI's `chebfd bench` (chebfd.cpp:326-357)
over chebfd_bench_filter -- block-size sweep, text table on stdout and
bench_report.json in the reference's schema.

    python tools/bench_filter.py --model ti --lattice 64 64 64 --degree 100 \
        --block-sizes 1 2 4 8 16 32 [--bandwidth 0] [--out gpurun_out/bench_report.json]
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
    ap.add_argument("--model", default="ti", choices=["ti", "graphene"])
    ap.add_argument("--lattice", type=int, nargs="+", default=[64, 64, 64])
    ap.add_argument("--disorder", type=float, default=0.5)
    ap.add_argument("--seed", type=int, default=1)
    ap.add_argument("--boundary", default=None)
    ap.add_argument("--degree", type=int, default=100)
    ap.add_argument("--block-sizes", type=int, nargs="+", default=[1, 2, 4, 8, 16, 32])
    ap.add_argument("--bandwidth", type=float, default=0.0, help="GB/s; 0 = run the probe")
    ap.add_argument("--out", default="bench_report.json")
    args = ap.parse_args()
    ctx = cf.Context(0)
    l = args.lattice
    kw = dict(disorder=args.disorder, seed=args.seed)
    if args.boundary:
        kw["boundary"] = args.boundary
    if args.model == "ti":
        A = cf.SparseMatrix.topological_insulator(ctx, cf.LatticeSpec(l[0], l[1], l[2], **kw))
    else:
        A = cf.SparseMatrix.graphene(ctx, cf.LatticeSpec(l[0], l[1], **kw))
    rep = cf.bench_filter(A, args.block_sizes, args.degree, args.bandwidth)
    print(rep.table())
    with open(args.out, "w") as f:
        json.dump(rep.to_json(), f, indent=2)


if __name__ == "__main__":
    main()
