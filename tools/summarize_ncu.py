"""Summarise ncu captures into profiles/ (committed evidence).

    python tools/summarize_ncu.py --launches gpurun_out/launches_r1.csv \
        --full gpurun_out/prof_tma_r1.ncu-rep --out profiles/r01 \
        --algo-bytes 2915418112
"""
import argparse
import collections
import csv
import io
import json
import re
import subprocess

RAW_KEYS = [
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "l1tex__t_sector_hit_rate.pct", "sm__warps_active.avg.pct_of_peak_sustained_active",
    "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
    "smsp__inst_executed.sum", "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warp_latency_per_inst_issued.ratio", "lts__t_sectors_srcunit_tex_op_read.sum",
    "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "launch__shared_mem_per_block_dynamic",
]


def launches(path):
    text = open(path).read()
    start = text.find('"ID"')
    rows = list(csv.reader(io.StringIO(text[start:])))
    hdr = rows[0]
    ki = hdr.index("Kernel Name")
    vi = hdr.index("Metric Value")
    ui = hdr.index("Metric Unit")
    mi = hdr.index("Metric Name") if "Metric Name" in hdr else None
    per = collections.defaultdict(list)
    for r in rows[1:]:
        if len(r) <= vi:
            continue
        if mi is not None and r[mi] != "gpu__time_duration.sum":
            continue  # launch lists captured with extra metrics: durations only
        v = float(r[vi].replace(",", ""))
        if r[ui] == "ms":
            v *= 1e3
        elif r[ui] in ("nsecond", "ns"):
            v /= 1e3
        elif r[ui] in ("usecond", "us"):
            pass
        name = re.sub(r"\(.*", "", r[ki])[:90]
        per[name].append(v)
    tot = sum(sum(v) for v in per.values())
    out = []
    for name, v in sorted(per.items(), key=lambda kv: -sum(kv[1])):
        out.append({"kernel": name, "launches": len(v), "total_us": round(sum(v), 1),
                    "avg_us": round(sum(v) / len(v), 2), "share": round(sum(v) / tot, 4)})
    return out, tot


def raw(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(io.StringIO(txt)))
    hdr, units = rows[0], rows[1]
    res = []
    for r in rows[2:]:
        d = {"kernel": r[hdr.index("Kernel Name")]}
        for k in RAW_KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        res.append(d)
    return res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--launches")
    ap.add_argument("--full")
    ap.add_argument("--out", required=True)
    ap.add_argument("--algo-bytes", type=float, default=None)
    args = ap.parse_args()
    summary = {}
    if args.launches:
        lst, tot = launches(args.launches)
        summary["launch_list"] = {"total_us": round(tot, 1), "kernels": lst}
    if args.full:
        summary["full"] = raw(args.full)
        if args.algo_bytes:
            for d in summary["full"]:
                rd = float(d["dram__bytes_read.sum"].split()[0])
                wr = float(d["dram__bytes_write.sum"].split()[0])
                unit = d["dram__bytes_read.sum"].split()[1]
                scale = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1.0}[unit]
                d["traffic_bytes"] = (rd + wr) * scale
                d["algorithmic_bytes"] = args.algo_bytes
                d["traffic_over_algorithmic"] = round((rd + wr) * scale / args.algo_bytes, 4)
    json.dump(summary, open(args.out + ".json", "w"), indent=1)
    print(json.dumps(summary, indent=1)[:3000])


if __name__ == "__main__":
    main()
