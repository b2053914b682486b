"""Summarise an ncu report (--set full) into the committed profiles/*.json form.

    python tools/ncu_summary.py REPORT.ncu-rep OUT.json --lattice 512 512 8 --nb 64 \
        [--algorithmic BYTES] [--note TEXT]

Reads `ncu -i REPORT --page raw --csv` (first row names, second row units) and keeps
the counters the roofline and the latency diagnosis use, per captured launch, with
DRAM bytes converted to bytes."""
import argparse
import csv
import io
import json
import subprocess

KEEP = [
    "Kernel Name", "launch__grid_size", "launch__block_size", "launch__registers_per_thread",
    "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
    "sm__warps_active.avg.pct_of_peak_sustained_active",
    "smsp__issue_active.avg.pct_of_peak_sustained_active",
    "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
    "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
    "lts__t_sector_hit_rate.pct", "l1tex__t_sector_hit_rate.pct",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warp_latency_per_inst_issued.ratio",
    "smsp__inst_executed.sum", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
]
SCALE = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "Tbyte": 1e12,
         "nsecond": 1e-9, "usecond": 1e-6, "msecond": 1e-3, "second": 1.0,
         "ns": 1e-9, "us": 1e-6, "ms": 1e-3, "s": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--lattice", type=int, nargs=3, required=True)
    ap.add_argument("--nb", type=int, required=True)
    ap.add_argument("--algorithmic", type=float, default=None)
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", args.report, "--page", "raw", "--csv"], check=True,
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    names, units = rows[0], rows[1]
    launches = []
    for r in rows[2:]:
        d = {}
        for k in KEEP:
            if k not in names:
                continue
            i = names.index(k)
            v = r[i]
            try:
                x = float(v.replace(",", ""))
                u = units[i]
                if u in SCALE and ("bytes" in k or "duration" in k):
                    x *= SCALE[u]
                    k = k + (" [bytes]" if "bytes" in k else " [s]")
                d[k] = x
            except ValueError:
                d[k] = v
        launches.append(d)
    tr = [l.get("dram__bytes_read.sum [bytes]", 0) + l.get("dram__bytes_write.sum [bytes]", 0)
          for l in launches]
    out = {"lattice": args.lattice, "n_b": args.nb, "report": args.report, "note": args.note,
           "traffic_bytes": sum(tr) / len(tr), "algorithmic_bytes": args.algorithmic,
           "traffic_over_algorithmic": (sum(tr) / len(tr) / args.algorithmic)
           if args.algorithmic else None, "launches": launches}
    json.dump(out, open(args.out, "w"), indent=1)
    print(json.dumps({k: out[k] for k in ("traffic_bytes", "traffic_over_algorithmic")}))


if __name__ == "__main__":
    main()
