"""Where a kernel's warps wait and what they issue, from an `ncu --set full --import-source on`
report: the per-issue stall breakdown (raw page), the executed-instruction mix by opcode and
the most-sampled SASS instructions with their dominant stall reasons (source page).

    python tools/ncu_stalls.py REPORT.ncu-rep OUT.json [--launch -1] [--top 25] [--note TEXT]
"""
import argparse
import collections
import csv
import io
import json
import subprocess


def page(report, name, extra=()):
    out = subprocess.run(["ncu", "-i", report, "--page", name, "--csv", *extra], check=True,
                         capture_output=True, text=True).stdout
    return list(csv.reader(io.StringIO(out)))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("out")
    ap.add_argument("--launch", type=int, default=-1)
    ap.add_argument("--top", type=int, default=25)
    ap.add_argument("--note", default="")
    args = ap.parse_args()
    raw = page(args.report, "raw")
    hdr, data = raw[0], raw[2:]
    row = data[args.launch]
    col = {k: i for i, k in enumerate(hdr)}
    keep = ["gpu__time_duration.sum", "smsp__inst_executed.sum",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__average_warp_latency_per_inst_issued.ratio",
            "smsp__warps_eligible.avg.per_cycle_active",
            "sm__warps_active.avg.pct_of_peak_sustained_active",
            "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "dram__bytes_read.sum", "dram__bytes_write.sum", "launch__registers_per_thread"]
    rec = {"report": args.report, "note": args.note, "kernel": row[col["Kernel Name"]],
           "units": {k: raw[1][col[k]] for k in keep if k in col},
           "metrics": {k: float(row[col[k]].replace(",", "")) for k in keep if k in col}}
    stalls = {}
    for k, i in col.items():
        if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio") \
                and "not_issued" not in k:
            stalls[k[len("smsp__average_warps_issue_stalled_"):-len("_per_issue_active.ratio")]] = \
                round(float(row[i]), 4)
    rec["warps_stalled_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1]))
    src = page(args.report, "source", ("--print-source", "sass"))
    secs = [i for i, r in enumerate(src) if r and r[0] == "Kernel Name"]
    nl = len(secs)
    li = args.launch % nl
    shdr = src[secs[li] + 1]
    body = src[secs[li] + 2:secs[li + 1]] if li + 1 < nl else src[secs[li] + 2:]
    ix = {k: i for i, k in enumerate(shdr)}
    ex, sm = ix["Instructions Executed"], ix["# Samples"]

    def opcode(r):
        op = r[1].strip().split()
        if op and op[0].startswith("@"):
            op = op[1:]
        return op[0].split(".")[0] if op else "?"

    mix = collections.Counter()
    for r in body:
        mix[opcode(r)] += int(r[ex])
    tot = sum(mix.values())
    rec["sass_instructions"] = len(body)
    rec["executed_warp_instructions"] = tot
    rec["opcode_mix_pct"] = {o: round(100.0 * n / tot, 2) for o, n in mix.most_common(16)}
    stot = sum(int(r[sm]) for r in body)
    names = [k for k in shdr if k.startswith("stall_") and "Not Issued" not in k]
    top = sorted(range(len(body)), key=lambda i: -int(body[i][sm]))[:args.top]
    rec["samples"] = stot
    rec["top_sampled"] = []
    for i in sorted(top):
        r = body[i]
        st = sorted(((k, int(r[ix[k]])) for k in names), key=lambda kv: -kv[1])[:2]
        rec["top_sampled"].append({"index": i, "sass": r[1].strip(), "pct_samples": round(100.0 * int(r[sm]) / stot, 2),
                                   "stalls": {k: v for k, v in st if v}})
    json.dump(rec, open(args.out, "w"), indent=1)
    print(json.dumps({"kernel_ms": rec["metrics"].get("gpu__time_duration.sum"),
                      "stalls": rec["warps_stalled_per_issue"], "mix": rec["opcode_mix_pct"]}))


if __name__ == "__main__":
    main()
