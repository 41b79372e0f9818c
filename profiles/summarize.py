"""Summarise ncu output into profiles/ (run here, after gpurun brought gpurun_out/ back).

    python profiles/summarize.py TAG [--launches gpurun_out/launches_TAG.csv]
                                     [--rep gpurun_out/prof_tc_TAG.ncu-rep]

Writes profiles/launches_TAG.md (per-kernel device time from the
`--metrics gpu__time_duration.sum --clock-control none` pass; cold-cache and serialised,
so compare SHARES) and profiles/ncu_TAG.md (+ .json) with the key counters of the
`--set full` capture (duration, DRAM bytes, tensor-pipe activity, stall mix).
"""
from __future__ import annotations

import argparse
import csv
import io
import json
import os
import re
import subprocess
from collections import defaultdict

HERE = os.path.dirname(os.path.abspath(__file__))
REPO = os.path.dirname(HERE)

RAW_KEYS = [
    "gpu__time_duration.sum",
    "dram__bytes_read.sum",
    "dram__bytes_write.sum",
    "sm__cycles_active.avg",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
    "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_elapsed",
    "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
    "lts__t_bytes.sum",
    "lts__t_sectors.sum",
    "lts__cycles_elapsed.avg",
    "launch__grid_size",
    "launch__cluster_dim_x",
    "launch__registers_per_thread",
    "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio",
    "smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio",
    "gpc__cycles_elapsed.max",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed",
]


def summarize_launches(path: str, tag: str) -> str:
    rows = list(csv.reader(open(path)))
    hdr = None
    agg = defaultdict(list)
    for r in rows:
        if "Kernel Name" in r:
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            d = dict(zip(hdr, r))
            if d.get("Metric Name") == "gpu__time_duration.sum":
                name = re.sub(r"\(.*", "", d["Kernel Name"]).strip()
                agg[name].append(float(d["Metric Value"].replace(",", "")) / 1e3)
    total = sum(sum(v) for v in agg.values())
    lines = [f"# ncu launch list — {tag}", "",
             "`ncu --metrics gpu__time_duration.sum --clock-control none` over "
             "`python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-e2e`.",
             "Cold-cache, serialised launches: compare shares, not absolutes.", "",
             "| kernel | launches | mean µs | total µs | share |", "|---|---|---|---|---|"]
    for name, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
        lines.append(f"| `{name[:90]}` | {len(v)} | {sum(v)/len(v):.2f} | {sum(v):.1f} | "
                     f"{sum(v)/total:.1%} |")
    return "\n".join(lines) + "\n"


def summarize_rep(path: str, tag: str):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True, check=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": re.sub(r"\(.*", "", r[hdr.index("Kernel Name")]).strip(),
             "id": r[hdr.index("ID")]}
        for k in RAW_KEYS:
            if k in hdr:
                d[k] = f"{r[hdr.index(k)]} {units[hdr.index(k)]}".strip()
        out.append(d)
    lines = [f"# ncu --set full — {tag}", ""]
    for d in out:
        lines.append(f"## launch {d['id']}: `{d['kernel'][:100]}`")
        for k in RAW_KEYS:
            if k in d:
                lines.append(f"- {k}: {d[k]}")
        lines.append("")
    return "\n".join(lines), out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("tag")
    ap.add_argument("--launches")
    ap.add_argument("--rep")
    a = ap.parse_args()
    go = os.path.join(REPO, "gpurun_out")
    launches = a.launches or os.path.join(go, f"launches_{a.tag}.csv")
    rep = a.rep or os.path.join(go, f"prof_tc_{a.tag}.ncu-rep")
    if os.path.exists(launches):
        with open(os.path.join(HERE, f"launches_{a.tag}.md"), "w") as f:
            f.write(summarize_launches(launches, a.tag))
    if os.path.exists(rep):
        md, data = summarize_rep(rep, a.tag)
        with open(os.path.join(HERE, f"ncu_{a.tag}.md"), "w") as f:
            f.write(md)
        with open(os.path.join(HERE, f"ncu_{a.tag}.json"), "w") as f:
            json.dump(data, f, indent=1)
    print("wrote", [f for f in os.listdir(HERE) if a.tag in f])


if __name__ == "__main__":
    main()
