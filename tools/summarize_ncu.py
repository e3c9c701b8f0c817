"""Summarise an evidence run (tools/profile_round.sh outputs in gpurun_out/) into
profiles/<tag>_*.  Usage: python tools/summarize_ncu.py r01"""
import csv
import json
import os
import shutil
import sys
from collections import defaultdict

tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
os.makedirs(P, exist_ok=True)

# launch list: per-kernel share of one bench step
rows, hdr = [], None
for r in csv.reader(open(os.path.join(src, "launches.csv"))):
    if r and r[0] == "ID":
        hdr = r
    elif hdr and len(r) == len(hdr):
        rows.append(dict(zip(hdr, r)))
agg = defaultdict(lambda: [0, 0.0])
for d in rows:
    k = d["Kernel Name"].split("(")[0]
    agg[k][0] += 1
    agg[k][1] += float(d["Metric Value"]) / 1e3
tot = sum(v[1] for v in agg.values())
launch_table = [{"kernel": k, "launches": v[0], "us": round(v[1], 1), "share": round(v[1] / tot, 4)}
                for k, v in sorted(agg.items(), key=lambda x: -x[1][1])]
shutil.copy(os.path.join(src, "launches.csv"), os.path.join(P, f"{tag}_launches.csv"))

# full capture: per profiled kernel
raw = list(csv.reader(open(os.path.join(src, "prof_raw.csv"))))
h = raw[0]
want = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size",
        "launch__block_size", "launch__registers_per_thread", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__warp_issue_stalled_long_scoreboard_per_warp_active.pct", "lts__t_sector_hit_rate.pct"]
units = dict(zip(h, raw[1]))
labels = ["dup insert 2^29 -> 2^30 (k_walk W_DUP)", "r/w +1 per shard 2^30 (k_walk W_RW)",
          "r/w +1 global rw_g 2^30 (k_rw_global)", "flatten 2^30 (k_walk W_FLATTEN)",
          "insert CSR 2^28 from flat batch (k_walk W_INSERT)"]
algo = [8 * (1 << 29), 8 * (1 << 30), 8 * (1 << 30), 8 * (1 << 30), 8 * (1 << 28)]
kern = []
for i, row in enumerate(raw[2:]):
    d = dict(zip(h, row))
    e = {"label": labels[i] if i < len(labels) else "?", "kernel": d["Kernel Name"].split("(")[0]}
    for k in want:
        if k in d:
            e[k + " [" + units.get(k, "") + "]"] = d[k]
    ms = float(d["gpu__time_duration.sum"]) if units["gpu__time_duration.sum"] == "ms" else float(d["gpu__time_duration.sum"]) / 1e3
    rd = float(d["dram__bytes_read.sum"]) * (1e9 if units["dram__bytes_read.sum"] == "Gbyte" else 1e6)
    wr = float(d["dram__bytes_write.sum"]) * (1e9 if units["dram__bytes_write.sum"] == "Gbyte" else 1e6)
    if i < len(algo):
        e["algorithmic_bytes"] = algo[i]
        e["traffic_bytes"] = int(rd + wr)
        e["traffic_over_algorithmic"] = round((rd + wr) / algo[i], 4)
        e["ncu_gbs_algorithmic"] = round(algo[i] / (ms * 1e-3) / 1e9, 1)
    kern.append(e)
summary = {"tag": tag, "launch_list_one_bench_step": launch_table, "full_capture": kern}
json.dump(summary, open(os.path.join(P, f"{tag}_ncu_summary.json"), "w"), indent=1)
with open(os.path.join(P, f"{tag}_ncu_summary.md"), "w") as fh:
    fh.write(f"# ncu evidence {tag}\n\nLaunch list of one bench step (`ncu --metrics gpu__time_duration.sum "
             "--clock-control none`, cold-cache and serialised: compare shares):\n\n| kernel | launches | us | share |\n|---|---|---|---|\n")
    for r in launch_table:
        fh.write(f"| `{r['kernel']}` | {r['launches']} | {r['us']} | {100 * r['share']:.1f}% |\n")
    fh.write("\nFull capture (`ncu --set full`, tools/prof_target.py):\n\n")
    for e in kern:
        fh.write(f"## {e['label']}\n\n")
        for k, v in e.items():
            if k != "label":
                fh.write(f"- {k}: {v}\n")
        fh.write("\n")
print(json.dumps(summary, indent=1)[:3000])
