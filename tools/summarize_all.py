"""Summarise the per-kernel ncu metrics pass over tools/prof_all.py into
profiles/<tag>_all_kernels.{json,md}: every gg:: launch with its leg, duration,
DRAM bytes (read + write) against the leg's algorithmic bytes, L2 atomic and
reduction requests, launch shape.

Usage: python tools/summarize_all.py r02 [gpurun_out]
"""
import csv
import json
import os
import sys
from collections import OrderedDict

tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
P = os.path.join(ROOT, "profiles")
peaks = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))) if os.path.exists(
    os.path.join(ROOT, "MEASURED_PEAKS.json")) else {}
HBM = float(peaks.get("hbm_gbs", 6548.5))
legs = json.load(open(os.path.join(src, "prof_all_legs.json")))

SCALE = {"byte": 1, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "ns": 1e-3, "us": 1, "usecond": 1,
         "msecond": 1e3, "ms": 1e3, "nsecond": 1e-3}

launches = OrderedDict()
hdr = None
for row in csv.reader(open(os.path.join(src, "prof_all.csv"))):
    if row and row[0] == "ID":
        hdr = row
        continue
    if not hdr or len(row) != len(hdr):
        continue
    d = dict(zip(hdr, row))
    k = launches.setdefault(d["ID"], {"name": d["Kernel Name"], "grid": d["Grid Size"],
                                      "block": d["Block Size"], "m": {}})
    v = d["Metric Value"].replace(",", "")
    try:
        v = float(v) * SCALE.get(d["Metric Unit"], 1)
    except ValueError:
        pass
    k["m"][d["Metric Name"]] = v


def short(name):
    n = name.split("(")[0]
    n = n.replace("void ", "").replace("gg::", "")
    return n


segs, cur = [], None
for k in launches.values():
    if "spin_kernel" in k["name"]:
        cur = []
        segs.append(cur)
    elif cur is not None:
        cur.append(k)

rows = []
for i, lg in enumerate(legs):
    if lg["label"] == "end":
        continue
    ks = segs[i] if i < len(segs) else []
    tot_us = sum(k["m"].get("gpu__time_duration.sum", 0) for k in ks)
    rd = sum(k["m"].get("dram__bytes_read.sum", 0) for k in ks)
    wr = sum(k["m"].get("dram__bytes_write.sum", 0) for k in ks)
    atom = sum(k["m"].get("lts__t_requests_op_atom.sum", 0) + k["m"].get("lts__t_requests_op_red.sum", 0)
               for k in ks)
    ab = lg["algorithmic_bytes"]
    r = {"leg": lg["label"], "note": lg["note"], "launches": [
        {"kernel": short(k["name"]), "grid": k["grid"], "block": k["block"],
         "us": round(k["m"].get("gpu__time_duration.sum", 0), 2),
         "dram_bytes": int(k["m"].get("dram__bytes_read.sum", 0) + k["m"].get("dram__bytes_write.sum", 0)),
         "l2_atomic_requests": int(k["m"].get("lts__t_requests_op_atom.sum", 0)),
         "l2_red_requests": int(k["m"].get("lts__t_requests_op_red.sum", 0)),
         "regs": k["m"].get("launch__registers_per_thread"),
         "dram_pct_peak": k["m"].get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed")}
        for k in ks],
        "us": round(tot_us, 2), "dram_bytes": int(rd + wr), "l2_atomics": int(atom),
        "algorithmic_bytes": ab}
    if ab and tot_us:
        r["algorithmic_gbs"] = round(ab / (tot_us * 1e-6) / 1e9, 1)
        r["frac_of_hbm"] = round(ab / (tot_us * 1e-6) / 1e9 / HBM, 4)
        r["traffic_over_algorithmic"] = round((rd + wr) / ab, 4)
    if lg["elements"] and tot_us:
        r["gelem_s"] = round(lg["elements"] / (tot_us * 1e-6) / 1e9, 2)
        if atom:
            r["atomics_per_element"] = round(atom / lg["elements"], 6)
    rows.append(r)

kernels = sorted({l["kernel"].split("<")[0] for r in rows for l in r["launches"]})
out = {"tag": tag, "hbm_peak_gbs": HBM, "source": "ncu --metrics (cold cache, serialised, --clock-control none) "
       "over tools/prof_all.py", "kernels_seen": kernels, "legs": rows}
os.makedirs(P, exist_ok=True)
json.dump(out, open(os.path.join(P, f"{tag}_all_kernels.json"), "w"), indent=1)
with open(os.path.join(P, f"{tag}_all_kernels.md"), "w") as fh:
    fh.write(f"# Every library kernel under ncu ({tag})\n\n`ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,"
             "dram__bytes_write.sum,lts__t_requests_op_atom.sum,lts__t_requests_op_red.sum,... --clock-control none` "
             "over `tools/prof_all.py` (one leg per public operation; cold L2, serialised launches, so per-launch "
             f"times run above the warm bench's). HBM peak {HBM} GB/s (MEASURED_PEAKS.json). "
             "Algorithmic bytes per leg: see the note column and DESIGN.md section 3.\n\n")
    fh.write(f"Kernels seen ({len(kernels)}): " + ", ".join(f"`{k}`" for k in kernels) + "\n\n")
    fh.write("| leg | kernels (launches) | us | algorithmic B | DRAM B | DRAM / algo | GB/s (algo) | frac | Gelem/s | L2 atomics |\n"
             "|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        kn = {}
        for l in r["launches"]:
            b = l["kernel"].split("<")[0]
            kn[b] = kn.get(b, 0) + 1
        ks = ", ".join(f"`{k}`×{v}" for k, v in kn.items())
        fh.write(f"| {r['leg']} | {ks} | {r['us']} | {r['algorithmic_bytes'] or '—'} | {r['dram_bytes']} | "
                 f"{r.get('traffic_over_algorithmic', '—')} | {r.get('algorithmic_gbs', '—')} | "
                 f"{r.get('frac_of_hbm', '—')} | {r.get('gelem_s', '—')} | {r['l2_atomics']} |\n")
    fh.write("\n## Per launch\n\n| leg | kernel | grid | block | regs | us | DRAM B | DRAM % peak | L2 atom | L2 red |\n"
             "|---|---|---|---|---|---|---|---|---|---|\n")
    for r in rows:
        for l in r["launches"]:
            fh.write(f"| {r['leg'][:48]} | `{l['kernel'][:70]}` | {l['grid']} | {l['block']} | {l['regs']} | "
                     f"{l['us']} | {l['dram_bytes']} | {l['dram_pct_peak']} | {l['l2_atomic_requests']} | "
                     f"{l['l2_red_requests']} |\n")
print(json.dumps({"kernels_seen": kernels, "legs": len(rows)}, indent=1))

# --set full captures of the non-uniform paths (prof_paths_raw.csv), if present
fp = os.path.join(src, "prof_paths_raw.csv")
if os.path.exists(fp):
    raw = list(csv.reader(open(fp)))
    h, units = raw[0], dict(zip(raw[0], raw[1]))
    want = [("gpu__time_duration.sum", "duration"), ("dram__bytes_read.sum", "DRAM read"),
            ("dram__bytes_write.sum", "DRAM write"),
            ("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "DRAM % of peak"),
            ("sm__warps_active.avg.pct_of_peak_sustained_active", "warps active %"),
            ("launch__registers_per_thread", "regs"),
            ("smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio", "long-scoreboard warps per issue"),
            ("smsp__average_warps_issue_stalled_barrier_per_issue_active.ratio", "barrier warps per issue"),
            ("lts__t_sector_hit_rate.pct", "L2 hit %"), ("launch__grid_size", "grid")]
    full = []
    for row in raw[2:]:
        d = dict(zip(h, row))
        full.append({"kernel": short(d["Kernel Name"]),
                     **{lab: f"{d.get(k, '')} {units.get(k, '')}".strip() for k, lab in want}})
    out["paths_full_capture"] = full
    json.dump(out, open(os.path.join(P, f"{tag}_all_kernels.json"), "w"), indent=1)
    with open(os.path.join(P, f"{tag}_all_kernels.md"), "a") as fh:
        fh.write("\n## `ncu --set full` of the non-uniform paths (tools/prof_all.py, "
                 "kernels k_walk_shard / k_lanes_chunk / k_push_if / k_flat_insert_block / k_flat_append / k_gather)\n\n")
        fh.write("| kernel | " + " | ".join(l for _, l in want) + " |\n|" + "---|" * (len(want) + 1) + "\n")
        for e in full:
            fh.write(f"| `{e['kernel'][:60]}` | " + " | ".join(e[l] for _, l in want) + " |\n")
