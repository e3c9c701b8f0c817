"""profiles/<tag>_atomics.{json,md} from gpurun_out/atomics.csv (tools/profile_round.sh)."""
import csv, json, os, sys
tag = sys.argv[1]
src = sys.argv[2] if len(sys.argv) > 2 else "gpurun_out"
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
labels = [("static insert, one atomicAdd per element (paper 3-B-1)", 1 << 26),
          ("static insert, one atomicAdd per warp (3-B-2)", 1 << 26),
          ("static insert, one atomicAdd per block (3-B-3 without tensor cores)", 1 << 26),
          ("device push_back, warp-aggregated (ggarray_device.cuh)", (1 << 24) * 2 // 3),
          ("device push_back, block-aggregated", (1 << 24) * 2 // 3),
          ("per-lane-count insert, one atomicAdd per LFVector (Alg. 1)", None)]
rows, hdr, per = list(csv.reader(open(os.path.join(src, "atomics.csv")))), None, {}
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        per.setdefault(int(d["ID"]), {"kernel": d["Kernel Name"].split("(")[0]})[d["Metric Name"]] = float(d["Metric Value"])
out = []
for i in sorted(per):
    e = per[i]
    lab, n = labels[i] if i < len(labels) else ("?", None)
    ns = e["gpu__time_duration.sum"]
    at = e.get("lts__t_requests_op_atom.sum", 0) + e.get("lts__t_requests_op_red.sum", 0)
    row = {"label": lab, "kernel": e["kernel"], "us": round(ns / 1e3, 2), "l2_atomic_requests": int(at),
           "atomics_per_s": round(at / (ns * 1e-9), 1)}
    if n:
        row["elements"] = n
        row["atomics_per_element"] = round(at / n, 5)
        row["gelem_s"] = round(n / ns, 3)
    out.append(row)
json.dump(out, open(os.path.join(ROOT, "profiles", f"{tag}_atomics.json"), "w"), indent=1)
with open(os.path.join(ROOT, "profiles", f"{tag}_atomics.md"), "w") as fh:
    fh.write(f"# L2 atomics {tag} (ncu, `--clock-control none`, tools/prof_atomics.py)\n\n")
    fh.write("| path | kernel | us | L2 atomic requests | per element | Gatomics/s | Gelem/s |\n|---|---|---|---|---|---|---|\n")
    for r in out:
        fh.write(f"| {r['label']} | `{r['kernel']}` | {r['us']} | {r['l2_atomic_requests']} | "
                 f"{r.get('atomics_per_element', '')} | {r['atomics_per_s'] / 1e9:.3f} | {r.get('gelem_s', '')} |\n")
print(json.dumps(out, indent=1))
