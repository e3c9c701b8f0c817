"""Per-path probe outputs of the evidence run (tools/evidence_r02.sh ->
gpurun_out/probes/*.json) -> profiles/<round>_probes.json + .md.

Usage: python tools/summarize_probes.py r02 [gpurun_out]"""
import json
import os
import sys

rnd = sys.argv[1] if len(sys.argv) > 1 else "r02"
src = os.path.join(sys.argv[2] if len(sys.argv) > 2 else "gpurun_out", "probes")
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
data = {}
for f in sorted(os.listdir(src)):
    if not f.endswith(".json"):
        continue
    txt = open(os.path.join(src, f)).read().strip().splitlines()
    try:
        data[f[:-5]] = json.loads(txt[-1])
    except (IndexError, json.JSONDecodeError):
        data[f[:-5]] = {"error": "no JSON output"}
json.dump(data, open(os.path.join(ROOT, "profiles", f"{rnd}_probes.json"), "w"), indent=1)

L = [f"# {rnd} per-path probes (one B200, CUDA events around the public call, "
     "host planning inside; best of 5)", ""]
pk = data.get("push_if_probe", {})
if pk:
    L += ["## push_if (device push_back API, 2^28 candidates, 512 LFVectors, density 1/2 unless noted)",
          "", "Bytes = values + predicates read + kept values written.", "",
          "| config | ms | GB/s | frac of HBM | Gelem/s appended | multiset ok |", "|---|---|---|---|---|---|"]
    for k, v in pk.items():
        if isinstance(v, dict):
            L.append(f"| {k} | {v['ms']} | {v['gbs']} | {v['frac']} | {v['gelem_s']} | {v['multiset_ok']} |")
    L.append("")
lp = data.get("lanes_probe", {})
if lp:
    L += ["## insert_lanes (paper Alg. 1, per-lane counts uniform in [0, K], ~2^28 appended, 512 LFVectors)",
          "", "Bytes = counts (4 B / lane) + the [lanes x K] value block + the compacted output. "
          "`K{K}_e{element bytes}`.", "",
          "| config | lanes | appended | ms | GB/s | frac of HBM | contents ok |", "|---|---|---|---|---|---|---|"]
    for k, v in lp.items():
        if isinstance(v, dict) and "lanes" in v:
            L.append(f"| {k} | {v['lanes']} | {v['appended']} | {v['ms']} | {v['gbs']} | {v['frac']} | {v['contents_ok']} |")
    L.append("")
for name, title in (("lanes_host_probe", "insert_lanes host time per call (µs)"),
                    ("ragged_host_probe", "ragged insert / duplicate host time per call (µs)"),
                    ("view_cost_probe", "device-view path fixed cost")):
    d = data.get(name)
    if d:
        L += [f"## {title}", "", "```", json.dumps(d, indent=1), "```", ""]
gp = data.get("gather_probe")
if gp and "get_many" in gp:
    L += ["## get_many / set_many, 2^24 random global indices on a 2^30-element GGArray (512 LFVectors)", "",
          "Next to torch's index_select / index_put_ on the flat array with the same index stream (the "
          "random-access reference: each access costs a DRAM burst whatever the layout).", "",
          "| op | GGArray ms | Gelem/s | torch flat ms | Gelem/s | contents ok |", "|---|---|---|---|---|---|",
          f"| gather | {gp['get_many']['ms']} | {gp['get_many']['gelem_s']} | {gp['torch_flat_gather']['ms']} | "
          f"{gp['torch_flat_gather']['gelem_s']} | {gp['get_ok']} |",
          f"| scatter | {gp['set_many']['ms']} | {gp['set_many']['gelem_s']} | {gp['torch_flat_scatter']['ms']} | "
          f"{gp['torch_flat_scatter']['gelem_s']} | {gp['set_ok']} |", ""]
vm = data.get("vmm_fresh_probe")
if vm:
    L += ["## CUDA VMM cost in a fresh process (8 GiB, create + map + access, then unmap + release; "
          "runs in order)", "", "| chunk MiB | map total ms | cuMemCreate ms | release ms |", "|---|---|---|---|"]
    for r in vm if isinstance(vm, list) else []:
        L.append(f"| {r['chunk_mib']} | {r['map_total_ms']} | {r['create_ms']} | {r['release_ms']} |")
    L.append("")
open(os.path.join(ROOT, "profiles", f"{rnd}_probes.md"), "w").write("\n".join(L) + "\n")
print("\n".join(L))
