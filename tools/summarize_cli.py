"""profiles/<tag>_bench_cli/SUMMARY.md from the growarray-bench-schema CSVs
(python -m paper_2209_00103_b200.bench_cli ... --out ...): last-iteration
medians over repetitions per structure / algo / phase."""
import csv, glob, os, statistics, sys
from collections import defaultdict

d = sys.argv[1] if len(sys.argv) > 1 else "profiles/r01_bench_cli"
out = ["# growarray-bench schema on one B200 (bench_cli.py)", "",
       "Medians over repetitions; `elapsed_ns` is host wall clock around CUDA-synchronised phases "
       "(the reference harness's clock), `gelem_s` / `hbm_gbs` the B200 columns.", ""]
for f in sorted(glob.glob(os.path.join(d, "*.csv"))):
    rows = list(csv.DictReader(open(f)))
    if not rows or "phase" not in rows[0]:
        continue
    out += [f"## {os.path.basename(f)}", "", "| structure | algo | variant | iteration | phase | size_after | elapsed_us | gelem_s | hbm_gbs |",
            "|---|---|---|---|---|---|---|---|---|"]
    g = defaultdict(list)
    for r in rows:
        g[(r["structure"], r["algo"], r["variant"], r["iteration"], r["phase"], r["size_after"])].append(r)
    last_it = max(int(r["iteration"]) for r in rows if r["iteration"].lstrip("-").isdigit())
    for k, rs in g.items():
        if k[3].lstrip("-").isdigit() and int(k[3]) != last_it and k[4] not in ("total",):
            continue
        med = lambda c: statistics.median(float(r[c]) for r in rs if r.get(c) not in (None, "")) if any(r.get(c) not in (None, "") for r in rs) else ""
        e = med("elapsed_ns")
        out.append(f"| {k[0]} | {k[1]} | {k[2]} | {k[3]} | {k[4]} | {k[5]} | {'' if e == '' else round(e / 1e3, 1)} | "
                   f"{med('gelem_s')} | {med('hbm_gbs')} |")
    out.append("")
open(os.path.join(d, "SUMMARY.md"), "w").write("\n".join(out) + "\n")
print("\n".join(out[:40]))
