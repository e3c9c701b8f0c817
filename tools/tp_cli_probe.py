import json, os, sys
sys.path.insert(0, os.getcwd())
import torch
import paper_2209_00103_b200 as gg
from paper_2209_00103_b200 import bench_cli as B
cfg = B.BenchConfig(shards=512, initial_size=1 << 20, iterations=6, work_passes=10, repetitions=1)
final = B._check_final_size(cfg) if hasattr(B, "_check_final_size") else (1 << 20) * 2 ** 6
for k in (10,):
    start = max(1, final // (1 + k) ** cfg.iterations)
    for rep in range(3):
        for kind in ("chunktable", "ggarray"):
            p0 = gg.pool_stats(0)
            phases, total, end = B._two_phase_run(cfg, kind, start, k, final)
            p1 = gg.pool_stats(0)
            print(kind, rep, round(total / 1e6, 2), [(p["iteration"], p["phase"], round(p["elapsed_ns"] / 1e6, 2)) for p in phases if p["elapsed_ns"] > 500000],
                  "pool hits", p1["hits"] - p0["hits"], "misses", p1["misses"] - p0["misses"], "cached", p1["cached_bytes"] >> 20, "MiB")
