"""The growarray-bench two-phase GGArray candidate (bench_cli._two_phase_run)
phase by phase with the slab driver counters: where the insert / rebuild
time goes at insertion multipliers 1, 3 and 10 (512 LFVectors, 2^26 final)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_00103_b200 as gg
from paper_2209_00103_b200.sharded_array import split_offsets

S, FB, FINAL, IT = 512, 32, 1 << 26, 6
out = {}


def t(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    r = fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3, r


for k in (1, 3, 10):
    for rep in range(2):
        start = max(1, FINAL // (1 + k) ** IT)
        a = gg.GrowableArray.from_flat(torch.arange(start, dtype=torch.int32, device="cuda"), S, FB)
        tag, rows = start, []
        for it in range(IT):
            size = a.committed_size
            m = FINAL - size if it == IT - 1 else min(k * size, FINAL - size)
            vals = torch.arange(tag, tag + m, dtype=torch.int32, device="cuda")
            tag += m
            s0 = a.slab_stats()
            chunk = -(-m // S)
            off = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(chunk), np.uint64(m))
            ins, _ = t(lambda: a.insert_csr(vals, off))
            s1 = a.slab_stats()
            fl, flat = t(lambda: a.flatten_device())
            rb, _ = t(lambda: (a.shrink(0, release=False), a.insert_csr(flat, split_offsets(int(flat.numel()), S))))
            s2 = a.slab_stats()
            rows.append({"it": it, "m": m, "insert_ms": round(ins, 3),
                         "insert_map_ms": round((s1["map_ns"] - s0["map_ns"]) / 1e6, 3),
                         "insert_chunks": s1["chunks_mapped"] - s0["chunks_mapped"],
                         "flatten_ms": round(fl, 3), "rebuild_ms": round(rb, 3),
                         "rebuild_map_ms": round((s2["map_ns"] - s1["map_ns"]) / 1e6, 3)})
        out[f"k{k}_rep{rep}"] = rows
        a.close()
        gg.reclaim(True)
print(json.dumps(out))
