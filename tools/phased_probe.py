"""Config 4 (phased random insert / shrink) round by round: op, target,
needed / capacity / mapped bytes, slab counters -- to see where the mapped
footprint departs from 2x needed under a release policy (argv[1], default 2.0)."""
import json
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2209_00103_b200 as gg  # noqa: E402

S, FB = 512, 32
release = {"True": True, "False": False}.get(sys.argv[1], None) if len(sys.argv) > 1 else None
release = float(sys.argv[1]) if release is None and len(sys.argv) > 1 else (2.0 if release is None else release)
n0, cap_elems = 1 << 26, 1 << 28
src = torch.arange(cap_elems, dtype=torch.int32, device="cuda")
rng = np.random.default_rng(0)
a = gg.GrowableArray(S, FB, dtype=np.int32)
a.insert_csr(src[:n0], np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(n0 // S), n0))
n = n0
for r in range(100):
    target = int(min(cap_elems, round(rng.uniform(0, 2) * n0)))
    q, rem = divmod(target, S)
    new = np.full(S, q, np.int64)
    new[:rem] += 1
    cur = a._host()["sizes"].astype(np.int64)
    if target >= n:
        delta = new - cur
        off = np.concatenate([[0], np.cumsum(delta)]).astype(np.uint64)
        a.insert_csr(src[:int(off[-1])], off)
        op = "insert"
    else:
        a.shrink(new, release=release)
        op = "shrink"
    n = target
    ms = a.memory_stats()
    sl = a.slab_stats()
    print(json.dumps({"r": r, "op": op, "target": target, "rem": rem,
                      "mapped_over_needed": round(ms["mapped_bytes"] / max(1, ms["needed_bytes"]), 3),
                      "mapped_mib": ms["mapped_bytes"] >> 20, "cached_mib": ms["cached_bytes"] >> 20,
                      "cap_mib": ms["capacity_bytes"] >> 20, "need_mib": ms["needed_bytes"] >> 20,
                      "pending": ms["pending_unmap_bytes"], "extents": sl["chunks_mapped"],
                      "unmapped": sl["chunks_unmapped"]}))
