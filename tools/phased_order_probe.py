"""Config 4 (bench.phased_leg) under the three release policies, run
repeatedly in one process in the order 2.0, True, 2.0, True, False, 2.0: is
the default policy's occasional 150-730 ms of cuMemUnmap time a property of
the policy, of the box, or of being the first VMM-heavy run in the process?
Per run: wall ms, map / unmap ms from slab_stats, and the five slowest
shrink calls (wall, with the unmap time inside each)."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_00103_b200 as gg

S, FB = 512, 32
dev = torch.device("cuda", 0)
n0, cap_elems = 1 << 26, 1 << 28
src = torch.arange(cap_elems, dtype=torch.int32, device=dev)
split = lambda n: np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(-(-n // S)), np.uint64(n))


def run(release):
    rng = np.random.default_rng(0)
    a = gg.GrowableArray(S, FB, dtype=np.int32, device=dev)
    a.insert_csr(src[:n0], split(n0))
    n = n0
    sl0 = a.slab_stats()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    slow = []
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
        else:
            u0 = a.slab_stats()["unmap_ns"]
            c0 = time.perf_counter()
            a.shrink(new, release=release)
            slow.append((round((time.perf_counter() - c0) * 1e3, 3), round((a.slab_stats()["unmap_ns"] - u0) / 1e6, 3), r))
        n = target
        a.memory_stats()
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    sl = a.slab_stats()
    a.close()
    gg.reclaim(True)
    slow.sort(reverse=True)
    return {"release": str(release), "ms": round(ms, 2),
            "map_ms": round((sl["map_ns"] - sl0["map_ns"]) / 1e6, 2),
            "unmap_ms": round((sl["unmap_ns"] - sl0["unmap_ns"]) / 1e6, 2),
            "unmapped": sl["chunks_unmapped"] - sl0["chunks_unmapped"],
            "slowest_shrinks_wall_unmap_round": slow[:5]}


out = [run(p) for p in (2.0, True, 2.0, True, False, 2.0)]
print(json.dumps(out))
