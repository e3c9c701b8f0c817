"""Fixed per-call cost of the device-view path (push_if's host prepare /
finish around the kernel) on a config-sized array (512 LFVectors, 2^28
elements already appended, reset with shrink(0, release=False)):
wall and event time of push_if at 2^10 .. 2^20 candidates, and the
device_view(max) + device_sync pair alone (no kernel)."""
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
out = {}
N = 1 << 28
vals = torch.arange(N, dtype=torch.int32, device=dev)
pred = torch.ones(N, dtype=torch.uint8, device=dev)
a = gg.GrowableArray(S, FB, dtype=np.int32)
a.push_if(vals, pred, commit=False)
for lg in (10, 16, 20):
    n = 1 << lg
    v, p = vals[:n], pred[:n]
    walls, evs = [], []
    for _ in range(20):
        a.shrink(0, release=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        t0 = time.perf_counter()
        e0.record()
        a.push_if(v, p, commit=False)
        e1.record()
        torch.cuda.synchronize()
        walls.append((time.perf_counter() - t0) * 1e3)
        evs.append(e0.elapsed_time(e1))
    out[f"push_if_2p{lg}"] = {"wall_ms": round(float(np.median(walls)), 4), "event_ms": round(float(np.median(evs)), 4)}
walls = []
for _ in range(20):
    a.shrink(0, release=False)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.device_view(max_sizes=(1 << 20) // S)
    t1 = time.perf_counter()
    a.device_sync()
    t2 = time.perf_counter()
    walls.append(((t1 - t0) * 1e3, (t2 - t1) * 1e3))
w = np.median(np.array(walls), axis=0)
out["view_get_ms"], out["view_sync_ms"] = round(float(w[0]), 4), round(float(w[1]), 4)
walls = []
for _ in range(20):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    a.shrink(0, release=False)
    torch.cuda.synchronize()
    walls.append((time.perf_counter() - t0) * 1e3)
out["shrink0_ms"] = round(float(np.median(walls)), 4)
print(json.dumps(out))
