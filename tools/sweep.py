"""Sweep the streaming-kernel unroll (tile = 256 threads x U x 16 B, one tile
per CTA) on the config-2/3 state: duplicate-insert of the last doubling round
(2^29 -> 2^30), flatten of 2^30, and one +1 pass over 2^30."""
import json
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg
from paper_2209_00103_b200 import _lib

S, FB = 512, 32
a = gg.GrowableArray.from_flat(torch.arange(1 << 20, dtype=torch.int32, device="cuda"), S, FB)
for _ in range(9):
    a.grow(2 * a.committed_size)
    a.insert_duplicate()
a.grow(2 * a.committed_size)
half = np.full(S, 1 << 20, np.uint64)
out = torch.empty(1 << 30, dtype=torch.int32, device="cuda")


def ev():
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


def t_dup(reps=5):
    ts = []
    for _ in range(reps):
        e0, e1 = ev()
        e0.record(); a.insert_duplicate(commit=False); e1.record()
        a.shrink(half, release=False)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def t_op(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = ev()
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


# reference: torch copy of 2 GiB -> 2 GiB
x = torch.empty(1 << 29, dtype=torch.int32, device="cuda"); y = torch.empty_like(x)
ms = t_op(lambda: y.copy_(x))
print(json.dumps({"ref": "torch copy 2^29 int32", "ms": ms, "gbs": 8 * (1 << 29) / ms / 1e6}), flush=True)
del x, y
a.insert_duplicate()          # state at 2^30 for flatten / rw
full = np.full(S, 1 << 21, np.uint64)
res = []
for un in [1, 2, 4, 8]:
    _lib.check(_lib.lib.gg_set_tuning(-1, un, 0, 0))
    a.shrink(half, release=False)
    d = t_dup()
    a.insert_duplicate()
    f = t_op(lambda: a.flatten_device(out=out))
    r = t_op(lambda: a.rw_add(1))
    g = t_op(lambda: a.rw_add(1, mode="global"))
    row = {"unroll": un, "tile_bytes": un * 256 * 16,
           "dup_gbs": round(8 * (1 << 29) / d / 1e6, 1), "flatten_gbs": round(8 * (1 << 30) / f / 1e6, 1),
           "rw_gbs": round(8 * (1 << 30) / r / 1e6, 1), "rw_global_gbs": round(8 * (1 << 30) / g / 1e6, 1)}
    res.append(row)
    print(json.dumps(row), flush=True)
_lib.lib.gg_set_tuning(-1, -1, 0, 0)
for k in ("dup_gbs", "flatten_gbs", "rw_gbs"):
    best = max(res, key=lambda r: r[k])
    print("best", k, json.dumps(best))
