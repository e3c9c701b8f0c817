"""get_many / set_many (batched get_global / set_global,
sharded_array.py:152-158) at 2^24 random global indices on a config-2-sized
GGArray (512 LFVectors, 2^30 int32), next to the same random gather /
scatter on a flat 2^30 tensor with torch (index_select / index_put_): the
random-access reference for the same index stream.  Contents checked
against the flattened array.  CUDA events, best of 5."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_00103_b200 as gg

dev = torch.device("cuda", 0)
S, FB, N0 = 512, 32, 1 << 20
a = gg.GrowableArray.from_flat(torch.arange(N0, dtype=torch.int32, device=dev), S, FB)
for _ in range(10):
    a.grow(2 * a.committed_size)
    a.insert_duplicate()
n = a.committed_size
flat = a.flatten_device()
NI = 1 << 24
g = torch.Generator(device=dev).manual_seed(5)
idx = torch.randint(0, n, (NI,), dtype=torch.int64, device=dev, generator=g)


def best(fn, reps=5):
    ms = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ms = min(ms, e0.elapsed_time(e1))
    return ms


out = {"indices": NI, "elements": n}
got = a.get_many(idx)
out["get_ok"] = bool(torch.equal(got, flat[idx]))
ms = best(lambda: a.get_many(idx))
out["get_many"] = {"ms": round(ms, 4), "gelem_s": round(NI / ms / 1e6, 2)}
ms = best(lambda: torch.index_select(flat, 0, idx))
out["torch_flat_gather"] = {"ms": round(ms, 4), "gelem_s": round(NI / ms / 1e6, 2)}
vals = torch.arange(NI, dtype=torch.int32, device=dev)
uidx = torch.unique(idx)                          # distinct targets: deterministic contents
uv = vals[:uidx.numel()]
a.set_many(uidx, uv)
chk = flat.clone()
chk[uidx] = uv
out["set_ok"] = bool(torch.equal(a.flatten_device(), chk))
ms = best(lambda: a.set_many(idx, vals))
out["set_many"] = {"ms": round(ms, 4), "gelem_s": round(NI / ms / 1e6, 2)}
ms = best(lambda: flat.index_put_((idx,), vals))
out["torch_flat_scatter"] = {"ms": round(ms, 4), "gelem_s": round(NI / ms / 1e6, 2)}
print(json.dumps(out))
