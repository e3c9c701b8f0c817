"""Does the L2 fetch granularity bound the random gather / scatter?

get_many / set_many (2^24 random global indices on a config-2 GGArray, as
tools/gather_probe.py) and torch's flat index_select / index_put_ on the
same index stream, under cudaLimitMaxL2FetchGranularity = default / 32 / 64 /
128 B (a context-wide hint: how many bytes L2 fetches from DRAM on a miss).
ncu of the gather reported ~137 DRAM bytes per random 4 B element
(profiles/r02_all_kernels.md); if that is the fetch granularity, 32 B cuts
it.  CUDA events, best of 5.  GG_PROBE_ONE=<gran> runs one gather only (for
an ncu capture of the DRAM bytes)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from cuda.bindings import runtime as rt

import paper_2209_00103_b200 as gg

dev = torch.device("cuda", 0)
torch.cuda.init()
LIM = rt.cudaLimit.cudaLimitMaxL2FetchGranularity


def get_lim():
    err, v = rt.cudaDeviceGetLimit(LIM)
    return int(v)


def set_lim(v):
    (err,) = rt.cudaDeviceSetLimit(LIM, v)
    return str(err)


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
vals = torch.arange(NI, dtype=torch.int32, device=dev)


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
    return round(ms, 4)


one = os.environ.get("GG_PROBE_ONE")
if one is not None:
    if int(one):
        set_lim(int(one))
    a.get_many(idx)
    a.set_many(idx, vals)
    torch.cuda.synchronize()
    print(json.dumps({"gran": get_lim()}))
    sys.exit(0)

out = {"indices": NI, "elements": n, "default_gran": get_lim(), "runs": []}
ref = flat[idx]
for gran in [0, 32, 64, 128, 32]:
    r = {"requested": gran}
    if gran:
        r["set"] = set_lim(gran)
    r["gran"] = get_lim()
    r["get_ok"] = bool(torch.equal(a.get_many(idx), ref))
    r["get_many_ms"] = best(lambda: a.get_many(idx))
    r["torch_gather_ms"] = best(lambda: torch.index_select(flat, 0, idx))
    r["set_many_ms"] = best(lambda: a.set_many(idx, vals))
    r["torch_scatter_ms"] = best(lambda: flat.index_put_((idx,), vals))
    out["runs"].append(r)
print(json.dumps(out))
