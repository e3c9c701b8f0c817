"""Where the first config-2 step of a fresh array in a fresh process spends
its wall time: every API call of the step synchronised and timed on the
host, with the slab driver counters beside it.  Run twice in one process
(fresh array each time, pool trimmed before the first) and under
CUDA_MODULE_LOADING=EAGER to separate lazy kernel loading from driver
mapping."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

t_imp = time.perf_counter()
import paper_2209_00103_b200 as gg  # noqa: E402

S, FB, N0, ROUNDS = 512, 32, 1 << 20, 10
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
torch.zeros(1, device=dev)
out = {"module_loading": os.environ.get("CUDA_MODULE_LOADING", "default(lazy)"),
       "import_ms": round((time.perf_counter() - t_imp) * 1e3, 2)}


def timed(fn):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    fn()
    torch.cuda.synchronize()
    return (time.perf_counter() - t0) * 1e3


gg.pool_trim(0)
for trial in ("first", "second"):
    rec = {}
    vals = torch.arange(N0, dtype=torch.int32, device=dev)
    off = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(N0 // S), N0)
    arr = [None]
    rec["construct_ms"] = round(timed(lambda: arr.__setitem__(0, gg.GrowableArray(S, FB, dtype=np.int32))), 3)
    a = arr[0]
    rec["reset_ms"] = round(timed(lambda: a.shrink(0, release=False)), 3)
    rec["insert_csr_ms"] = round(timed(lambda: a.insert_csr(vals, off)), 3)
    rounds = []
    for _ in range(ROUNDS):
        n = a.committed_size
        g = timed(lambda: a.grow(2 * n))
        d = timed(lambda: a.insert_duplicate())
        rounds.append((round(g, 3), round(d, 3)))
    rec["rounds_grow_dup_ms"] = rounds
    rec["step_ms"] = round(rec["reset_ms"] + rec["insert_csr_ms"] + sum(g + d for g, d in rounds), 3)
    sl = a.slab_stats()
    rec["map_ms"] = round(sl["map_ns"] / 1e6, 3)
    rec["slab"] = {k: sl[k] for k in ("chunks_mapped", "handles_created", "handles_from_pool") if k in sl}
    rec["warm_step_ms"] = round(timed(lambda: (a.shrink(0, release=False), a.insert_csr(vals, off),
                                               [(a.grow(2 * a.committed_size), a.insert_duplicate())
                                                for _ in range(ROUNDS)])), 3)
    out[trial] = rec
    a.close()
    del a, arr
    gg.reclaim(True)
    if trial == "first":
        gg.pool_trim(0)
print(json.dumps(out))
