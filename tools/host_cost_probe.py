"""Host cost per API call (eager path), S=512 int32: no-op grow, allocating
grow, duplicate insert, commit -- microseconds of host time per call."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S = int(os.environ.get("PROBE_S", "512"))
a = gg.GrowableArray(S, 32, dtype=np.int32)
a.insert_csr(torch.arange(1 << 16, dtype=torch.int32, device="cuda"),
             np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64((1 << 16) // S), 1 << 16))
torch.cuda.synchronize()
res = {}


def tm(name, fn, n=300, reset=None):
    ts = []
    for _ in range(n):
        if reset:
            reset()
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    torch.cuda.synchronize()
    res[name] = round(1e6 * float(np.median(ts)), 2)


n0 = a.committed_size
tm("grow_noop", lambda: a.grow(n0))
half = np.full(S, (1 << 16) // S, np.uint64)
tm("grow_alloc_512_buckets", lambda: a.grow(4 * n0), reset=lambda: a.shrink(half, release=False))
tm("insert_duplicate", lambda: a.insert_duplicate(), reset=lambda: a.shrink(half, release=False))
tm("commit", lambda: a.commit())
tm("shrink_cached", lambda: a.shrink(half, release=False))
tm("committed_size", lambda: a.committed_size)
from paper_2209_00103_b200 import _lib
st = a._stream()
cap = np.full(S, 4 * n0 // S, np.uint64)
fa = __import__("ctypes").c_int64(-1)
tm("raw_gg_reserve_noop", lambda: _lib.lib.gg_reserve(a._h, _lib.ptr(np.full(S, 1, np.uint64)), __import__("ctypes").byref(fa), st))
tm("raw_gg_commit", lambda: _lib.lib.gg_commit(a._h, st))
res["S"] = S
print(json.dumps(res))
