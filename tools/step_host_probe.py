"""Host time of each API call inside one config-2 step (op by op), median over
20 steps, next to the GPU time of the same op: where the eager/e2e step is
host-bound (the small early rounds)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S, N0 = 512, 1 << 20
a = gg.GrowableArray(S, 32, dtype=np.int32)
vals = torch.arange(N0, dtype=torch.int32, device="cuda")
offs = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(N0 // S), N0)
rows = []
for it in range(25):
    torch.cuda.synchronize()
    t = [time.perf_counter()]
    a.shrink(0, release=False); t.append(time.perf_counter())
    a.insert_csr(vals, offs); t.append(time.perf_counter())
    for r in range(10):
        a.grow(2 * a.committed_size); t.append(time.perf_counter())
        a.insert_duplicate(); t.append(time.perf_counter())
    torch.cuda.synchronize(); t.append(time.perf_counter())
    if it >= 5:
        rows.append(np.diff(t) * 1e6)
m = np.median(np.asarray(rows), axis=0)
names = ["shrink0", "insert_csr"] + [f"{k}{r}" for r in range(10) for k in ("grow", "dup")] + ["sync_wait"]
print(json.dumps({n: round(float(v), 1) for n, v in zip(names, m)}))
print(json.dumps({"host_enqueue_us": round(float(m[:-1].sum()), 1), "total_us": round(float(m.sum()), 1)}))
# python-level split of one dup call: ctypes call alone vs the wrapper
from paper_2209_00103_b200 import _lib as L
st = a._stream()
import ctypes as C
ts = []
for _ in range(200):
    t0 = time.perf_counter(); a._stream(); ts.append(time.perf_counter() - t0)
print(json.dumps({"_stream_us": round(1e6 * float(np.median(ts)), 2)}))
ts = []
for _ in range(200):
    t0 = time.perf_counter(); a.committed_size; ts.append(time.perf_counter() - t0)
print(json.dumps({"committed_size_us": round(1e6 * float(np.median(ts)), 2)}))
# raw C-ABI calls (no Python wrapper) on the same state
import ctypes as C
zeros = np.zeros(S, np.uint64)
keep = (1 << 64) - 1
off_u = L.u64_array(offs)
status = np.zeros(S, np.int32)
raw = {"shrink_raw": [], "insert_raw": [], "shrink_py": [], "insert_py": [], "u64": [], "devvals": []}
for it in range(30):
    torch.cuda.synchronize()
    t0 = time.perf_counter(); L.lib.gg_shrink_ex(a._h, L.ptr(zeros), keep, st); t1 = time.perf_counter()
    L.lib.gg_insert_ex(a._h, C.c_void_p(vals.data_ptr()), L.ptr(off_u), None, L.GG_F_COMMIT,
                       L.ptr(status, C.c_int32), st); t2 = time.perf_counter()
    a._dirty()
    torch.cuda.synchronize()
    t3 = time.perf_counter(); a.shrink(0, release=False); t4 = time.perf_counter()
    a.insert_csr(vals, offs); t5 = time.perf_counter()
    L.u64_array(offs); t6 = time.perf_counter()
    a._device_values(vals); t7 = time.perf_counter()
    if it >= 5:
        for k, v in zip(raw, (t1 - t0, t2 - t1, t4 - t3, t5 - t4, t6 - t5, t7 - t6)):
            raw[k].append(v)
print(json.dumps({k: round(1e6 * float(np.median(v)), 1) for k, v in raw.items()}))
