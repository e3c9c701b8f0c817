"""e2e variants in one process: op by op (bench's e2e) vs the same with the
next step's host batch prefetched on a side stream (double-buffered)."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S, FB, N0, R = 512, 32, 1 << 20, 10
dev = torch.device("cuda", 0)
host = torch.arange(N0, dtype=torch.int32).pin_memory()
offs = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(N0 // S), N0)
arr = gg.GrowableArray(S, FB, dtype=np.int32, device=dev)
pre_d = torch.empty(S + 1, dtype=torch.int64, device=dev)
pre_h = torch.empty(S + 1, dtype=torch.int64).pin_memory()
main = torch.cuda.current_stream()

def rounds():
    for _ in range(R):
        arr.grow(2 * arr.committed_size)
        arr.insert_duplicate()

def plain(k):
    t0 = time.perf_counter()
    for _ in range(k):
        arr.shrink(0, release=False)
        arr.insert_csr(host.to(dev, non_blocking=True), offs)
        rounds()
        pre_h.copy_(arr.prefix_device(out=pre_d), non_blocking=True)
        main.synchronize()
    return time.perf_counter() - t0

cs = torch.cuda.Stream()
bufs = [torch.empty(N0, dtype=torch.int32, device=dev) for _ in range(2)]
ready = [torch.cuda.Event() for _ in range(2)]
def prefetch(i):
    with torch.cuda.stream(cs):
        bufs[i].copy_(host, non_blocking=True)
        ready[i].record(cs)

def piped(k):
    t0 = time.perf_counter()
    prefetch(0)
    for j in range(k):
        c = j & 1
        main.wait_event(ready[c])
        arr.shrink(0, release=False)
        arr.insert_csr(bufs[c], offs)
        if j + 1 < k:
            prefetch(c ^ 1)
        rounds()
        pre_h.copy_(arr.prefix_device(out=pre_d), non_blocking=True)
        main.synchronize()
    return time.perf_counter() - t0

for f in (plain, piped, plain, piped):
    f(3)
res = {}
for name, f in (("plain", plain), ("piped", piped)):
    ts = sorted(f(10) for _ in range(5))
    res[name] = round(10 * (1 << 30) / ts[2] / 1e9, 1)
print(json.dumps(res))
