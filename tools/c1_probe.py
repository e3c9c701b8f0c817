"""Config-1 host API breakdown: construction, insert_parallel (pack + H2D +
kernels), rw_add, flatten (D2H) -- wall clock per piece, median of 15."""
import json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

vals = np.arange(1 << 20, dtype=np.int32)
b = gg.split_batches(vals, 512)
T = {"create": [], "insert_parallel": [], "rw_add": [], "flatten": [], "destroy": []}
for _ in range(17):
    t0 = time.perf_counter(); a = gg.GrowableArray(512, 32, dtype=np.int32); torch.cuda.synchronize()
    t1 = time.perf_counter(); a.insert_parallel(b); torch.cuda.synchronize()
    t2 = time.perf_counter(); a.rw_add(1); torch.cuda.synchronize()
    t3 = time.perf_counter(); f = a.flatten()
    t4 = time.perf_counter(); a.close(); del a
    t5 = time.perf_counter()
    for k, v in zip(T, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4)):
        T[k].append(v)
print(json.dumps({k: round(1e3 * float(np.median(v[2:])), 3) for k, v in T.items()}))
