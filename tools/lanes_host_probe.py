"""Host time inside one insert_lanes call (paper Alg. 1, K = 1 / 8, int32,
2^28 lanes-worth over 512 LFVectors, reset with shrink(0, release=False)):
wall time of the public call (it returns once the kernel is queued), of the
raw C-ABI call, and the event time around the call -- where the gap between
the event time and the kernel's ncu duration goes."""
import ctypes as C
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_00103_b200 as gg
from paper_2209_00103_b200 import _lib as L

S, FB = 512, 32
dev = torch.device("cuda", 0)
out = {}
for K in (1, 8):
    Ln = (1 << 28) if K == 1 else (1 << 29) // K
    cnt = torch.randint(0, K + 1, (Ln,), dtype=torch.int32, device=dev)
    vals = torch.arange(Ln * K, dtype=torch.int32, device=dev)
    lo = np.arange(S + 1, dtype=np.uint64) * np.uint64(Ln // S)
    a = gg.GrowableArray(S, FB, dtype=np.int32)
    a.insert_lanes(vals, cnt, lo, K, commit=False)
    rec = {"api_wall_us": [], "cabi_wall_us": [], "event_us": [], "shrink_wall_us": []}
    lo_c = L.u64_array(lo)
    status = np.zeros(S, np.int32)
    for i in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.shrink(0, release=False)
        rec["shrink_wall_us"].append((time.perf_counter() - t0) * 1e6)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        t0 = time.perf_counter()
        if i % 2 == 0:
            a.insert_lanes(vals, cnt, lo, K, commit=False)
            rec["api_wall_us"].append((time.perf_counter() - t0) * 1e6)
        else:
            with a._mu:
                rc = L.lib.gg_insert_lanes(a._h, C.c_void_p(vals.data_ptr()), C.c_void_p(cnt.data_ptr()),
                                           L.ptr(lo_c), K, L.ptr(status, C.c_int32), a._stream())
                a._dirty()
            rec["cabi_wall_us"].append((time.perf_counter() - t0) * 1e6)
            assert rc == 0, rc
        e1.record()
        torch.cuda.synchronize()
        rec["event_us"].append(e0.elapsed_time(e1) * 1e3)
    out[f"K{K}"] = {k: round(float(np.median(v[2:] if len(v) > 4 else v)), 1) for k, v in rec.items()}
    a.close()
    del a, cnt, vals
    torch.cuda.empty_cache()
print(json.dumps(out))
