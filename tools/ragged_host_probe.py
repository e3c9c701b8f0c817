"""Host time inside the ragged insert paths (bench.py insert_paths leg: 2^28
int32 over 512 LFVectors, per-LFVector batch sizes uniform in [0, 2 x
mean], reset with shrink(0, release=False)): wall time of insert_csr and
insert_duplicate (they return once the work is queued; GPU idle at entry),
the event time around each, and the shrink(0) reset."""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_00103_b200 as gg

S, FB, N = 512, 32, 1 << 28
dev = torch.device("cuda", 0)
rng = np.random.default_rng(0)
counts = rng.integers(0, 2 * (N // S) + 1, S).astype(np.int64)
counts = (counts * (N / counts.sum())).astype(np.int64)
counts[-1] += N - counts.sum()
off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
src = torch.arange(N, dtype=torch.int32, device=dev)
a = gg.GrowableArray(S, FB, dtype=np.int32)
a.insert_csr(src, off)
a.insert_duplicate()
out = {}


def timed(name, fn, reset):
    rec = {"wall_us": [], "event_us": [], "reset_wall_us": []}
    for _ in range(12):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        reset()
        rec["reset_wall_us"].append((time.perf_counter() - t0) * 1e6)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        t0 = time.perf_counter()
        fn()
        rec["wall_us"].append((time.perf_counter() - t0) * 1e6)
        e1.record()
        torch.cuda.synchronize()
        rec["event_us"].append(e0.elapsed_time(e1) * 1e3)
    out[name] = {k: round(float(np.median(v[2:])), 1) for k, v in rec.items()}


timed("insert_csr", lambda: (a.insert_csr(src, off), a.flush()), lambda: a.shrink(0, release=False))


def reset_dup():
    a.shrink(0, release=False)
    a.insert_csr(src, off)


timed("insert_duplicate", lambda: (a.insert_duplicate(), a.flush()), reset_dup)
print(json.dumps(out))
