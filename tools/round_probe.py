"""Per-round cost of the config-2 doubling schedule inside a CUDA graph:
graphs of reset + r rounds for r = 0..10 are replayed; the increment of
round r is compared with its HBM time at the measured copy bandwidth.
Also: a graph of 20 back-to-back gg_commit launches (pure per-kernel cost)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_00103_b200 as gg

S, FB, N0 = 512, 32, 1 << 20
dev = torch.device("cuda", 0)
a = gg.GrowableArray(S, FB, dtype=np.int32, device=dev)
vals = torch.arange(N0, dtype=torch.int32, device=dev)
offs = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(N0 // S), N0)


def seq(r):
    a.shrink(0, release=False)
    a.insert_csr(vals, offs)
    for _ in range(r):
        a.grow(2 * a.committed_size)
        a.insert_duplicate()


for _ in range(2):
    seq(10)
torch.cuda.synchronize()
st = torch.cuda.Stream()


def graph_time(fn, reps=20):
    with torch.cuda.stream(st):
        fn()
        torch.cuda.synchronize()
        g = a.capture(fn, stream=st)
    g.replay(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3   # us


ts = [graph_time(lambda r=r: seq(r)) for r in range(11)]
hbm = json.load(open("MEASURED_PEAKS.json")).get("hbm_gbs", 6547.5) if os.path.exists("MEASURED_PEAKS.json") else 6547.5
out = []
for r in range(1, 11):
    n = N0 << (r - 1)
    ideal = 8 * n / (hbm * 1e3)     # us
    out.append({"round": r, "elems": n, "us": round(ts[r] - ts[r - 1], 2), "hbm_ideal_us": round(ideal, 2)})
print(json.dumps({"reset_insert_us": round(ts[0], 2), "rounds": out, "step_us": round(ts[10], 2)}))
c = graph_time(lambda: [a.commit() for _ in range(20)])
print(json.dumps({"commit_x20_us": round(c, 2), "per_kernel_us": round(c / 20, 2)}))
g = graph_time(lambda: [a.grow(a.committed_size) for _ in range(20)])
print(json.dumps({"noop_grow_x20_us": round(g, 2)}))
