"""Where the reset's 2^20 insert spends its time (graph-replayed pairs of
shrink(0) + insert): batch size per shard 1 / 64 / 2048, i.e. 1 / 2 / 7 new
buckets per shard to publish, against the copy volume."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S = int(os.environ.get("PROBE_S", "512"))
a = gg.GrowableArray(S, 32, dtype=np.int32)
res = {"S": S, "fuse": os.environ.get("GG_FUSE_META", "1")}
for per in (1, 64, 2048, 4096):
    n = per * S
    vals = torch.arange(n, dtype=torch.int32, device="cuda")
    offs = np.arange(S + 1, dtype=np.uint64) * np.uint64(per)

    def pairs():
        for _ in range(20):
            a.shrink(0, release=False)
            a.insert_csr(vals, offs)
    pairs()
    g = a.capture(pairs)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        e0.record()
        for _ in range(10):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / 10 / 20 * 1e3)
    res[f"per{per}_us"] = round(best, 2)
print(json.dumps(res))
