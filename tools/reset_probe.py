"""Device time of the config-2 reset (shrink(0) + 2^20 insert) and of the whole
step, graph-replayed (no host in the loop).  A/B builds: GG_LIB_PATH=..."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S, N0 = 512, 1 << 20
a = gg.GrowableArray(S, 32, dtype=np.int32)
vals = torch.arange(N0, dtype=torch.int32, device="cuda")
offs = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(N0 // S), N0)


def step():
    a.shrink(0, release=False)
    a.insert_csr(vals, offs)
    for _ in range(10):
        a.grow(2 * a.committed_size)
        a.insert_duplicate()


def reset_only():
    for _ in range(20):
        a.shrink(0, release=False)
        a.insert_csr(vals, offs)
        a.grow(2 * a.committed_size)     # a bucket to drop on the next reset
        a.insert_duplicate()


def timed(g, reps):
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    best = 1e9
    for _ in range(5):
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1) / reps)
    return best


step()
gs = a.capture(step)
gr = a.capture(reset_only)
print(json.dumps({"lib": os.environ.get("GG_LIB_PATH", "default"),
                  "step_us": round(1e3 * timed(gs, 50), 2),
                  "reset_plus_round_us": round(1e3 * timed(gr, 20) / 20, 2)}))
# components: 20 x shrink(0) alone; 20 x (shrink(0) + 2^20 insert)


def shrinks():
    for _ in range(20):
        a.shrink(0, release=False)


def pairs():
    for _ in range(20):
        a.shrink(0, release=False)
        a.insert_csr(vals, offs)


step()
g1 = a.capture(shrinks)
g2 = a.capture(pairs)
print(json.dumps({"shrink_us": round(1e3 * timed(g1, 20) / 20, 2),
                  "shrink_plus_insert_us": round(1e3 * timed(g2, 20) / 20, 2)}))
