"""Throughput of the non-uniform insert paths at 2^28 int32 over 512
LFVectors: ragged CSR insert (per-shard counts uniform in [0, 2 x mean]),
duplicate of the ragged array (misaligned source/destination), the paper
Alg. 1 lanes insert (per-lane counts uniform in [0, K]) and push_if
(predicate density 1/2).  CUDA events on the current stream, best of 5."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S, FB = 512, 32
N = 1 << int(os.environ.get("PROBE_LOG2N", "28"))
PEAK = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json"))).get("hbm_gbs", 6540.0) \
    if os.path.exists(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")) else 6540.0
rng = np.random.default_rng(0)
out = {"n": N, "S": S, "peak_gbs": PEAK}


def timed(fn, reset, reps=5):
    best = 1e9
    for _ in range(reps):
        reset()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


def rec(name, ms, nbytes, elems):
    gbs = nbytes / (ms * 1e-3) / 1e9
    out[name] = {"ms": round(ms, 4), "gbs": round(gbs, 1), "frac": round(gbs / PEAK, 4),
                 "gelem_s": round(elems / (ms * 1e-3) / 1e9, 2)}


# ragged CSR insert
mean = N // S
counts = rng.integers(0, 2 * mean + 1, S).astype(np.int64)
counts = (counts * (N / counts.sum())).astype(np.int64)
counts[-1] += N - counts.sum()
off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
src = torch.arange(N, dtype=torch.int32, device="cuda")
a = gg.GrowableArray(S, FB, dtype=np.int32)
a.insert_csr(src, off)
a.insert_duplicate()
a.shrink(0, release=False)
torch.cuda.synchronize()
rec("ragged_insert_csr", timed(lambda: (a.insert_csr(src, off), a.flush()), lambda: a.shrink(0, release=False)),
    8 * N, N)                                 # flush(): the deferred metadata pass is inside the timing


def graph_ms(fn, reps=10):
    """device time per replay of fn captured once (host planning excluded)"""
    g = a.capture(fn)
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


rec("ragged_insert_csr_graph", graph_ms(lambda: (a.shrink(0, release=False), a.insert_csr(src, off))), 8 * N, N)
out["ragged_insert_csr_graph"]["note"] = "reset + insert replayed as a CUDA graph (device time)"
rec("ragged_insert_dup_graph", graph_ms(lambda: (a.shrink(0, release=False), a.insert_csr(src, off),
                                                  a.insert_duplicate())), 16 * N, 2 * N)
out["ragged_insert_dup_graph"]["note"] = "reset + insert + duplicate replayed as a CUDA graph (device time)"
# duplicate of the ragged array (source and destination misaligned per shard)
def reset_dup():
    a.shrink(0, release=False)
    a.insert_csr(src, off)
rec("ragged_duplicate", timed(lambda: (a.insert_duplicate(), a.flush()), reset_dup), 8 * N, N)
exp = torch.cat([torch.cat([src[int(off[s]):int(off[s + 1])]] * 2) for s in range(S)])
out["ragged_contents_ok"] = bool(torch.equal(a.flatten_device(), exp))
del exp
rec("ragged_flatten", timed(lambda: a.flatten_device(), lambda: None), 8 * 2 * N, 2 * N)
rec("ragged_rw_per_shard", timed(lambda: a.rw_add(1), lambda: None), 8 * 2 * N, 2 * N)
exp = torch.cat([torch.cat([src[int(off[s]):int(off[s + 1])]] * 2) for s in range(S)]) + 5
out["ragged_rw_contents_ok"] = bool(torch.equal(a.flatten_device(), exp))
del exp

# lanes insert (paper Alg. 1 with per-lane counts)
for K in (8, 1):
    L = N // max(1, K // 2)                      # expected elements ~ N
    lanes_per = L // S
    lo = (np.arange(S + 1, dtype=np.uint64) * np.uint64(lanes_per))
    cnt = torch.from_numpy(rng.integers(0, K + 1, S * lanes_per).astype(np.int32)).cuda()
    vals = torch.arange(S * lanes_per * K, dtype=torch.int32, device="cuda")
    tot = int(cnt.sum())
    b = gg.GrowableArray(S, FB, dtype=np.int32)
    b.insert_lanes(vals, cnt, lo, K, commit=False)
    torch.cuda.synchronize()
    ms = timed(lambda: b.insert_lanes(vals, cnt, lo, K, commit=False), lambda: b.shrink(0, release=False))
    useful = 2 * 4 * tot + 4 * S * lanes_per
    rec(f"lanes_K{K}", ms, useful, tot)
    b.commit()
    mask = torch.arange(K, device="cuda")[None, :] < cnt[:, None]
    out[f"lanes_K{K}_contents_ok"] = bool(torch.equal(b.flatten_device(), vals.view(-1, K)[mask]))
    del mask
    out[f"lanes_K{K}"]["layout_bytes"] = 4 * S * lanes_per * K + 4 * tot + 4 * S * lanes_per
    out[f"lanes_K{K}"]["elements"] = tot
    b.close()
    del vals, cnt

# push_if (predicate density 1/2)
vals = torch.arange(N, dtype=torch.int32, device="cuda")
pred = (torch.rand(N, device="cuda") < 0.5).to(torch.uint8)
tot = int(pred.sum())
for mode in ("block", "warp"):
    c = gg.GrowableArray(S, FB, dtype=np.int32)
    c.push_if(vals, pred, mode=mode, commit=False)
    torch.cuda.synchronize()
    ms = timed(lambda: c.push_if(vals, pred, mode=mode, commit=False), lambda: c.shrink(0, release=False))
    rec(f"push_if_{mode}", ms, 4 * N + N + 4 * tot, tot)
    c.close()
print(json.dumps(out))
