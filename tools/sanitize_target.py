"""Small run of every kernel for compute-sanitizer (memcheck / racecheck /
synccheck): ragged CSR insert, duplicate, r/w both modes, flatten,
flatten_range, grow, shrink, lanes insert, device push_back (warp / block),
gather / scatter, static baselines, many-shard metadata."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

rng = np.random.default_rng(0)
for S, fb, dt in [(37, 4, np.int32), (5, 1, np.int8), (1100, 8, np.int64)]:
    counts = rng.integers(0, 300, S)
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    vals = torch.from_numpy(rng.integers(0, 50, int(off[-1])).astype(dt)).cuda()
    a = gg.GrowableArray(S, fb, dtype=dt)
    a.insert_csr(vals, off)
    a.grow(3 * a.committed_size)
    a.insert_duplicate()
    a.rw_add(1)
    a.rw_add(1, mode="global")
    f = a.flatten_device()
    r = a.flatten_range(3, max(3, a.committed_size - 7))
    idx = torch.from_numpy(rng.integers(0, a.committed_size, 1000)).cuda()
    g = a.get_many(idx)
    a.set_many(idx, g)
    a.shrink(np.maximum(a._host()["sizes"].astype(np.int64) // 3, 0))
    lanes = 64
    cnt = torch.randint(0, 3, (S * lanes,), dtype=torch.int32, device="cuda")
    lv = torch.arange(S * lanes * 2, device="cuda").to(torch.from_numpy(np.zeros(1, dt)).dtype)
    a.insert_lanes(lv, cnt, np.arange(S + 1, dtype=np.uint64) * lanes, 2)
    m = min(5000, lv.numel())
    for mode in ("warp", "block"):
        pred = (torch.arange(m, device="cuda") % 3 == 0).to(torch.uint8)
        a.push_if(lv[:m], pred, mode=mode)
    a.close()
# lanes inserts with many tiles per chunk: the TMA ring (k_lanes_bulk, 32 B
# lanes) refills its stages, the register path (k_lanes_chunk, 4 B lanes)
for K in (8, 1):
    b = gg.GrowableArray(8, 32, dtype=np.int32)
    Ln = 8 * 20011
    cnt = torch.randint(0, K + 1, (Ln,), dtype=torch.int32, device="cuda")
    b.insert_lanes(torch.arange(Ln * K, dtype=torch.int32, device="cuda"), cnt,
                   np.arange(9, dtype=np.uint64) * 20011, K)
    b.close()
st = gg.StaticArray(1 << 16, dtype=np.int32)
for algo in ("atomic", "warp", "block"):
    st._count = 0
    st._d_count.fill_(0)
    st.insert_batch(torch.arange(1000, dtype=torch.int32, device="cuda"), algo=algo)
torch.cuda.synchronize()
print("sanitize target done")
# uniform CSR inserts over uniform shards (plan-shard-0-once path), fused and unfused metadata
from paper_2209_00103_b200 import _lib as _L
for fuse in (1, 0):
    _L.lib.gg_set_fuse(fuse)
    u = gg.GrowableArray(64, 8, dtype=np.int32)
    for c in (3, 13, 40):
        u.insert_csr(torch.arange(64 * c, dtype=torch.int32, device="cuda"),
                     np.arange(65, dtype=np.uint64) * np.uint64(c))
        u.insert_duplicate()
    assert u.committed_size == ((3 * 2 + 13) * 2 + 40) * 2 * 64
    u.flatten_device()
_L.lib.gg_set_fuse(1)
torch.cuda.synchronize()
print("uniform insert ok")
# S > 4096: uniform appends take the store-only multi-CTA metadata kernel;
# uniform resets take the store-only shrink
w = gg.GrowableArray(5000, 4, dtype=np.int32)
for rnd in range(2):
    w.shrink(0, release=False)
    w.insert_csr(torch.arange(5000 * 7, dtype=torch.int32, device="cuda"),
                 np.arange(5001, dtype=np.uint64) * np.uint64(7))
    w.grow(2 * w.committed_size)
    w.insert_duplicate()
assert w.committed_size == 5000 * 14
w.flatten_device()
torch.cuda.synchronize()
print("large-S uniform ok")
