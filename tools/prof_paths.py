"""One launch of each non-uniform insert path at 2^28 int32 over 512
LFVectors, for ncu --set full: ragged CSR insert, duplicate and flatten of
the ragged array, lanes insert (K = 8 and K = 1: k_lanes_chunk),
push_if (block mode)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S, FB, N = 512, 32, 1 << 28
rng = np.random.default_rng(0)
counts = rng.integers(0, 2 * (N // S) + 1, S).astype(np.int64)
counts = (counts * (N / counts.sum())).astype(np.int64)
counts[-1] += N - counts.sum()
off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
src = torch.arange(N, dtype=torch.int32, device="cuda")
a = gg.GrowableArray(S, FB, dtype=np.int32)
a.insert_csr(src, off)                 # k_walk<4,0> ragged
a.insert_duplicate()                   # k_walk<4,1> ragged
a.flatten_device()                     # k_walk<4,2> ragged
torch.cuda.synchronize()
a.close()
for K in (8, 1):
    L = N // max(1, K // 2)
    lo = np.arange(S + 1, dtype=np.uint64) * np.uint64(L // S)
    cnt = torch.randint(0, K + 1, (L,), dtype=torch.int32, device="cuda")
    vals = torch.arange(L * K, dtype=torch.int32, device="cuda")
    b = gg.GrowableArray(S, FB, dtype=np.int32)
    b.insert_lanes(vals, cnt, lo, K, commit=False)
    torch.cuda.synchronize()
    b.close()
    del vals, cnt
pred = (torch.rand(N, device="cuda") < 0.5).to(torch.uint8)
c = gg.GrowableArray(S, FB, dtype=np.int32)
c.push_if(src, pred, mode="block", commit=False)
torch.cuda.synchronize()
print("prof paths done")
