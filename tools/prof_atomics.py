"""Launch the atomic-bound kernels once each for an ncu atomics capture:
static insert of 2^26 int32 with one atomicAdd per element / per warp / per
block (paper section 3-B), the device push_back (warp and block aggregated)
on 2^24 candidates, and the per-lane-count insert (paper Alg. 1)."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

n = 1 << 26
vals = torch.arange(n, dtype=torch.int32, device="cuda")
for algo in ("atomic", "warp", "block"):
    st = gg.StaticArray(n, dtype=np.int32)
    st.insert_batch(vals, algo=algo)
    torch.cuda.synchronize()
    del st
m = 1 << 24
a = gg.GrowableArray(512, 32, dtype=np.int32)
pred = (torch.arange(m, device="cuda") % 3 != 0).to(torch.uint8)
a.push_if(vals[:m], pred, mode="warp")
a.push_if(vals[:m], pred, mode="block")
S, lanes = 512, 1024
counts = torch.randint(0, 5, (S * lanes,), dtype=torch.int32, device="cuda")
lv = torch.arange(S * lanes * 4, dtype=torch.int32, device="cuda")
a.insert_lanes(lv, counts, np.arange(S + 1, dtype=np.uint64) * lanes, 4)
torch.cuda.synchronize()
print("atomics target done")
