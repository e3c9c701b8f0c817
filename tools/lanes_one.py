"""One insert_lanes launch (K from argv, int32, ~2^28 appended over 512
LFVectors) for ncu captures of the lanes kernels."""
import os
import sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

K = int(sys.argv[1]) if len(sys.argv) > 1 else 8
S, FB, L = 512, 32, (1 << 29) // max(K, 1) if K > 1 else 1 << 28
cnt = torch.randint(0, K + 1, (L,), dtype=torch.int32, device="cuda")
vals = torch.arange(L * K, dtype=torch.int32, device="cuda")
lo = np.arange(S + 1, dtype=np.uint64) * np.uint64(L // S)
a = gg.GrowableArray(S, FB, dtype=np.int32)
a.insert_lanes(vals, cnt, lo, K, commit=False)
a.shrink(0, release=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled")
a.insert_lanes(vals, cnt, lo, K, commit=False)
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("lanes_one done", K)
