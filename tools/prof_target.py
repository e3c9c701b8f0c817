"""Launch each hot kernel once at config-2 scale, for ncu captures.

Sequence: from_flat(2^20) and 9 doubling rounds (warm state, 2^29 elements),
then the profiled launches: [dup 2^29 -> 2^30] [rw per_shard] [rw global]
[flatten] [insert_csr 2^28 from a flat device batch].
"""
import sys
import os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S, FB = 512, 32
a = gg.GrowableArray.from_flat(torch.arange(1 << 20, dtype=torch.int32, device="cuda"), S, FB)
for _ in range(9):
    a.grow(2 * a.committed_size)
    a.insert_duplicate()
a.grow(2 * a.committed_size)
torch.cuda.synchronize()
torch.cuda.nvtx.range_push("profiled")
a.insert_duplicate()                 # k_walk<4,1> over 2^29 elements
a.rw_add(1, mode="per_shard")        # k_walk<4,3>
a.rw_add(1, mode="global")           # k_rw_global
out = a.flatten_device()             # k_walk<4,2>
b = gg.GrowableArray(S, FB, dtype=np.int32)
vals = torch.arange(1 << 28, dtype=torch.int32, device="cuda")
off = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64((1 << 28) // S), 1 << 28)
b.insert_csr(vals, off)              # k_walk<4,0>
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
print("prof target done", a.committed_size, b.committed_size)
