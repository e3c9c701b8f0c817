"""ncu target: one walk r/w pass (S=512, fb=32, 2^30 int32), one walk pass over a
few-bucket layout (S=1, fb=2^26), and one contiguous +1 pass -- to separate
per-tile/per-piece overhead from memory behaviour."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg
n = 1 << 30
src = torch.zeros(n, dtype=torch.int32, device="cuda")
a = gg.GrowableArray.from_flat(src, 512, 32)
b = gg.GrowableArray.from_flat(src, 1, 1 << 26)
st = gg.StaticArray(n, dtype=np.int32); st.insert_batch(src)
del src
torch.cuda.synchronize()
for _ in range(2):
    a.rw_add(1); b.rw_add(1); st.rw_add(1)
torch.cuda.synchronize()
print("done")
