"""Is VMM-mapped memory slower to stream than cudaMalloc memory?  +1 sweeps and
D2D copies over torch (cudaMalloc) vs memMap (cuMemCreate/cuMemMap) buffers."""
import ctypes as C
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg
from paper_2209_00103_b200 import _lib

n = 1 << 30
def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps): fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
st = gg.StaticArray(n, dtype=np.int32); st.insert_batch(torch.zeros(n, dtype=torch.int32, device="cuda"))
ms = t(lambda: st.rw_add(1))
print(json.dumps({"what": "flat_add torch mem", "gbs": 8 * n / ms / 1e6}))
mm = gg.ChunkTableArray(chunk_size=1 << 20, dtype=np.int32); mm.resize(n); mm.insert_batch(torch.zeros(n, dtype=torch.int32, device="cuda"))
ms = t(lambda: mm.rw_add(1))
print(json.dumps({"what": "flat_add vmm mem (2MiB granules)", "gbs": 8 * n / ms / 1e6}))
v1, v2 = mm.view()[: n // 2], mm.view()[n // 2:]
ms = t(lambda: v2.copy_(v1))
print(json.dumps({"what": "torch copy vmm->vmm 2^29", "gbs": 8 * (n // 2) / ms / 1e6}))
x, y = st.view()[: n // 2], st.view()[n // 2:]
ms = t(lambda: y.copy_(x))
print(json.dumps({"what": "torch copy torchmem 2^29", "gbs": 8 * (n // 2) / ms / 1e6}))
