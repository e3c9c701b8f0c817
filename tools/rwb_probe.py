"""rw_b (+1 per pass, in place on the slabs) GB/s on the config-2 end state,
3 x 50 passes; A/B builds via GG_LIB_PATH."""
import json, os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import paper_2209_00103_b200 as gg
a = gg.GrowableArray.from_flat(torch.arange(1 << 20, dtype=torch.int32, device="cuda"), 512, 32)
for _ in range(10):
    a.grow(2 * a.committed_size); a.insert_duplicate()
n = a.committed_size
a.rw_add(1, passes=5)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
res = []
for _ in range(3):
    e0.record(); a.rw_add(1, passes=50); e1.record(); torch.cuda.synchronize()
    res.append(round(8 * n / (e0.elapsed_time(e1) / 50) / 1e6, 1))
print(json.dumps({"lib": os.environ.get("GG_LIB_PATH", "new"), "rw_b_gbs": res}))
