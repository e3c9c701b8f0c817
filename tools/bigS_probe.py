"""Reset + 2^25 insert + one doubling round at S = 16384 LFVectors x 2048
int32 (run under ncu for the per-kernel launch list)."""
import os, sys
sys.path.insert(0, os.getcwd())
import numpy as np, torch, paper_2209_00103_b200 as gg
S = 16384; per = 2048
a = gg.GrowableArray(S, 32, dtype=np.int32)
vals = torch.arange(S * per, dtype=torch.int32, device="cuda")
offs = np.arange(S + 1, dtype=np.uint64) * np.uint64(per)
for _ in range(3):
    a.shrink(0, release=False); a.insert_csr(vals, offs)
    a.grow(2 * a.committed_size); a.insert_duplicate()
torch.cuda.synchronize()
