"""rw_g vs rw_b HBM GB/s on the config-2 end state (2^30 int32, S=512) and on a
ragged array; contents checked."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg

S, N0 = 512, 1 << 20
a = gg.GrowableArray.from_flat(torch.arange(N0, dtype=torch.int32, device="cuda"), S, 32)
for _ in range(10):
    a.grow(2 * a.committed_size)
    a.insert_duplicate()
n = a.committed_size


def t(fn, reps):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record(); fn(); e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


before = a.flatten_device().clone()
out = {"U": os.environ.get("GG_RWG_U", "4")}
for mode in ("global", "per_shard"):
    ms = t(lambda: a.rw_add(1, passes=20, mode=mode), 20)
    out[mode + "_gbs"] = round(8 * n / ms / 1e6, 1)
after = a.flatten_device()
out["ok"] = bool(torch.equal(after, before + 80))   # 2 modes x (warm-up + timed) x 20 passes
# ragged: random shard sizes, int8 / int64
rng = np.random.default_rng(1)
for dt, tdt in ((np.int8, torch.int8), (np.int64, torch.int64)):
    cnt = rng.integers(0, 100000, 300)
    off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
    v = torch.from_numpy(rng.integers(0, 100, int(off[-1])).astype(dt)).cuda()
    r = gg.GrowableArray(300, 4, dtype=dt)
    r.insert_csr(v, off)
    r.rw_add(3, passes=2, mode="global")
    out[f"ragged_{np.dtype(dt).name}_ok"] = bool(torch.equal(r.flatten_device(), v + 6))
print(json.dumps(out))
