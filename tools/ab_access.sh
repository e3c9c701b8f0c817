# A/B of batched cuMemSetAccess on the same box: cold first step + config-1 probe
for v in 1 0 1 0; do
  echo "GG_BATCH_ACCESS=$v"
  GG_BATCH_ACCESS=$v python tools/c1_probe.py
  GG_BATCH_ACCESS=$v python -c "
import time, numpy as np, torch, paper_2209_00103_b200 as gg
torch.zeros(1, device='cuda'); gg.pool_trim(0)
a = gg.GrowableArray(512, 32, dtype=np.int32)
v = torch.arange(1 << 20, dtype=torch.int32, device='cuda')
off = np.arange(513, dtype=np.uint64) * np.uint64(2048)
torch.cuda.synchronize(); t0 = time.perf_counter()
a.insert_csr(v, off)
for _ in range(10):
    a.grow(2 * a.committed_size); a.insert_duplicate()
torch.cuda.synchronize(); print('cold step ms', round((time.perf_counter() - t0) * 1e3, 2), a.slab_stats()['chunks_mapped'], round(a.slab_stats()['map_ns'] / 1e6, 2))
"
done
