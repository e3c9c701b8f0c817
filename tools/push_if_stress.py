"""Stress the device push_back path (k_push_if: warp / block aggregated
appends with CAS-once bucket allocation under contention): repeat the
multiset + layout check of tests/test_gpu_device_api.py many times."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import paper_2209_00103_b200 as gg
from oracle import ggoracle as O

fails = 0
iters = int(os.environ.get("ITERS", "100"))
for it in range(iters):
    for mode in ("warp", "block"):
        for S, fb, grid in ((7, 4, 64), (1, 1, 200), (32, 32, 512)):
            rng = np.random.default_rng(it * 1000 + S * 31 + fb)
            n = 200_000
            vals = rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(np.int32)
            pred = rng.random(n) < 0.37
            a = gg.GrowableArray(S, fb, dtype=np.int32)
            pre = [np.arange(int(k), dtype=np.int32) for k in rng.integers(0, 100, S)]
            a.insert_parallel(pre)
            a.push_if(vals, pred, mode=mode, grid=grid)
            blk = (np.arange(n) // 1024) % grid           # kPushSlice
            shard = blk % S
            st = a._parity_state()
            for s in range(S):
                got = a.shards[s].to_numpy()
                exp = np.sort(vals[(shard == s) & pred])
                size = len(pre[s]) + len(exp)
                k = O.min_buckets_for(size, fb)
                problems = []
                if not np.array_equal(got[:len(pre[s])], pre[s]):
                    problems.append("pre contents")
                if not np.array_equal(np.sort(got[len(pre[s]):]), exp):
                    g2 = np.sort(got[len(pre[s]):])
                    bad = np.flatnonzero(g2 != exp) if len(g2) == len(exp) else []
                    problems.append(f"multiset (len {len(g2)} vs {len(exp)}, {len(bad)} differ)")
                    app = got[len(pre[s]):]
                    zeros = int((app == 0).sum())
                    allv = set(vals[pred].tolist())
                    foreign = int(sum(1 for x in app[:5000].tolist() if x not in set(exp.tolist())))
                    in_vals = int(sum(1 for x in app[:5000].tolist() if x in allv))
                    # where do wrong elements sit (bucket index of the local position)?
                    wrong_pos = [i + len(pre[s]) for i, x in enumerate(app.tolist()) if x not in set(exp.tolist())]
                    bk = sorted(set(O.locate(i, fb)[0] for i in wrong_pos[:2000]))
                    ptrs = a._bucket_ptrs()
                    bb = bk[0] if bk else 0
                    col = ptrs[:, bb].astype(np.int64)
                    stride = (fb << bb) * 4 if (fb << bb) * 4 >= 16 else 16
                    devs = [int(x) for x in np.flatnonzero((col - col[0]) != np.arange(S) * stride)]
                    fl = a.flatten_device().cpu().numpy()
                    pr = a._host()["prefix"].astype(np.int64)
                    via_walk = fl[pr[s]:pr[s + 1]]
                    walk_ok = np.array_equal(np.sort(via_walk[len(pre[s]):]), exp)
                    again_ok = np.array_equal(np.sort(a.shards[s].to_numpy()[len(pre[s]):]), exp)
                    problems.append(f"ptr[{s}][{bb}]={int(ptrs[s, bb]):#x} col0={int(col[0]):#x} stride={stride} "
                                    f"shards_off_stride={devs} walk_read_ok={walk_ok} reread_ok={again_ok} "
                                    f"slab={a.slab_stats()}")
                    problems.append(f"pre={len(pre[s])} zeros={zeros} foreign={foreign} from_other_shards={in_vals - (len(app[:5000]) - foreign)} "
                                    f"wrong_buckets={bk} first_wrong={wrong_pos[:3]} size={size}")
                if st["sizes"][s] != size:
                    problems.append(f"size {st['sizes'][s]} != {size}")
                if st["caps"][s] != O.capacity_of(k, fb):
                    problems.append(f"cap {st['caps'][s]} != {O.capacity_of(k, fb)}")
                if st["flags"][s] != (1 << k) - 1:
                    problems.append(f"flags {st['flags'][s]:#x} != {(1 << k) - 1:#x}")
                if problems:
                    fails += 1
                    print(f"FAIL it={it} mode={mode} S={S} fb={fb} grid={grid} shard={s}: {problems}", flush=True)
            a.close()
print(f"done: {iters} iterations, {fails} failing shard checks", flush=True)
