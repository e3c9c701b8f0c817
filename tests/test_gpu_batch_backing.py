"""Batched (run) backing of new bucket classes against one slab call per
bucket and against the per-shard fallback a run takes when it cannot be
backed (gg_set_batch_backing 1 / 0 / 2): ragged CSR inserts, a duplicate,
the lanes insert (mode 2 sends it down the exact two-pass path) and a
push_if device view must give the same per-LFVector contents, sizes and
capacities as the oracle's bucket arithmetic (bucket_vector.py:62-79), and
return their unused headroom."""
import numpy as np
import pytest

from oracle import ggoracle as O

pytestmark = pytest.mark.gpu


@pytest.mark.parametrize("mode", [1, 0, 2])
def test_backing_modes_agree(mode):
    import torch
    import paper_2209_00103_b200 as gg
    from paper_2209_00103_b200 import _lib as L
    assert L.lib.gg_set_batch_backing(mode) == 0
    try:
        S, fb = 48, 8
        rng = np.random.default_rng(11)
        a = gg.GrowableArray(S, fb, dtype=np.int32)
        want = [np.zeros(0, np.int32) for _ in range(S)]
        tag = 0
        for rnd in range(3):                          # ragged CSR inserts, growing
            cnt = rng.integers(0, 40 << rnd, S)
            cnt[rng.integers(0, S, 5)] = 0                # empty batches break the runs
            off = np.concatenate([[0], np.cumsum(cnt)]).astype(np.uint64)
            vals = np.arange(tag, tag + int(off[-1]), dtype=np.int32)
            tag += int(off[-1])
            a.insert_csr(torch.from_numpy(vals).cuda(), off)
            for s in range(S):
                want[s] = np.concatenate([want[s], vals[int(off[s]):int(off[s + 1])]])
        a.insert_duplicate()
        want = [np.concatenate([w, w]) for w in want]
        K = 4                                         # paper Alg. 1 lanes
        lanes = rng.integers(0, 30, S)
        lo = np.concatenate([[0], np.cumsum(lanes)]).astype(np.uint64)
        lc = rng.integers(0, K + 1, int(lo[-1])).astype(np.int32)
        lv = np.arange(tag, tag + int(lo[-1]) * K, dtype=np.int32)
        tag += lv.size
        a.insert_lanes(torch.from_numpy(lv).cuda(), torch.from_numpy(lc).cuda(), lo, K)
        for s in range(S):
            parts = [lv[j * K:j * K + lc[j]] for j in range(int(lo[s]), int(lo[s + 1]))]
            want[s] = np.concatenate([want[s]] + parts)
        for s in range(S):
            got = a.shards[s].to_numpy()
            assert np.array_equal(got, want[s]), f"shard {s}"
        n = 20000                                     # device-side appends through a view
        pv = np.arange(tag, tag + n, dtype=np.int32)
        pp = (rng.random(n) < 0.5).astype(np.uint8)
        a.push_if(torch.from_numpy(pv).cuda(), torch.from_numpy(pp).cuda())
        tails = np.concatenate([a.shards[s].to_numpy()[len(want[s]):] for s in range(S)])
        assert np.array_equal(np.sort(tails), pv[pp.astype(bool)])
        st = a._parity_state()
        for s in range(S):
            k = O.min_buckets_for(int(st["sizes"][s]), fb)
            assert st["caps"][s] == O.capacity_of(k, fb)
        ms = a.memory_stats()
        assert ms["bucket_bytes"] == ms["capacity_bytes"]    # unused headroom given back
        a.close()
    finally:
        L.lib.gg_set_batch_backing(1)
