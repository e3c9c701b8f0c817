"""Device-side push_back (include/ggarray_device.cuh, paper Alg. 1/2): appends
from inside a kernel with warp-ballot or block-scan offsets, one atomicAdd per
warp / block and on-demand CAS-once bucket allocation under contention."""
import numpy as np
import pytest

from oracle import ggoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gg():
    import paper_2209_00103_b200 as gg
    return gg


def _expected(vals, pred, S, grid, B=1024):   # slice = 1024 candidates (kPushSlice)
    blk = (np.arange(len(vals)) // B) % grid
    shard = blk % S
    return [np.sort(vals[(shard == s) & pred]) for s in range(S)]


@pytest.mark.parametrize("mode", ["block", "warp"])
@pytest.mark.parametrize("S,fb,grid", [(7, 4, 64), (1, 1, 200), (32, 32, 512)])
def test_push_if_multiset_and_layout(gg, mode, S, fb, grid):
    rng = np.random.default_rng(S * 31 + fb)
    n = 200_000
    vals = rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(np.int32)
    pred = rng.random(n) < 0.37
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    pre = [np.arange(int(k), dtype=np.int32) for k in rng.integers(0, 100, S)]
    a.insert_parallel(pre)
    a.push_if(vals, pred, mode=mode, grid=grid)
    exp = _expected(vals, pred, S, grid)
    st = a._parity_state()
    for s in range(S):
        got = a.shards[s].to_numpy()
        assert np.array_equal(got[:len(pre[s])], pre[s])               # earlier contents untouched
        assert np.array_equal(np.sort(got[len(pre[s]):]), exp[s])        # multiset of the appends
        size = len(pre[s]) + len(exp[s])
        k = O.min_buckets_for(size, fb)
        assert st["sizes"][s] == size
        assert st["caps"][s] == O.capacity_of(k, fb)                     # demand-driven: minimal prefix
        assert st["flags"][s] == (1 << k) - 1
    ms = a.memory_stats()
    if fb * 4 % 16 == 0:                                                 # no 16 B padding
        assert ms["bucket_bytes"] == ms["capacity_bytes"]
    assert ms["mapped_bytes"] - ms["bucket_bytes"] < 64 << 20        # headroom trimmed


def test_block_order_within_a_block(gg):
    # with one block per shard and one round, block_push_back keeps thread order
    S, n = 4, 4 * 1024
    vals = np.arange(n, dtype=np.int32)
    pred = (vals % 3) != 0
    a = gg.GrowableArray(S, 32, dtype=np.int32)
    a.push_if(vals, pred, mode="block", grid=4)
    for s in range(S):
        sl = vals[s * 1024:(s + 1) * 1024]
        assert np.array_equal(a.shards[s].to_numpy(), sl[(sl % 3) != 0])


def test_device_append_oom_keeps_reservation(gg):
    a = gg.GrowableArray(2, 32, dtype=np.int32)
    from paper_2209_00103_b200 import _lib
    _lib.lib.gg_set_arena_limit(a._h, 1 << 12)           # 4 KiB of arena
    vals = np.arange(100_000, dtype=np.int32)
    with pytest.raises(gg.ShardInsertError) as e:
        a.push_if(vals, np.ones(len(vals), bool), mode="warp", grid=2)
    assert set(e.value.failures) <= {0, 1} and e.value.failures
    assert all(isinstance(x, MemoryError) for x in e.value.failures.values())
    assert a.total_size == 100_000                        # reservations kept


def test_push_if_repeated_contention(gg):
    """Many repetitions of the contended warp / block appends: a bucket another
    warp is still allocating must be waited for (the once-flag is read with
    acquire order), never written through a missing pointer.  Before the fix
    about 1 run in 150 lost a run of appends."""
    fails = []
    for it in range(60):
        for mode in ("warp", "block"):
            S, fb, grid = (7, 4, 64) if it % 2 else (32, 32, 512)
            rng = np.random.default_rng(10_000 + it)
            n = 100_000
            vals = rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(np.int32)
            pred = rng.random(n) < 0.37
            a = gg.GrowableArray(S, fb, dtype=np.int32)
            a.insert_parallel([np.arange(int(k), dtype=np.int32) for k in rng.integers(0, 100, S)])
            pre = [a.shards[s].size for s in range(S)]
            a.push_if(vals, pred, mode=mode, grid=grid)
            exp = _expected(vals, pred, S, grid)
            for s in range(S):
                if not np.array_equal(np.sort(a.shards[s].to_numpy()[pre[s]:]), exp[s]):
                    fails.append((it, mode, s))
            a.close()
    assert not fails, fails[:5]


def test_push_if_chained_calls(gg):
    """Consecutive push_if calls whose appends cannot fail chain: each plans on
    the previous calls' upper bounds and headroom without waiting for their
    readback.  12 calls per array (block / warp, several grids and
    densities); with max_buckets = 12 some calls' upper bounds exceed the
    bucket table, so they take the synchronous path mid-chain, which settles
    the calls before them.  Every shard holds the multiset of its appends,
    sizes / capacities / flags are the minimal bucket prefix, and the
    headroom is returned once the chain settles."""
    import torch
    rng = np.random.default_rng(77)
    S, fb = 11, 8
    for mb in (64, 12):
        a = gg.GrowableArray(S, fb, dtype=np.int32, max_buckets=mb)   # 12: 32760 elements per shard
        exp = [[] for _ in range(S)]
        for it in range(12):
            if mb == 12 and it % 4 in (0, 3):
                # one block -> shard 0 only: its upper bound grows by 20000 a
                # call (the third such call in a chain exceeds the table), its
                # appends by ~1000
                n, grid, dens = 20_000, 1, 0.05
            else:
                n = int(rng.integers(1, 60_000 if mb == 64 else 20_000))
                grid, dens = [64, 11, 200, 33][it % 4], [0.5, 0.05, 0.95][it % 3]
            vals = rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(np.int32)
            pred = rng.random(n) < dens
            a.push_if(torch.from_numpy(vals).cuda(), torch.from_numpy(pred).cuda(),
                      mode="block" if it % 2 else "warp", grid=grid, commit=False)
            for s, e in enumerate(_expected(vals, pred, S, grid)):
                exp[s].append(e)
        a.commit()
        st = a._parity_state()
        for s in range(S):
            got = a.shards[s].to_numpy()
            assert np.array_equal(np.sort(got), np.sort(np.concatenate(exp[s]))), (mb, s)
            k = O.min_buckets_for(len(got), fb)
            assert st["sizes"][s] == len(got)
            assert st["caps"][s] == O.capacity_of(k, fb)
            assert st["flags"][s] == (1 << k) - 1
        ms = a.memory_stats()
        assert ms["mapped_bytes"] - ms["bucket_bytes"] < 64 << 20
        a.close()
