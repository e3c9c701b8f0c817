"""Full-size parity through size-independent properties (BASELINE configs 1-3):
closed-form sizes / capacities (memory_model.py:152-166) and closed-form
contents of the doubling schedule, checked on the device; the oracle checks
the same schedule bit for bit at reduced size."""
import numpy as np
import pytest

from oracle import ggoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gg():
    import paper_2209_00103_b200 as gg
    return gg


def _expected_schedule_state(S, fb, n0, rounds):
    per = n0 // S
    k = O.min_buckets_for(per << rounds, fb)
    return per << rounds, O.capacity_of(k, fb)


def test_config2_reduced_bit_exact_vs_oracle(gg):
    """2^16 -> 2^22 doubling rounds, S=512: grow(2n), duplicate, +1 -- every round."""
    S, fb = 512, 32
    init = np.arange(1 << 16, dtype=np.int32)
    a = gg.GrowableArray.from_flat(init, S, fb)
    o = O.OracleGGArray.from_flat(init, S, fb)
    for r in range(6):
        n = a.committed_size
        a.grow(2 * n); o.grow(2 * n)
        a.insert_duplicate(); o.insert_duplicate()
        a.rw_add(1); o.rw_add(1)
        st = a._parity_state()
        assert st["sizes"] == [int(x) for x in o.size]
        assert st["caps"] == [int(x) for x in o.capacity]
        assert st["prefix"] == [int(x) for x in o.prefix]
    assert a.flatten().tobytes() == o.flatten().tobytes()


def test_config2_full_2p30_closed_form(gg):
    """The BASELINE config-2 schedule at full size: 2^20 -> 2^30 int32, S=512."""
    import torch
    S, fb, n0, rounds = 512, 32, 1 << 20, 10
    a = gg.GrowableArray.from_flat(torch.arange(n0, dtype=torch.int32, device="cuda"), S, fb)
    for r in range(rounds):
        n = a.committed_size
        a.grow(2 * n)
        a.insert_duplicate()
        a.rw_add(1)
        per, cap = _expected_schedule_state(S, fb, n0, r + 1)
        st = a.device_state()
        assert np.all(st["sizes"] == per) and np.all(st["caps"] == cap), r
        ms = a.memory_stats()
        assert ms["capacity_bytes"] == int(O.sharded_capacity_elements([n0 << (r + 1)], S, fb)[0]) * 4
        assert ms["bucket_bytes"] == ms["capacity_bytes"]
    assert a.committed_size == 1 << 30
    ms = a.memory_stats()
    assert ms["capacity_bytes"] == 2_147_467_264 * 4
    assert ms["mapped_bytes"] <= 2 * ms["needed_bytes"]            # paper's <= 2x claim, mapped
    flat = a.flatten_device()
    per = (n0 // S) << rounds
    g = torch.arange(1 << 30, dtype=torch.int64, device="cuda")
    exp = ((g // per) * (n0 // S) + (g % (n0 // S)) + rounds).to(torch.int32)
    del g
    assert torch.equal(flat, exp)


def test_config1_full_vs_reference_hash(gg, golden):
    """Config 1 (512 LFVectors, 2^20 int32 insert, +1 pass, flatten) against the
    hash recorded from the reference."""
    import hashlib
    a = gg.GrowableArray(512, 32, dtype=np.int32)
    a.insert_parallel(gg.split_batches(np.arange(1 << 20, dtype=np.int32), 512))
    a.rw_add(1)
    want = golden["ggarray"]["config1_2p20"]["states"][-1]["flat"]
    assert "sha256:" + hashlib.sha256(a.flatten().tobytes()).hexdigest() == want


def test_ragged_csr_insert_large_misaligned(gg):
    """Random ragged batches (odd sizes -> unaligned source/destination) at 2^22."""
    import torch
    rng = np.random.default_rng(9)
    S, fb = 333, 32
    counts = rng.integers(0, 25000, S)
    counts[rng.random(S) < 0.1] = 0
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    vals = rng.integers(-2**31, 2**31 - 1, int(off[-1]), dtype=np.int64).astype(np.int32)
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    o = O.OracleGGArray(S, fb, dtype=np.int32)
    pre = [np.arange(int(k), dtype=np.int32) for k in rng.integers(0, 77, S)]
    a.insert_parallel(pre); o.insert_parallel(pre)
    a.insert_csr(torch.from_numpy(vals).cuda(), off)
    o.insert_parallel([vals[off[s]:off[s + 1]] for s in range(S)])
    a.insert_duplicate(); o.insert_duplicate()
    assert a.flatten().tobytes() == o.flatten().tobytes()
    assert a._parity_state()["caps"] == [int(x) for x in o.capacity]


@pytest.mark.parametrize("dtype", ["int8", "int16", "int64", "float64"])
def test_element_sizes_misaligned_paths(gg, dtype):
    rng = np.random.default_rng(1)
    S, fb = 7, 1
    counts = rng.integers(0, 5000, S)
    vals = (rng.integers(0, 100, int(counts.sum()))).astype(dtype)
    off = np.concatenate([[0], np.cumsum(counts)])
    batches = [vals[off[s]:off[s + 1]] for s in range(S)]
    a = gg.GrowableArray(S, fb, dtype=dtype)
    o = O.OracleGGArray(S, fb, dtype=dtype)
    for _ in range(3):
        a.insert_parallel(batches); o.insert_parallel(batches)
        a.insert_duplicate(); o.insert_duplicate()
        a.rw_add(1, mode="global"); o.rw_add(1)
    assert a.flatten().tobytes() == o.flatten().tobytes()


def test_slab_release_and_cache(gg):
    """Shrink unmaps slab chunks that lost their last live bucket (footprint
    follows the live capacity down), release=False keeps them cached for
    in-place reuse, trim() returns the cache; contents survive throughout."""
    import torch
    S, fb, n = 512, 32, 1 << 24
    a = gg.GrowableArray.from_flat(torch.arange(n, dtype=torch.int32, device="cuda"), S, fb)
    o_per = n // S
    ms0 = a.memory_stats()
    assert ms0["mapped_bytes"] <= 2 * ms0["needed_bytes"]
    small = n >> 6
    a.shrink(small // S, release=True)
    ms = a.memory_stats()
    assert ms["cached_bytes"] == 0
    assert ms["capacity_bytes"] == int(O.sharded_capacity_elements([small], S, fb)[0]) * 4
    assert ms["mapped_bytes"] <= 2 * ms["needed_bytes"] + (2 << 20)      # + the packed small-class granule
    a.grow(n)
    a.insert_duplicate()                                                   # regrow into fresh chunks
    per = small // S
    g = torch.arange(2 * small, dtype=torch.int64, device="cuda")
    s_, i_ = g // (2 * per), g % (2 * per)
    exp = (s_ * o_per + (i_ % per)).to(torch.int32)
    assert torch.equal(a.flatten_device(), exp)
    mapped_before = a.memory_stats()["mapped_bytes"]
    a.shrink(0, release=False)
    ms = a.memory_stats()
    assert ms["mapped_bytes"] == mapped_before and ms["cached_bytes"] > 0
    a.insert_csr(torch.arange(n, dtype=torch.int32, device="cuda"),
                 np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(o_per), np.uint64(n)))
    assert a.memory_stats()["mapped_bytes"] == mapped_before               # reused in place
    assert torch.equal(a.flatten_device(), torch.arange(n, dtype=torch.int32, device="cuda"))
    a.shrink(0, release=False)
    a.trim()
    ms = a.memory_stats()
    assert ms["cached_bytes"] == 0 and ms["mapped_bytes"] <= 2 << 20


def test_phased_footprint_follows_live_capacity(gg):
    """Config 4 shape at 2^22: after every insert/shrink round the mapped slab
    bytes stay within 2x needed plus one chunk per partly live class."""
    import torch
    rng = np.random.default_rng(0)
    S, fb, n0 = 512, 32, 1 << 22
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    src = torch.arange(4 * n0, dtype=torch.int32, device="cuda")
    off = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(n0 // S), np.uint64(n0))
    a.insert_csr(src[:n0], off)
    n, worst = n0, 0.0
    for _ in range(40):
        target = int(round(rng.uniform(0, 2) * n0))
        q, r = divmod(target, S)
        new = np.full(S, q, np.int64)
        new[:r] += 1
        cur = a._host()["sizes"].astype(np.int64)
        if target >= n:
            d = new - cur
            offs = np.concatenate([[0], np.cumsum(d)]).astype(np.uint64)
            a.insert_csr(src[:int(offs[-1])], offs)
        else:
            a.shrink(new)                       # default policy: keep mapped <= 2x needed
        n = target
        ms = a.memory_stats()
        if target >= n0 // 8:
            worst = max(worst, ms["mapped_bytes"] / ms["needed_bytes"])
            assert ms["mapped_bytes"] <= 2 * ms["needed_bytes"] + (8 << 20)
    assert worst <= 2.5


@pytest.mark.parametrize("unroll", [1, 2, 4, 8])
def test_walk_tile_sizes_ragged_parity(gg, unroll):
    """Every tile size of the one-tile-per-CTA walker (U = 1..8 vectors per
    thread) on ragged, misaligned shards: CSR insert, duplicate, rw (per shard
    and global), flatten -- bit-exact against the oracle."""
    import torch
    from paper_2209_00103_b200 import _lib
    rng = np.random.default_rng(100 + unroll)
    S, fb = 97, 8
    counts = rng.integers(0, 40000, S)
    counts[rng.random(S) < 0.15] = 0
    counts[5] = 1
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    vals = rng.integers(-2**31, 2**31 - 1, int(off[-1]), dtype=np.int64).astype(np.int32)
    _lib.check(_lib.lib.gg_set_tuning(-1, unroll, 0, 0))
    try:
        a = gg.GrowableArray(S, fb, dtype=np.int32)
        o = O.OracleGGArray(S, fb, dtype=np.int32)
        pre = [np.arange(int(k), dtype=np.int32) for k in rng.integers(0, 33, S)]
        a.insert_parallel(pre); o.insert_parallel(pre)
        a.insert_csr(torch.from_numpy(vals).cuda(), off)
        o.insert_parallel([vals[off[s]:off[s + 1]] for s in range(S)])
        a.insert_duplicate(); o.insert_duplicate()
        a.rw_add(3); o.rw_add(3)
        a.rw_add(-1, mode="global"); o.rw_add(-1)
        assert a.flatten().tobytes() == o.flatten().tobytes()
        assert a._parity_state()["sizes"] == [int(x) for x in o.size]
    finally:
        _lib.lib.gg_set_tuning(-1, -1, 0, 0)


@pytest.mark.parametrize("dtype", ["int32", "int8", "float64"])
def test_flatten_range_slices(gg, dtype):
    """flatten_range(lo, hi) == flatten()[lo:hi] for random (misaligned) ranges,
    including empty, single-element and full ranges; IndexError past the end."""
    import torch
    rng = np.random.default_rng(7)
    S, fb = 29, 4
    counts = rng.integers(0, 3000, S)
    counts[::7] = 0
    vals = (rng.integers(0, 120, int(counts.sum()))).astype(dtype)
    off = np.concatenate([[0], np.cumsum(counts)])
    a = gg.GrowableArray(S, fb, dtype=dtype)
    a.insert_parallel([vals[off[s]:off[s + 1]] for s in range(S)])
    a.insert_duplicate()
    full = a.flatten()
    n = len(full)
    cases = [(0, n), (0, 0), (n, n), (5, 6), (n - 1, n)] + [tuple(sorted(rng.integers(0, n + 1, 2))) for _ in range(20)]
    for lo, hi in cases:
        got = a.flatten_range(int(lo), int(hi)).cpu().numpy()
        assert got.tobytes() == full[lo:hi].tobytes(), (lo, hi)
    with pytest.raises(IndexError):
        a.flatten_range(0, n + 1)


@pytest.mark.parametrize("defer,rounds", [(True, 5), (True, 4), (False, 5)])
def test_captured_schedule_replays_match_eager(gg, defer, rounds):
    """GrowableArray.capture (deferred metadata kept on and flushed in-capture)
    and plain capture_mode: replays of reset + insert + doubling rounds end
    in the eager state, device tables == host mirror, contents == closed form."""
    import torch
    S, fb, n0 = 64, 32, 1 << 14                # rounds 4: an odd number of fused walks (parity restore)
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    src = torch.arange(n0, dtype=torch.int32, device="cuda")
    off = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(n0 // S), np.uint64(n0))

    def step():
        a.shrink(0, release=False)
        a.insert_csr(src, off)
        for _ in range(rounds):
            a.grow(2 * a.committed_size)
            a.insert_duplicate()

    step()
    torch.cuda.synchronize()
    if defer:
        g = a.capture(step)
    else:
        g = torch.cuda.CUDAGraph()
        with a.capture_mode():
            with torch.cuda.graph(g):
                step()
    for _ in range(3):
        g.replay()
    torch.cuda.synchronize()
    dev, host = a.device_state(), a._host()     # device tables == host mirror (ops counts replays)
    for k in ("sizes", "caps", "flags", "prefix"):
        assert np.array_equal(dev[k], host[k]), k
    assert int(dev["prefix"][-1]) == n0 << rounds
    per = (n0 // S) << rounds
    idx = torch.arange(n0 << rounds, device="cuda")
    exp = ((idx // per) * (n0 // S) + idx % (n0 // S)).to(torch.int32)
    assert torch.equal(a.flatten_device(), exp)


def test_dropped_arrays_free_at_once(gg):
    """No reference cycle keeps a GrowableArray alive: dropping it (gc off)
    destroys the handle immediately -- shards views, size counters, the
    allocator hook and device views included -- and its memory is reclaimed
    stream-ordered, without a cyclic-GC pass landing in someone's timed loop."""
    import gc
    import weakref
    import torch
    gc.collect()
    gc.disable()
    try:
        gg.pool_trim(0)
        vals = torch.arange(1 << 16, dtype=torch.int32, device="cuda")
        for i in range(4):
            a = gg.GrowableArray.from_flat(vals, 64, 32, allocator=lambda n: None)
            _ = [sh.size_counter for sh in a.shards]             # counters cached in the array
            _ = a.shards[3].table.allocated_flags
            a.rw_add(1)
            r = weakref.ref(a)
            del a, _
            assert r() is None, "GrowableArray kept alive by a reference cycle"
            gg.reclaim(True)
            st = gg.pool_stats(0)
            assert st["graves"] == 0 and st["slabs_cached"] == 1, st
    finally:
        gc.enable()
        gg.pool_trim(0)


def test_chunk_pool_reuse_and_trim(gg):
    """Shrink releases go to the process pool (asynchronously), growth maps
    pooled handles, destroyed arrays leave their whole slab for a same-shape
    successor, trim empties everything."""
    import gc
    import torch
    gc.collect()                       # earlier tests' arrays die now, not mid-test
    gc.disable()
    try:
        _chunk_pool_body(gg, torch)
    finally:
        gc.enable()


def _chunk_pool_body(gg, torch):
    """Physical-memory lifecycle: a shrink unmaps released extents
    asynchronously into the process pool; the next growth maps pooled
    handles (no cuMemCreate); a destroyed array's slab is kept whole and a
    same-shape array adopts it with no driver call at all."""
    gg.pool_trim(0)
    s0 = gg.pool_stats(0)
    assert s0["cached_bytes"] == 0 and s0["slab_cache_bytes"] == 0 and s0["cap_bytes"] > 0
    vals = torch.arange(1 << 20, dtype=torch.int32, device="cuda")
    offs = np.minimum(np.arange(65, dtype=np.uint64) * np.uint64((1 << 20) // 64), 1 << 20)
    a = gg.GrowableArray.from_flat(vals, 64, 32)
    mapped0 = a.memory_stats()["mapped_bytes"]
    created0 = a.slab_stats()["handles_created"]
    assert mapped0 > 0 and created0 > 0
    a.shrink(0, release=True)
    ms = a.memory_stats()                                    # settles the asynchronous unmap
    assert ms["mapped_bytes"] == 0 and ms["pending_unmap_bytes"] == 0
    assert gg.pool_stats(0)["cached_bytes"] == mapped0       # released handles -> the pool
    a.insert_csr(vals, offs)
    st = a.slab_stats()
    assert st["handles_created"] == created0 and st["handles_from_pool"] > 0
    assert a.memory_stats()["mapped_bytes"] == mapped0
    a.close()
    gg.reclaim(True)
    p1 = gg.pool_stats(0)
    assert p1["slab_cache_bytes"] == mapped0 and p1["slabs_cached"] == 1
    b = gg.GrowableArray.from_flat(vals * 3, 64, 32)          # same shape: adopts the slab
    sb = b.slab_stats()
    assert gg.pool_stats(0)["slab_cache_hits"] == p1["slab_cache_hits"] + 1
    assert sb["handles_created"] == 0 and sb["handles_from_pool"] == 0 and sb["chunks_mapped"] == 0
    assert torch.equal(b.flatten_device(), vals * 3)
    assert b.memory_stats()["mapped_bytes"] == mapped0
    c = gg.GrowableArray.from_flat(vals, 32, 32)              # another shape: no adoption
    assert c.slab_stats()["handles_created"] + c.slab_stats()["handles_from_pool"] > 0
    assert torch.equal(c.flatten_device(), vals)
    b.close()
    c.close()
    gg.pool_trim(0)
    p2 = gg.pool_stats(0)
    assert p2["cached_bytes"] == 0 and p2["slab_cache_bytes"] == 0 and p2["graves"] == 0


@pytest.mark.parametrize("S", [1025, 5000, 70000])
def test_many_shards_ragged(gg, S):
    """Shard counts past one CTA of metadata threads and past two levels of
    the 32-ary directory search: ragged insert, duplicate, +1 (per shard and
    global), flatten and capacities against a direct numpy construction."""
    import torch
    rng = np.random.default_rng(S)
    fb = 4
    counts = rng.integers(0, 40, S)
    counts[rng.random(S) < 0.3] = 0
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    vals = rng.integers(-1000, 1000, int(off[-1])).astype(np.int32)
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    a.insert_csr(torch.from_numpy(vals).cuda(), off)
    a.insert_duplicate()
    a.rw_add(1)
    a.rw_add(2, mode="global")
    want = np.concatenate([np.concatenate([vals[off[s]:off[s + 1]]] * 2) for s in range(S)]) + 3
    assert a.flatten().tobytes() == want.astype(np.int32).tobytes()
    st = a.device_state()
    sizes = 2 * counts
    assert np.array_equal(st["sizes"], sizes)
    assert np.array_equal(st["caps"], [O.capacity_of(O.min_buckets_for(int(n), fb), fb) for n in sizes])
    assert int(st["prefix"][-1]) == int(sizes.sum())
    g = torch.from_numpy(rng.integers(0, int(sizes.sum()), 4096)).cuda()
    assert torch.equal(a.get_many(g).cpu(), torch.from_numpy(want[g.cpu().numpy()]))


@pytest.mark.parametrize("S", [3000, 40000])
def test_many_shards_uniform_doubling(gg, S):
    """The uniform fast paths (grow, duplicate, deferred metadata fused into
    the next grow) with more shards than one metadata CTA has threads."""
    import torch
    fb, per0, rounds = 8, 12, 5
    n0 = S * per0
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    a.insert_csr(torch.arange(n0, dtype=torch.int32, device="cuda"),
                 np.arange(S + 1, dtype=np.uint64) * np.uint64(per0))
    for _ in range(rounds):
        a.grow(2 * a.committed_size)
        a.insert_duplicate()
    per = per0 << rounds
    st = a.device_state()
    assert np.all(st["sizes"] == per) and int(st["prefix"][-1]) == S * per
    assert np.all(st["caps"] == O.capacity_of(O.min_buckets_for(per, fb), fb))
    g = torch.arange(S * per, device="cuda")
    assert torch.equal(a.flatten_device(), ((g // per) * per0 + g % per0).to(torch.int32))


@pytest.mark.parametrize("dtype,fb,S", [("int8", 1, 3), ("int64", 1, 5), ("uint16", 2, 130), ("float64", 64, 7)])
def test_large_ragged_dtypes(gg, dtype, fb, S):
    """Large ragged shards with 1/2/8-byte elements and tiny first buckets
    (up to ~25 buckets per shard): insert, duplicate, +1 passes, flatten and
    capacities against direct numpy construction."""
    import torch
    rng = np.random.default_rng(fb * 100 + S)
    counts = rng.integers(1 << 18, 1 << 21, S)
    counts[0] = 1
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    vals = rng.integers(0, 100, int(off[-1])).astype(dtype)
    a = gg.GrowableArray(S, fb, dtype=dtype)
    a.insert_csr(torch.from_numpy(vals).cuda(), off)
    a.insert_duplicate()
    a.rw_add(1)
    a.rw_add(1, mode="global")
    one = np.asarray(2, dtype=dtype)
    want = np.concatenate([np.concatenate([vals[off[s]:off[s + 1]]] * 2) for s in range(S)])
    want = (want + one).astype(dtype)
    assert a.flatten().tobytes() == want.tobytes()
    st = a.device_state()
    assert np.array_equal(st["caps"], [O.capacity_of(O.min_buckets_for(2 * int(c), fb), fb) for c in counts])


def test_deferred_grow_is_flushed_by_every_device_reader(gg):
    """A uniform grow is deferred into the next append's metadata CTA; any
    other call that reads or writes device state must see it applied."""
    import torch
    S, fb = 16, 8
    a = gg.GrowableArray.from_flat(np.arange(16 * 100, dtype=np.int32), S, fb)
    o = O.OracleGGArray.from_flat(np.arange(16 * 100, dtype=np.int32), S, fb)
    checks = [
        lambda: a.device_state(),                                   # device tables read back
        lambda: a.shards[3].table.buckets,                          # bucket pointers
        lambda: a.get_global(5),                                    # single element
        lambda: a.flatten(),                                        # walk
        lambda: a.rw_add(0),                                        # walk in place
        lambda: a.commit(),                                         # commit kernel
    ]
    for i, chk in enumerate(checks):
        a.grow((3 + i) * a.committed_size)
        o.grow((3 + i) * o.committed_size)
        chk()
        st = a.device_state()
        assert [int(x) for x in st["caps"]] == [int(x) for x in o.capacity], i
        assert [int(x) for x in st["flags"]] == [int(sum(1 << b for b in range(o.mb) if o.flags[s, b]))
                                                 for s in range(S)], i
    # a deferred grow followed by a non-uniform append (ragged) and a shrink
    a.grow(2 * a.committed_size); o.grow(2 * o.committed_size)
    batches = [np.arange(s * 7, dtype=np.int32) for s in range(S)]
    a.insert_parallel(batches); o.insert_parallel(batches)
    a.grow(4 * a.committed_size); o.grow(4 * o.committed_size)
    a.shrink(np.full(S, 50)); o.shrink(np.full(S, 50))
    st = a._parity_state()
    assert st["sizes"] == [int(x) for x in o.size] and st["caps"] == [int(x) for x in o.capacity]
    assert a.flatten().tobytes() == o.flatten().tobytes()


@pytest.mark.parametrize("fuse", [1, 0])
@pytest.mark.parametrize("S", [64, 4100])
def test_uniform_insert_fast_path_vs_oracle(gg, fuse, S):
    """Uniform CSR inserts over uniform shards take the plan-shard-0-once path
    (fused metadata CTA, or the unfused walk + metadata kernel when the CTA is
    off / S > 4096); interleaved with duplicates, grows and a shrink, the
    state and contents equal the oracle's."""
    import torch
    from paper_2209_00103_b200 import _lib as L
    fb = 8
    L.lib.gg_set_fuse(fuse)
    try:
        a = gg.GrowableArray(S, fb, dtype=np.int32)
        o = O.OracleGGArray(S, fb, dtype=np.int32)
        base = 0
        for step, c in enumerate([3, 8, 13, 40, 1, 100]):
            vals = np.arange(base, base + c * S, dtype=np.int32)
            base += c * S
            offs = np.arange(S + 1, dtype=np.uint64) * np.uint64(c)
            a.insert_csr(torch.from_numpy(vals).cuda(), offs)
            o.insert_parallel([vals[s * c:(s + 1) * c] for s in range(S)])
            if step % 2:
                a.insert_duplicate(); o.insert_duplicate()
            if step == 3:
                a.grow(4 * a.committed_size); o.grow(4 * o.committed_size)
            if step == 4:
                a.shrink(17, release=False); o.shrink(np.full(S, 17))
            st = a._parity_state()
            assert st["sizes"] == [int(x) for x in o.size], step
            assert st["caps"] == [int(x) for x in o.capacity], step
            assert st["prefix"] == [int(x) for x in o.prefix], step
        assert a.flatten().tobytes() == o.flatten().tobytes()
        dev = a.device_state()
        assert np.array_equal(dev["sizes"], a._host()["sizes"])
    finally:
        L.lib.gg_set_fuse(1)


@pytest.mark.parametrize("dtype", [np.int8, np.int32, np.float64])
def test_short_piece_tiles_vs_oracle(gg, dtype):
    """Tiles covering many LFVectors with a few elements each take the
    element-by-element walk (insert, duplicate, r/w, flatten, flatten_range):
    uniform 1 element per shard, then ragged 0..5 per shard, with a failing
    allocator hook (the unplanned, per-shard-controlled walk) in between."""
    import torch
    from paper_2209_00103_b200 import ShardInsertError
    S, fb = 1000, 2
    rng = np.random.default_rng(7)
    a = gg.GrowableArray(S, fb, dtype=dtype)
    o = O.OracleGGArray(S, fb, dtype=dtype)
    one = np.arange(S).astype(dtype)
    a.insert_parallel([one[s:s + 1] for s in range(S)]); o.insert_parallel([one[s:s + 1] for s in range(S)])
    for r in range(3):
        cnt = rng.integers(0, 6, S)
        vals = rng.integers(0, 100, int(cnt.sum())).astype(dtype)
        off = np.concatenate([[0], np.cumsum(cnt)])
        batches = [vals[off[s]:off[s + 1]] for s in range(S)]
        a.insert_parallel(batches); o.insert_parallel(batches)
        a.insert_duplicate(); o.insert_duplicate()
        a.rw_add(1); o.rw_add(1)
        mode = ("fused", "global", "per_shard")[r]
        a.rw_add(3, passes=3, mode=mode); o.rw_add(3, passes=3)
        st = a._parity_state()
        assert st["sizes"] == [int(x) for x in o.size], r
        assert st["prefix"] == [int(x) for x in o.prefix], r
        assert a.flatten().tobytes() == o.flatten().tobytes(), r
    n = a.committed_size
    lo, hi = 123, n - 77
    assert np.array_equal(a.flatten_range(lo, hi).cpu().numpy(), o.flatten()[lo:hi])
    # failing allocator on every 3rd shard's next bucket: unplanned walk with ctl words
    calls = {"n": 0}

    def alloc(nelem):
        calls["n"] += 1
        if calls["n"] % 3 == 0:
            raise MemoryError("injected")
        return np.zeros(nelem, dtype)
    b = gg.GrowableArray(S, fb, dtype=dtype, allocator=alloc)
    ob = O.OracleGGArray(S, fb, dtype=dtype, allocator=alloc)
    batches = [np.full(3, s % 100, dtype) for s in range(S)]
    calls["n"] = 0
    with pytest.raises(ShardInsertError) as e1:
        b.insert_parallel(batches)
    calls["n"] = 0
    with pytest.raises(O.ShardInsertError) as e2:
        ob.insert_parallel(batches)
    assert sorted(e1.value.failures) == sorted(e2.value.failures)
    assert b._parity_state()["sizes"] == [int(x) for x in ob.size]
