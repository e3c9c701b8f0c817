"""Round-2 handle semantics on the device: stream order across streams
(deferred metadata / grow passes never race a call on another stream),
device views block mutating calls, concurrent push_back_batch callers get
the ranges they reserved, reserved-but-unwritten indices read 0 (reference
buckets are np.zeros), and the physical-memory lifecycle (asynchronous unmap
into the pool, slab adoption) keeps contents and footprint exact."""
import threading

import numpy as np
import pytest

from oracle import ggoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gg():
    import paper_2209_00103_b200 as gg
    return gg


def test_grow_and_insert_on_different_streams(gg):
    """grow() deferred on stream A, insert_duplicate() on stream B, flatten on
    A again: the deferred grow / metadata passes are ordered before B's walk
    (ADVICE r01 item 1); contents and tables equal the oracle's."""
    import torch
    S, fb = 128, 32
    init = np.arange(1 << 16, dtype=np.int32)
    a = gg.GrowableArray.from_flat(init, S, fb, dtype=np.int32)
    o = O.OracleGGArray.from_flat(init, S, fb, dtype=np.int32)
    sa, sb = torch.cuda.Stream(), torch.cuda.Stream()
    for r in range(6):
        n = a.committed_size
        with torch.cuda.stream(sa if r % 2 == 0 else sb):
            a.grow(2 * n)
        with torch.cuda.stream(sb if r % 2 == 0 else sa):
            a.insert_duplicate()
        o.grow(2 * n)
        o.insert_duplicate()
    with torch.cuda.stream(sa):
        flat = a.flatten_device()
    sa.synchronize()
    assert flat.cpu().numpy().tobytes() == o.flatten().tobytes()
    st = a._parity_state()
    assert st["sizes"] == [int(x) for x in o.size] and st["caps"] == [int(x) for x in o.capacity]
    masks = [int(sum(1 << b for b in np.flatnonzero(row))) for row in o.flags]
    assert st["flags"] == masks and st["prefix"] == [int(x) for x in o.prefix]


def test_device_view_blocks_mutations(gg):
    """While a device view is out, every mutating call is refused (ValueError)
    and reads still work; device_sync releases it."""
    a = gg.GrowableArray.from_flat(np.arange(4096, dtype=np.int32), 8, 32, dtype=np.int32)
    a.device_view(max_sizes=1024)
    vals = np.arange(8, dtype=np.int32)
    for call in (lambda: a.insert_parallel(gg.split_batches(vals, 8)),
                 lambda: a.insert_duplicate(),
                 lambda: a.grow(10 ** 5),
                 lambda: a.shrink(0),
                 lambda: a.commit(),
                 lambda: a.shards[0].size_counter.fetch_add(1),
                 lambda: a.shards[1].new_bucket(9)):
        with pytest.raises(ValueError, match="device view"):
            call()
    with pytest.raises(ValueError, match="device view"):
        a.device_view(max_sizes=2048)                 # one view at a time
    assert a.flatten().tobytes() == np.arange(4096, dtype=np.int32).tobytes()
    a.device_sync()
    a.insert_duplicate()
    assert a.committed_size == 8192


def test_concurrent_push_back_batch_ranges(gg):
    """64 threads push into ONE shard: the returned ReservedRanges are
    disjoint, cover [0, total) and each holds exactly its caller's values
    (the reference returns the range it reserved)."""
    a = gg.GrowableArray(4, 32, dtype=np.int64)
    sh = a.shards[2]
    out = {}

    def push(t):
        v = np.full(17 + t, t, np.int64)
        out[t] = sh.push_back_batch(v)

    ths = [threading.Thread(target=push, args=(t,)) for t in range(64)]
    for th in ths:
        th.start()
    for th in ths:
        th.join()
    a.commit()
    flat = a.flatten()
    spans = sorted((r.start, r.count, t) for t, r in out.items())
    pos = 0
    for start, count, t in spans:
        assert start == pos and count == 17 + t
        assert (flat[start:start + count] == t).all()
        pos += count
    assert pos == len(flat) == sum(17 + t for t in range(64))


def test_reserved_unwritten_reads_zero(gg):
    """size_counter.fetch_add reserves without writing: the reserved indices
    read 0 after commit even when the bucket's memory held other data (slab
    chunks are recycled through the pool / slab cache)."""
    import torch
    # leave a same-shape slab full of non-zero data behind
    junk = gg.GrowableArray.from_flat(torch.full((1 << 16,), 7, dtype=torch.int32, device="cuda"), 4, 32)
    junk.close()
    gg.reclaim(True)
    a = gg.GrowableArray(4, 32, dtype=np.int32)           # adopts that slab
    assert a.slab_stats()["chunks_mapped"] == 0 and a.memory_stats()["mapped_bytes"] > 0
    sh = a.shards[1]
    sh.reserve(2048)                                      # buckets exist before the reservation
    start = sh.size_counter.fetch_add(1000)
    sh.push_back_batch(np.arange(5, dtype=np.int32) + 1)
    start2 = sh.size_counter.fetch_add(3000)              # reaches buckets allocated later
    sh.push_back_batch(np.arange(3, dtype=np.int32) + 9)
    a.commit()
    got = sh.to_numpy()
    assert start == 0 and start2 == 1005 and len(got) == 4008
    assert (got[:1000] == 0).all() and got[1000:1005].tolist() == [1, 2, 3, 4, 5]
    assert (got[1005:4005] == 0).all() and got[4005:].tolist() == [9, 10, 11]
    # as in the reference, indices whose buckets were never allocated stay unreadable
    b = gg.GrowableArray(4, 32, dtype=np.int32)
    b.shards[0].size_counter.fetch_add(1000)
    b.shards[0].push_back_batch(np.ones(5, np.int32))
    b.commit()
    with pytest.raises(RuntimeError, match="unpublished"):
        b.shards[0].to_numpy()


def test_async_shrink_release_keeps_contents(gg):
    """Shrink with release=True unmaps emptied extents only after the work
    queued before it: a flatten issued right before the shrink still reads
    every element; growth afterwards maps pooled handles; contents exact."""
    import torch
    gg.pool_trim(0)
    vals = torch.arange(1 << 22, dtype=torch.int32, device="cuda")
    a = gg.GrowableArray.from_flat(vals, 64, 32)
    for _ in range(3):
        flat = a.flatten_device()                        # queued; reads the buckets being released
        a.shrink(1 << 10, release=True)
        assert torch.equal(flat, vals)
        ms = a.memory_stats()
        assert ms["pending_unmap_bytes"] == 0 and ms["mapped_bytes"] <= 2 * ms["needed_bytes"] + (64 << 21)
        a.shrink(0, release=False)
        a.insert_csr(vals, np.minimum(np.arange(65, dtype=np.uint64) * np.uint64((1 << 22) // 64), 1 << 22))
    assert a.slab_stats()["handles_from_pool"] > 0
    assert torch.equal(a.flatten_device(), vals)
    a.close()
    gg.pool_trim(0)


def test_uniform_growth_maps_one_extent_per_class(gg):
    """A uniform doubling schedule maps each bucket class region as ONE extent
    (one cuMemCreate/Map per class, not one per grid chunk)."""
    import torch
    gg.pool_trim(0)
    S = 512
    a = gg.GrowableArray.from_flat(torch.arange(1 << 20, dtype=torch.int32, device="cuda"), S, 32)
    for _ in range(6):
        a.grow(2 * a.committed_size)
        a.insert_duplicate()
    st = a.slab_stats()
    classes = int(np.count_nonzero(a._host()["flags"][0] >> np.arange(64, dtype=np.uint64) & np.uint64(1)))
    assert st["chunks_mapped"] <= classes + 1, st     # + the packed small-class region
    n = a.committed_size
    per = (1 << 20) // S << 6
    idx = torch.randint(0, n, (1 << 14,), device="cuda")
    assert torch.equal(a.get_many(idx).to(torch.int64), (idx // per) * ((1 << 20) // S) + idx % ((1 << 20) // S))
    a.close()
