"""Paper Alg. 1 with per-lane counts (insert_lanes): the tiled device path
(host backs the upper bound, device reserves once per LFVector and scatters,
sizes come back asynchronously) and the exact two-pass path it falls back to,
both against the oracle (oracle/ggoracle.py) fed with the same compaction --
lane j of shard s appends values[j*K : j*K + counts[j]] in lane order, i.e.
insert_parallel of each shard's compacted batch (insert_index.py:125-143
reservation semantics: one reservation per LFVector with a non-empty batch)."""
import numpy as np
import pytest

from oracle import ggoracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def gg():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a GPU")
    import paper_2209_00103_b200 as gg
    return gg


def _lanes(rng, S, K, max_lanes, empty_every=0):
    lanes = rng.integers(0, max_lanes, S)
    if empty_every:
        lanes[::empty_every] = 0
    lo = np.concatenate([[0], np.cumsum(lanes)]).astype(np.uint64)
    counts = rng.integers(0, K + 1, int(lo[-1])).astype(np.int32)
    return lo, counts


def _compact(vals, counts, lo, K, S):
    out = []
    for s in range(S):
        parts = [vals[j * K: j * K + int(counts[j])] for j in range(int(lo[s]), int(lo[s + 1]))]
        out.append(np.concatenate(parts) if parts else vals[:0])
    return out


def _check(a, o):
    st = a._parity_state()
    ost = o._parity_state()
    for k in ("sizes", "caps", "flags", "prefix", "ops"):
        assert st[k] == ost[k], k
    assert a.flatten().tobytes() == o.flatten().tobytes()


@pytest.mark.parametrize("dtype,K,fb", [("int32", 8, 32), ("int32", 1, 32), ("int32", 3, 32),
                                        ("int8", 5, 16), ("int16", 8, 8), ("int64", 2, 32),
                                        ("float32", 33, 32), ("int32", 8, 1), ("float64", 7, 2),
                                        ("int32", 1000, 32), ("int32", 2, 32), ("int8", 64, 16),
                                        ("int64", 1, 32), ("int16", 16, 32)])
def test_lanes_tiled_matches_oracle(gg, dtype, K, fb):
    import torch
    rng = np.random.default_rng(K * 7 + fb)
    S = 37
    a = gg.GrowableArray(S, fb, dtype=dtype)
    o = O.OracleGGArray(S, fb, dtype=dtype)
    pre = [rng.integers(0, 100, int(x)).astype(dtype) for x in rng.integers(0, 60, S)]
    a.insert_parallel(pre)
    o.insert_parallel(pre)
    for rnd in range(3):                 # consecutive inserts: each resolves the previous one
        lo, counts = _lanes(rng, S, K, 3000 if K < 100 else 40, empty_every=5)
        vals = (rng.integers(-1000, 1000, int(lo[-1]) * K)).astype(dtype)
        a.insert_lanes(torch.from_numpy(vals).cuda(), counts, lo, values_per_lane=K, commit=(rnd == 2))
        o.insert_parallel(_compact(vals, counts, lo, K, S))
    _check(a, o)


def test_lanes_tiled_large_multi_tile(gg):
    """Shards with thousands of tiles (2^22 lanes), counts with long zero runs."""
    import torch
    S, K = 64, 8
    a = gg.GrowableArray(S, 32, dtype=np.int32)
    L = 1 << 22
    lo = np.linspace(0, L, S + 1).astype(np.uint64)
    g = torch.Generator(device="cuda").manual_seed(3)
    cnt = torch.randint(0, K + 1, (L,), device="cuda", generator=g, dtype=torch.int32)
    cnt[: L // 8] = 0
    vals = torch.arange(L * K, dtype=torch.int32, device="cuda")
    a.insert_lanes(vals, cnt, lo, K)
    mask = torch.arange(K, device="cuda")[None, :] < cnt[:, None]
    exp = vals.view(L, K)[mask]
    assert torch.equal(a.flatten_device(), exp)
    sizes = a._parity_state()["sizes"]
    per = cnt.view(S, -1).sum(1).cpu().numpy() if L % S == 0 else None
    assert sizes == [int(x) for x in per]


def test_lanes_counts_clamped_to_values_per_lane(gg):
    import torch
    S, K = 4, 4
    a = gg.GrowableArray(S, 32, dtype=np.int32)
    lo = np.array([0, 3, 3, 5, 6], np.uint64)
    counts = np.array([9, 1, 4, 0, 7, 2], np.int32)     # 9 and 7 > K: clamped to K
    vals = np.arange(6 * K, dtype=np.int32)
    a.insert_lanes(torch.from_numpy(vals).cuda(), counts, lo, K)
    assert a._parity_state()["sizes"] == [4 + 1 + 4, 0, 0 + 4, 2]


def test_lanes_exact_path_with_allocator_hook(gg):
    """An allocator hook makes every allocation host-visible in (shard, bucket)
    order: the exact two-pass path runs, with the same result."""
    import torch
    rng = np.random.default_rng(4)
    S, K = 9, 4
    calls = []

    def alloc(n):
        calls.append(n)
        return np.zeros(n, np.int32)
    a = gg.GrowableArray(S, 32, dtype=np.int32, allocator=alloc)
    o = O.OracleGGArray(S, 32, dtype=np.int32)
    lo, counts = _lanes(rng, S, K, 500)
    vals = np.arange(int(lo[-1]) * K, dtype=np.int32)
    a.insert_lanes(torch.from_numpy(vals).cuda(), counts, lo, K)
    o.insert_parallel(_compact(vals, counts, lo, K, S))
    _check(a, o)
    assert len(calls) == o._parity_state()["alloc_calls"]


def test_lanes_capacity_bound_takes_exact_path(gg):
    """max_buckets small enough that the upper bound would not fit but the
    actual counts do: the exact path inserts without error."""
    import torch
    S, K = 2, 64
    a = gg.GrowableArray(S, 4, dtype=np.int32, max_buckets=4)     # capacity 60 per shard
    lo = np.array([0, 2, 4], np.uint64)
    counts = np.array([10, 5, 0, 30], np.int32)
    vals = np.arange(4 * K, dtype=np.int32)
    a.insert_lanes(torch.from_numpy(vals).cuda(), counts, lo, K)
    assert a._parity_state()["sizes"] == [15, 30]


def test_lanes_footprint_settles(gg):
    """The upper-bound backing is returned once the sizes are known: the
    settled mapped bytes stay within 2x needed (+ the packed small-class
    granule) for a K = 8 insert with counts averaging K/2."""
    import torch
    S, K, L = 512, 8, 1 << 22
    a = gg.GrowableArray(S, 32, dtype=np.int32)
    lo = (np.arange(S + 1, dtype=np.uint64) * np.uint64(L // S))
    cnt = torch.randint(0, K + 1, (L,), device="cuda", dtype=torch.int32)
    vals = torch.arange(L * K, dtype=torch.int32, device="cuda")
    a.insert_lanes(vals, cnt, lo, K)
    ms = a.memory_stats()
    assert ms["mapped_bytes"] <= 2 * ms["needed_bytes"] + (2 << 20)


@pytest.mark.parametrize("K,shift", [(1, 1), (4, 3), (8, 2)])
def test_lanes_values_not_16B_aligned(gg, K, shift):
    """Value blocks that do not start on a 16 B boundary cannot be streamed
    by the bulk copy (k_lanes_bulk): every tile takes the register path (K = 1)
    or the exact two-pass path (lanes wider than their alignment); the result
    is the same compaction."""
    import torch
    rng = np.random.default_rng(K + shift)
    S = 21
    a = gg.GrowableArray(S, 32, dtype=np.int32)
    o = O.OracleGGArray(S, 32, dtype=np.int32)
    lo, counts = _lanes(rng, S, K, 9000, empty_every=4)
    n = int(lo[-1]) * K
    base = torch.arange(n + shift, dtype=torch.int32, device="cuda") * 3 - 7
    vals = base[shift:]                                 # 4 B aligned, not 16 B
    a.insert_lanes(vals, counts, lo, values_per_lane=K)
    o.insert_parallel(_compact(vals.cpu().numpy(), counts, lo, K, S))
    _check(a, o)


def test_lanes_chained_calls(gg):
    """Consecutive tiled lanes inserts chain without a host round trip (each
    plans on the previous calls' upper bounds, kLanesChain = 8 pending at
    most): 20 calls with mixed widths, element-sized ragged shards, a call
    that must take the exact path mid-chain (unaligned values) and calls on a
    second stream; sizes, capacities, bucket flags, ops and contents equal
    the oracle fed the same compactions in order, and the upper-bound
    backing is returned once the chain resolves."""
    import torch
    rng = np.random.default_rng(2024)
    S, fb = 29, 8
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    o = O.OracleGGArray(S, fb, dtype=np.int32)
    side = torch.cuda.Stream()
    for rnd in range(20):
        K = [1, 2, 4, 8, 16, 3][rnd % 6]
        lo, counts = _lanes(rng, S, K, [5, 300, 4000][rnd % 3], empty_every=3 + rnd % 4)
        n = int(lo[-1]) * K
        shift = 1 if rnd == 11 else 0                  # 4 B aligned only: exact path mid-chain
        base = torch.from_numpy(rng.integers(-2**31, 2**31 - 1, n + shift).astype(np.int32)).cuda()
        vals = base[shift:]
        if rnd in (6, 7, 15):
            torch.cuda.current_stream().synchronize()
            with torch.cuda.stream(side):
                a.insert_lanes(vals, counts, lo, values_per_lane=K, commit=False)
        else:
            a.insert_lanes(vals, counts, lo, values_per_lane=K, commit=False)
        o.insert_parallel(_compact(vals.cpu().numpy(), counts, lo, K, S))
    a.commit()
    o.commit()
    _check(a, o)
    ms = a.memory_stats()
    assert ms["mapped_bytes"] <= 2 * ms["needed_bytes"] + (4 << 20)
