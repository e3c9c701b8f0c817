"""Parity of the B200 drop-in against the reference-generated goldens and the CPU
oracle.  Every state compared here is read back from DEVICE memory
(``_parity_state`` asserts the host mirror agrees with it)."""
import json
import os

import numpy as np
import pytest

import scenarios
from oracle import ggoracle as O

pytestmark = pytest.mark.gpu

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


@pytest.fixture(scope="module")
def gg():
    import paper_2209_00103_b200 as gg
    return gg


@pytest.mark.parametrize("name", sorted(GOLDEN["ggarray"]))
def test_golden_scenario_bit_exact(gg, name):
    case = GOLDEN["ggarray"][name]
    got = scenarios.run_scenario(gg, case["ops"])
    for k, (g, want) in enumerate(zip(got, case["states"])):
        assert g == want, f"{name} step {k} ({case['ops'][k]})"


@pytest.mark.parametrize("name", sorted(GOLDEN["baselines"]))
def test_golden_baselines(gg, name):
    case = GOLDEN["baselines"][name]
    got = scenarios.run_baseline_scenario(gg, case["ops"])
    for k, (g, want) in enumerate(zip(got, case["states"])):
        assert g == want, f"{name} step {k}"


@pytest.mark.parametrize("seed", range(24))
def test_random_scenarios_vs_oracle(gg, seed):
    ops = scenarios._random_scenario(500 + seed)
    assert scenarios.run_scenario(gg, ops) == scenarios.run_scenario(O, ops)


@pytest.mark.parametrize("mode", ["per_shard", "global", "fused"])
@pytest.mark.parametrize("dtype", ["int32", "int64", "float32", "float64", "int8", "uint16", "float16"])
def test_rw_modes_agree_with_oracle(gg, mode, dtype):
    rng = np.random.default_rng(3)
    S, fb = 37, 4
    sizes = rng.integers(0, 3000, S)
    sizes[::5] = 0
    vals = (np.arange(sizes.sum()) % 1000).astype(dtype)
    off = np.concatenate([[0], np.cumsum(sizes)])
    batches = [vals[off[s]:off[s + 1]] for s in range(S)]
    a = gg.GrowableArray(S, fb, dtype=dtype)
    o = O.OracleGGArray(S, fb, dtype=dtype)
    a.insert_parallel(batches)
    o.insert_parallel(batches)
    a.rw_add(3, passes=5, mode=mode)
    o.rw_add(3, passes=5)
    assert a.flatten().tobytes() == o.flatten().tobytes()


def test_get_many_set_many(gg):
    a = gg.GrowableArray.from_flat(np.arange(100000, dtype=np.int64), shards=13, first_bucket_size=8)
    idx = np.random.default_rng(0).integers(0, 100000, 5000)
    assert np.array_equal(a.get_many(idx).cpu().numpy(), idx)
    a.set_many(idx, -idx)
    flat = a.flatten()
    ref = np.arange(100000)
    ref[idx] = -idx
    assert np.array_equal(flat, ref)
    with pytest.raises(IndexError):
        a.get_many([100000])


@pytest.mark.parametrize("dtype", [np.int8, np.int16, np.float32, np.int64])
def test_get_many_checked_in_kernel(gg, dtype):
    """get_many's bounds check rides in the gather kernel (gg_gather_checked):
    one bad index anywhere in a large batch, negative indices, an empty
    array -> IndexError (get_global, sharded_array.py:152-155); the array and
    later gathers are unaffected."""
    import ctypes as C
    import torch
    from paper_2209_00103_b200 import _lib as L
    n = 300007
    vals = (np.arange(n) % 120).astype(dtype)
    a = gg.GrowableArray.from_flat(vals, shards=37, first_bucket_size=16)
    rng = np.random.default_rng(3)
    idx = rng.integers(0, n, 1 << 18)
    assert np.array_equal(a.get_many(idx).cpu().numpy(), vals[idx])
    for bad in (n, n + 12345, -1, -(1 << 40)):
        j = idx.copy()
        j[rng.integers(0, j.size)] = bad
        with pytest.raises(IndexError):
            a.get_many(j)
    assert np.array_equal(a.get_many(idx[:1000]).cpu().numpy(), vals[idx[:1000]])
    assert a.get_many(np.zeros(0, np.int64)).numel() == 0
    # the C-ABI entry directly: GG_EINDEX, and GG_OK on in-range indices
    d = torch.as_tensor(np.array([0, n - 1, n], np.int64), device="cuda")
    out = torch.empty(3, dtype=torch.from_numpy(vals[:1]).dtype, device="cuda")
    assert L.lib.gg_gather_checked(a._h, C.c_void_p(d.data_ptr()), 3, C.c_void_p(out.data_ptr()),
                                   a._stream()) == L.GG_EINDEX
    assert L.lib.gg_gather_checked(a._h, C.c_void_p(d.data_ptr()), 2, C.c_void_p(out.data_ptr()),
                                   a._stream()) == L.GG_OK
    assert out[:2].cpu().numpy().tolist() == [vals[0], vals[n - 1]]
    e = gg.GrowableArray(4, 8, dtype=dtype)
    with pytest.raises(IndexError):
        e.get_many([0])
    with pytest.raises(IndexError):
        e.set_many([0], np.zeros(1, dtype))


@pytest.mark.parametrize("dtype", [np.int8, np.float32, np.int64])
def test_set_many_checked_no_partial_update(gg, dtype):
    """set_many (gg_scatter_checked): a bounds pass flags any index outside
    the committed size and the scatter behind it writes NOTHING (set_global,
    sharded_array.py:156-158, raises before touching the array); a clean
    batch lands exactly (distinct targets), odd lengths and unaligned index
    slices included."""
    n = 200003
    vals = (np.arange(n) % 100).astype(dtype)
    a = gg.GrowableArray.from_flat(vals, shards=29, first_bucket_size=8)
    rng = np.random.default_rng(9)
    idx = rng.permutation(n)[:(1 << 16) + 1]
    new = (rng.integers(0, 100, idx.size)).astype(dtype)
    for bad in (n, -1, 1 << 50):
        j = idx.copy()
        j[rng.integers(0, j.size)] = bad
        with pytest.raises(IndexError):
            a.set_many(j, new)
        assert np.array_equal(a.flatten(), vals)          # untouched
    import torch
    dj = torch.as_tensor(np.concatenate([[0], idx]), device="cuda")[1:]   # 8 B-aligned, not 16 B
    a.set_many(dj, new)
    want = vals.copy()
    want[idx] = new
    assert np.array_equal(a.flatten(), want)
    a.set_many(np.zeros(0, np.int64), np.zeros(0, dtype))
    assert np.array_equal(a.flatten(), want)


def test_lanes_insert_matches_compaction(gg):
    import torch
    rng = np.random.default_rng(11)
    S, K = 19, 3
    lanes = rng.integers(0, 4000, S)
    lo = np.concatenate([[0], np.cumsum(lanes)]).astype(np.uint64)
    L = int(lo[-1])
    counts = rng.integers(0, K + 1, L).astype(np.int32)
    vals = np.arange(L * K, dtype=np.int32)
    a = gg.GrowableArray(S, 32, dtype=np.int32)
    a.insert_parallel([np.arange(int(x), dtype=np.int32) for x in rng.integers(0, 50, S)])
    before = [a.shards[s].to_numpy() for s in range(S)]
    a.insert_lanes(torch.from_numpy(vals).cuda(), counts, lo, values_per_lane=K)
    for s in range(S):
        exp = [before[s]]
        for j in range(int(lo[s]), int(lo[s + 1])):
            exp.append(vals[j * K: j * K + counts[j]])
        assert np.array_equal(a.shards[s].to_numpy(), np.concatenate(exp)), s
    st = a._parity_state()
    assert st["sizes"] == [len(b) + int(counts[int(lo[s]):int(lo[s + 1])].sum()) for s, b in enumerate(before)]


def test_predicated_push_back_one_value_per_lane(gg):
    # the paper's Alg. 1: each thread pushes its element iff its predicate holds
    S = 8
    n = 1 << 16
    vals = np.arange(n, dtype=np.int32)
    keep = (vals % 3 == 0).astype(np.int32)
    lo = np.linspace(0, n, S + 1).astype(np.uint64)
    a = gg.GrowableArray(S, 32, dtype=np.int32)
    a.insert_lanes(vals, keep, lo)
    exp = np.concatenate([vals[int(lo[s]):int(lo[s + 1])][keep[int(lo[s]):int(lo[s + 1])] == 1]
                          for s in range(S)])
    assert np.array_equal(a.flatten(), exp)


def test_shrink_matches_oracle_model(gg):
    rng = np.random.default_rng(5)
    S, fb = 16, 4
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    o = O.OracleGGArray(S, fb, dtype=np.int32)
    tag = 0
    for _ in range(12):
        if rng.random() < 0.5 or not a.committed_size:
            sizes = rng.integers(0, 400, S)
            batches = [np.arange(tag + 1000 * s, tag + 1000 * s + k, dtype=np.int32) for s, k in enumerate(sizes)]
            tag += 7
            a.insert_parallel(batches)
            o.insert_parallel(batches)
        else:
            cur = np.asarray(o.size)
            new = (cur * rng.random(S)).astype(np.int64)
            a.shrink(new)
            o.shrink(new)
        assert a._parity_state() == {k: v for k, v in o._parity_state().items() if k != "alloc_calls"}
        assert a.flatten().tobytes() == o.flatten().tobytes()
    ms = a.memory_stats()
    assert ms["capacity_bytes"] == int(o.capacity.sum()) * 4


def test_flatten_device_and_views(gg):
    import torch
    a = gg.GrowableArray.from_flat(np.arange(5000, dtype=np.float32), shards=3, first_bucket_size=2)
    f = a.flatten_device()
    assert f.is_cuda and f.dtype == torch.float32
    assert torch.equal(f.cpu(), torch.arange(5000, dtype=torch.float32))
    # for_each_shard hands out writable device views
    a.for_each_shard(lambda v: v.add_(1))
    assert np.array_equal(a.flatten(), np.arange(5000, dtype=np.float32) + 1)
    segs = list(a.shards[1].iter_segments(11, start=3))
    assert torch.equal(torch.cat(segs).cpu(), torch.arange(1667 + 3, 1667 + 11, dtype=torch.float32) + 1)


def test_scan_reserver_rendezvous_on_device_counter(gg):
    # reference test_bucket_vector.py:228-239: 6 lanes, groups of 4 -> 2 counter ops
    import threading
    sv = gg.ShardVector(first_bucket_size=4, dtype=np.int64)
    reserver = gg.ScanReserver(6, group_size=4)
    batches = [10_000 * t + np.arange(50 * (t % 3)) for t in range(6)]
    ops0 = sv.size_counter.op_count
    ths = [threading.Thread(target=sv.push_back_batch, args=(b, reserver)) for b in batches]
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    assert sv.size_counter.op_count - ops0 == 2
    assert np.array_equal(np.sort(sv.to_numpy()), np.sort(np.concatenate(batches)))


def test_memory_footprint_config1(gg):
    a = gg.GrowableArray(512, 32, dtype=np.int32)
    a.insert_parallel(gg.split_batches(np.arange(1 << 20, dtype=np.int32), 512))
    ms = a.memory_stats()
    assert ms["capacity_bytes"] == 2_080_768 * 4                 # SURVEY 8c golden
    assert ms["bucket_bytes"] == ms["capacity_bytes"]          # no 16 B padding in the slots
    assert ms["capacity_bytes"] == gg.ggarray_capacity_for(1 << 20, 512, 32, 4)


def test_phased_insert_shrink_vs_oracle_model(gg):
    """Config 4 at reduced size: uniform(0,2) total-size factors, even split,
    insert or shrink; state and contents vs the oracle's (unpinned) shrink model."""
    rng = np.random.default_rng(0)
    S, fb = 64, 32
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    o = O.OracleGGArray(S, fb, dtype=np.int32)
    n = 1 << 14
    vals = np.arange(1 << 17, dtype=np.int32)
    off = np.minimum(np.arange(S + 1) * (-(-n // S)), n)
    a.insert_parallel([vals[off[s]:off[s + 1]] for s in range(S)])
    o.insert_parallel([vals[off[s]:off[s + 1]] for s in range(S)])
    for _ in range(30):
        target = int(min(1 << 16, round(rng.uniform(0, 2) * (1 << 14))))
        q, r = divmod(target, S)
        new = np.full(S, q, np.int64)
        new[:r] += 1
        cur = np.asarray(o.size)
        if target >= n:
            d = new - cur
            offs = np.concatenate([[0], np.cumsum(d)])
            batches = [vals[offs[s]:offs[s + 1]] for s in range(S)]
            a.insert_parallel(batches)
            o.insert_parallel(batches)
        else:
            a.shrink(new)
            o.shrink(new)
        n = target
        st = a._parity_state()
        assert st["sizes"] == [int(x) for x in o.size] and st["caps"] == [int(x) for x in o.capacity]
        ms = a.memory_stats()
        assert ms["capacity_bytes"] <= 2 * ms["needed_bytes"] + S * fb * 4
    assert a.flatten().tobytes() == o.flatten().tobytes()


def test_reference_quickstart_verbatim(gg):
    """pkg/README.md's library quickstart with only the import swapped: numpy
    ufunc ops in for_each_shard run on the device views."""
    from paper_2209_00103_b200 import GrowableArray, split_batches

    arr = GrowableArray(shards=32, first_bucket_size=32, dtype=np.int32)
    arr.insert_parallel(split_batches(np.arange(10_000, dtype=np.int32), 32))

    assert arr.get_global(1234) == 1234
    arr.for_each_shard(lambda view: np.add(view, 1, out=view), workers=4)

    flat = arr.flatten()
    again = GrowableArray.from_flat(flat, shards=32)
    assert np.array_equal(flat, np.arange(10_000, dtype=np.int32) + 1)
    assert again.flatten().tobytes() == flat.tobytes()


@pytest.mark.parametrize("dtype", ["int8", "int32", "float16", "float64"])
def test_for_each_shard_numpy_ops_match_oracle(gg, dtype):
    rng = np.random.default_rng(3)
    S, fb = 9, 4
    batches = [(rng.integers(0, 100, int(k))).astype(dtype) for k in rng.integers(0, 300, S)]
    a = gg.GrowableArray(S, fb, dtype=dtype)
    o = O.OracleGGArray(S, fb, dtype=dtype)
    a.insert_parallel(batches); o.insert_parallel(batches)
    c = np.asarray(3).astype(dtype)
    a.for_each_shard(lambda v: np.add(v, c, out=v, casting="unsafe"))
    a.for_each_shard(lambda v: np.multiply(v, 2, out=v, casting="unsafe"))
    a.for_each_shard(lambda v: v.sub_(1))                 # torch methods still work
    want = ((o.flatten() + c).astype(dtype) * np.asarray(2, dtype)).astype(dtype) - np.asarray(1, dtype)
    assert a.flatten().tobytes() == want.astype(dtype).tobytes()
