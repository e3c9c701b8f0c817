"""Property-based parity on the B200: hypothesis-drawn op scripts through the
drop-in and the oracle (itself pinned to the reference), identical recorded
states (sizes, capacities, flags, prefix, counter ops, allocator calls,
flattened bytes, get_global samples, exceptions) after every op."""
import os

import pytest
from hypothesis import HealthCheck, given, settings
from hypothesis import strategies as st

from hyp_scripts import op_scripts, run
from oracle import ggoracle as O

pytestmark = pytest.mark.gpu
_SCALE = int(os.environ.get("GG_HYP_SCALE", "1"))     # stress runs: more examples


@settings(max_examples=40 * _SCALE, deadline=None, suppress_health_check=[HealthCheck.too_slow],
          database=None)
@given(ops=op_scripts())
def test_gpu_equals_oracle_on_random_scripts(ops):
    import paper_2209_00103_b200 as gg
    assert run(gg, ops) == run(O, ops)


@settings(max_examples=25 * _SCALE, deadline=None, suppress_health_check=[HealthCheck.too_slow], database=None)
@given(S=st.sampled_from([1, 3, 8, 33]), fb=st.sampled_from([1, 2, 4, 32]), n=st.integers(1, 20000),
       grid=st.integers(1, 300), dens=st.floats(0.0, 1.0), mode=st.sampled_from(["warp", "block"]),
       seed=st.integers(0, 2**16))
def test_device_push_back_random(S, fb, n, grid, dens, mode, seed):
    """Device push_back (warp_push_back_n / block_push_back through push_if) on
    random shapes: per-shard multiset, sizes and minimal capacities."""
    import numpy as np
    import paper_2209_00103_b200 as gg
    rng = np.random.default_rng(seed)
    vals = rng.integers(-2**31, 2**31 - 1, n, dtype=np.int64).astype(np.int32)
    pred = rng.random(n) < dens
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    pre = [np.arange(int(k), dtype=np.int32) for k in rng.integers(0, 3 * fb + 5, S)]
    a.insert_parallel(pre)
    grid = max(grid, S)
    a.push_if(vals, pred, mode=mode, grid=grid)
    blk = (np.arange(n) // 1024) % grid           # slice = 1024 candidates (kPushSlice)
    st_ = a._parity_state()
    for s in range(S):
        got = a.shards[s].to_numpy()
        want = vals[(blk % S == s) & pred]
        assert np.array_equal(got[:len(pre[s])], pre[s])
        assert np.array_equal(np.sort(got[len(pre[s]):]), np.sort(want))
        k = O.min_buckets_for(len(got), fb)
        assert st_["sizes"][s] == len(got) and st_["caps"][s] == O.capacity_of(k, fb)
