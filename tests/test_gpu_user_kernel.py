"""The device-side push_back API from a separately compiled user kernel
(tests/c/user_kernel.cu, nvcc against include/ggarray_device.cuh only):
get a view (backs each shard's worst-case buckets), launch, sync; the
appended multiset per shard, sizes and capacities must match."""
import ctypes as C
import os
import subprocess

import numpy as np
import pytest

from oracle import ggoracle as O

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")


@pytest.fixture(scope="module")
def user_lib(tmp_path_factory):
    so = str(tmp_path_factory.mktemp("uk") / "user_kernel.so")
    subprocess.run([NVCC, "-std=c++17", "-O2", "-gencode", "arch=compute_100a,code=sm_100a",
                    "-Xcompiler", "-fPIC", "-shared", "-I", os.path.join(ROOT, "include"),
                    os.path.join(ROOT, "tests", "c", "user_kernel.cu"), "-o", so],
                   check=True, capture_output=True, text=True)
    lib = C.CDLL(so)
    lib.user_emit_launch.argtypes = [C.c_void_p, C.c_uint64, C.c_void_p, C.c_uint64, C.c_uint32,
                                     C.c_int, C.c_void_p]
    lib.user_emit_launch.restype = C.c_int
    return lib


@pytest.mark.parametrize("block_mode", [0, 1, 2, 3, 4, 5])   # warp, block, warp_mask, block_mask, block_staged, warp_staged
def test_user_kernel_appends(user_lib, block_mode):
    import torch
    import paper_2209_00103_b200 as gg
    S, fb, grid, n = 12, 8, 96, 300_000
    rng = np.random.default_rng(block_mode % 2)
    x = rng.integers(0, 1 << 30, n).astype(np.int32)
    d = torch.from_numpy(x).cuda()
    a = gg.GrowableArray(S, fb, dtype=np.int32)
    pre = [np.full(int(k), -1, np.int32) for k in rng.integers(0, 50, S)]
    a.insert_parallel(pre)
    # worst case per shard: every element of its blocks' slices is odd
    blk = (np.arange(n) // 256) % grid
    cand = np.bincount(blk % S, minlength=S)
    view = a.device_view(max_sizes=a._host()["sizes"].astype(np.int64) + cand)
    rc = user_lib.user_emit_launch(view, len(view), C.c_void_p(d.data_ptr()), n, grid, block_mode,
                                   C.c_void_p(torch.cuda.current_stream().cuda_stream))
    assert rc == 0
    a.device_sync()
    a.commit()
    shard = blk % S
    for s in range(S):
        got = a.shards[s].to_numpy()
        want = x[(shard == s) & (x % 2 == 1)]
        assert np.array_equal(got[:len(pre[s])], pre[s])
        assert np.array_equal(np.sort(got[len(pre[s]):]), np.sort(want))
        k = O.min_buckets_for(len(got), fb)
        st = a._parity_state()
        assert st["caps"][s] == O.capacity_of(k, fb) and st["sizes"][s] == len(got)
    ms = a.memory_stats()
    assert ms["bucket_bytes"] == ms["capacity_bytes"]        # unused headroom given back
