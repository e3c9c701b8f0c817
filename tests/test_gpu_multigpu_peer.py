"""The fused gather-flatten over peer memory (multigpu.py) with two
processes.  The GPU boxes of this run have one GPU, so both ranks share
cuda:0: the root's buffer is still mapped into the other process with CUDA
IPC and written by that process's flatten kernel, exactly the code path that
crosses NVLink when the ranks sit on different GPUs.  Control plane: gloo."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_batches(rank, per_rank, sizes, vals, off):
    lo = rank * per_rank
    return [vals[off[s]:off[s + 1]] for s in range(lo, lo + per_rank)]


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch
    import torch.distributed as dist
    import paper_2209_00103_b200 as gg
    from paper_2209_00103_b200.multigpu import DistributedGrowableArray
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        per_rank = 16
        rng = np.random.default_rng(5)
        sizes = rng.integers(0, 3000, per_rank * world)
        sizes[3] = 0
        vals = rng.integers(-2**31, 2**31 - 1, int(sizes.sum()), dtype=np.int64).astype(np.int32)
        off = np.concatenate([[0], np.cumsum(sizes)])
        a = gg.GrowableArray(per_rank, 8, dtype=np.int32)
        a.insert_parallel(_rank_batches(rank, per_rank, sizes, vals, off))
        for _ in range(2 + rank):                      # ranks grow independently
            a.grow(2 * a.committed_size)
            a.insert_duplicate()
        a.rw_add(rank + 1)
        d = DistributedGrowableArray(a, device=torch.device("cuda", 0))
        flat = d.flatten_global(root=0, method="peer")
        assert d.peer_topology() == (True, None) and d.last_method == "peer"   # same GPU: reachable
        allg = d.all_gather_flat_peer()
        reb, rng_ = d.rebalance_flat_peer()
        part = a.flatten_range(3, max(3, a.committed_size - 5)).cpu().numpy()
        q.put((rank, None if flat is None else flat.cpu().numpy(), allg.cpu().numpy(), a.flatten(),
               reb.cpu().numpy(), rng_, part))
        dist.barrier()
    finally:
        dist.destroy_process_group()


def test_peer_gather_flatten_two_processes():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    res = {}
    for _ in range(world):
        r, flat, allg, local, reb, rng_, part = q.get(timeout=300)
        res[r] = (flat, allg, local, reb, rng_, part)
    for p in ps:
        p.join(timeout=60)
        assert p.exitcode == 0
    want = np.concatenate([res[r][2] for r in range(world)])   # GPU-major, then shard-major
    assert res[0][0] is not None and res[0][0].tobytes() == want.tobytes()
    assert res[1][0] is None
    for r in range(world):
        assert res[r][1].tobytes() == want.tobytes()
        lo, hi = res[r][4]
        assert res[r][3].tobytes() == want[lo:hi].tobytes()          # even rebalance slice
        local = res[r][2]
        assert res[r][5].tobytes() == local[3:max(3, len(local) - 5)].tobytes()   # flatten_range
    assert sum(res[r][4][1] - res[r][4][0] for r in range(world)) == len(want)
