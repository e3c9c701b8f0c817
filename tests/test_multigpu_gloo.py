"""World-size-2 gloo tests of the multi-GPU host logic on CPU: every
rank owns a contiguous LFVector range (the oracle array stands in for the
device array); the all-gather directory and the gather-to-root flatten must
reproduce the single-array flatten of the concatenated shards."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch.distributed as dist
    import sys
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import ggoracle as O
    from paper_2209_00103_b200.multigpu import DistributedGrowableArray
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        S_total, per_rank = 8, 4
        rng = np.random.default_rng(0)
        sizes = rng.integers(0, 50, S_total)
        vals = np.arange(int(sizes.sum()), dtype=np.int32)
        off = np.concatenate([[0], np.cumsum(sizes)])
        lo, hi = rank * per_rank, (rank + 1) * per_rank
        local = O.OracleGGArray(per_rank, 4, dtype=np.int32)
        local.insert_parallel([vals[off[s]:off[s + 1]] for s in range(lo, hi)])
        for _ in range(2):                               # local growth, no communication
            local.grow(2 * local.committed_size)
            local.insert_duplicate()
            local.rw_add(1)
        d = DistributedGrowableArray(local)
        pre = d.global_prefix()
        flat = d.flatten_global(root=0)
        allg = d.allgather_flat().numpy()
        loc = d.locate_global(pre[-1] - 1, pre)
        probes = [0, pre[1], pre[-1] - 1] if pre[-1] else []
        got = [int(d.get_global(g, pre)) for g in probes]
        if probes:
            d.set_global(probes[-1], -7, pre)
            got.append(int(d.get_global(probes[-1], pre)))
        # a device-capable local whose peer stores are unavailable: the "peer"
        # request must fall back to NCCL-style point-to-point with the reason
        os.environ["GG_PEER"] = "0"
        fake = _PeerlessLocal(local)
        d2 = DistributedGrowableArray(fake)
        flat2 = d2.flatten_global(root=0, method="peer")
        reb, (rlo, rhi) = d2.rebalance_flat_peer()
        fb = (d2.last_method, d2.fallback_reason, d2.peer_topology(),
              None if flat2 is None else flat2.numpy(), reb.numpy(), rlo, rhi)
        q.put((rank, pre, None if flat is None else flat.numpy(), allg, loc, got, fb))
    finally:
        dist.destroy_process_group()


class _PeerlessLocal:
    """An array that offers device flatten_to (so "auto" would pick peer
    stores) on a group whose topology says no: flatten_to must never run."""

    def __init__(self, inner):
        self.inner = inner
        self.dtype = inner.dtype

    @property
    def committed_size(self):
        return self.inner.committed_size

    def flatten(self):
        return self.inner.flatten()

    def flatten_to(self, ptr):
        raise AssertionError("peer store attempted without peer access")

    flatten_range_to = flatten_to


def _single_array_reference():
    from oracle import ggoracle as O
    S_total = 8
    rng = np.random.default_rng(0)
    sizes = rng.integers(0, 50, S_total)
    vals = np.arange(int(sizes.sum()), dtype=np.int32)
    off = np.concatenate([[0], np.cumsum(sizes)])
    # the two ranks grow independently: reproduce per rank, then concatenate
    parts = []
    for r in range(2):
        a = O.OracleGGArray(4, 4, dtype=np.int32)
        a.insert_parallel([vals[off[s]:off[s + 1]] for s in range(4 * r, 4 * r + 4)])
        for _ in range(2):
            a.grow(2 * a.committed_size)
            a.insert_duplicate()
            a.rw_add(1)
        parts.append(a.flatten())
    return np.concatenate(parts), [0, len(parts[0]), len(parts[0]) + len(parts[1])]


def test_two_rank_directory_and_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = {}
    for _ in range(2):
        rank, pre, flat, allg, loc, got, fb = q.get(timeout=120)
        res[rank] = (pre, flat, allg, loc, got, fb)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    want, want_pre = _single_array_reference()
    assert res[0][0] == res[1][0] == want_pre
    assert np.array_equal(res[0][1], want)
    assert res[1][1] is None
    assert np.array_equal(res[0][2], want) and np.array_equal(res[1][2], want)
    assert res[0][3] == (1, want_pre[2] - want_pre[1] - 1)
    probes = [int(want[0]), int(want[want_pre[1]]), int(want[-1]), -7]      # distributed get/set_global
    assert res[0][4] == res[1][4] == probes
    want2 = want.copy()
    want2[-1] = -7                                     # the set_global above
    for r in (0, 1):                                   # peer request fell back, with the reason
        method, why, topo, flat2, reb, lo, hi = res[r][5]
        assert method == "nccl" and why == "GG_PEER=0" and topo == (False, "GG_PEER=0")
        assert reb.tobytes() == want2[lo:hi].tobytes()
    assert np.array_equal(res[0][5][3], want2) and res[1][5][3] is None
