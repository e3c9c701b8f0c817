"""bench.py's N > 1 path (torchrun, weak scaling, max-over-ranks timing, the
fused gather into rank 0) run with two ranks on the test box's one GPU
(GG_BENCH_SAME_GPU=1: gloo control plane, both ranks on cuda:0)."""
import json
import os
import socket
import subprocess
import sys

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(env):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(_port()), "bench.py", "--gpus", "2",
           "--steps", "1", "--warmup", "3", "--quick"]
    r = subprocess.run(cmd, cwd=ROOT, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-3000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    return json.loads(lines[0])


def test_bench_two_ranks_json_line():
    d = _run(dict(os.environ, GG_BENCH_SAME_GPU="1"))
    assert d["n_gpus"] == 2 and d["scaling"] == "weak" and d["value"] > 0
    g = d["gather_flatten"]
    assert g.get("root_slice_ok") is True and g["bytes_total"] == 2 * 4 * (1 << 30)
    assert g["peer_topology"] == "ok" and g["bytes_over_nvlink_per_rank"] == [0, 4 << 30]


def test_bench_two_ranks_without_peer_access():
    """The fallback branch: peer stores refused (GG_PEER=0 stands in for
    cudaDeviceCanAccessPeer = 0), the gather runs the NCCL-style path and the
    line says why."""
    d = _run(dict(os.environ, GG_BENCH_SAME_GPU="1", GG_PEER="0"))
    g = d["gather_flatten"]
    assert g.get("root_slice_ok") is True, g
    assert g["peer_topology"] == "unavailable" and g["fallback_reason"] == "GG_PEER=0"
    assert g["bytes_over_nvlink_per_rank"] == [0, 4 << 30]
