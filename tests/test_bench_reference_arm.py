"""bench.py's reference arm (the unmodified growarray from baseline/_ref on
the host cores; the oracle port when baseline/_ref is absent) keeps the
driver's JSON contract, on one process and under torchrun with two ranks
(rank 0 alone prints).  CPU only; the schedule is shortened (--ref-rounds)."""
import json
import os
import socket
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
ARGS = ["bench.py", "--impl", "reference", "--steps", "1", "--warmup", "3", "--cpu-rounds", "2",
        "--ref-rounds", "3"]
HAVE_REF = os.path.isfile(os.path.join(ROOT, "baseline", "_ref", "growarray", "__init__.py"))


def _check(line):
    d = json.loads(line)
    assert d["impl"] == "reference" and d["metric"] == "GGArray insert Gelem/s" and d["unit"] == "Gelem/s"
    assert d["value"] > 0 and d["higher_is_better"] is True and d["warmup"] >= 3 and d["steps"] == 1
    assert d["cpu_baseline"]["kind"] == ("reference" if HAVE_REF else "port") and d["cpu_baseline"]["cores"] >= 1
    assert d["cpu_baseline"]["value"] == d["value"]
    assert d["e2e"] == {"value": d["value"], "unit": "Gelem/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}
    assert "workload" in d["config"]
    return d


def test_reference_arm_single_process():
    r = subprocess.run([sys.executable] + ARGS, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert _check(lines[0])["n_gpus"] == 1


def test_reference_arm_torchrun_two_ranks():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "2",
           "--master-addr", "127.0.0.1", "--master-port", str(port)] + ARGS + ["--gpus", "2"]
    r = subprocess.run(cmd, cwd=ROOT, capture_output=True, text=True, timeout=300)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    assert _check(lines[0])["n_gpus"] == 2


def test_reference_install_is_unmodified():
    """baseline/_ref holds the reference package byte for byte (when both trees
    are present, i.e. in the build container)."""
    import filecmp
    import pytest
    src = "/root/reference/pkg/src/growarray"
    dst = os.path.join(ROOT, "baseline", "_ref", "growarray")
    if not (HAVE_REF and os.path.isdir(src)):
        pytest.skip("baseline/_ref or /root/reference absent")
    names = sorted(f for f in os.listdir(src) if f.endswith(".py"))
    assert names and names == sorted(f for f in os.listdir(dst) if f.endswith(".py"))
    match, mismatch, errors = filecmp.cmpfiles(src, dst, names, shallow=False)
    assert not mismatch and not errors, (mismatch, errors)
