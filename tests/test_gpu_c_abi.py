"""The C ABI driven from plain C (tests/c/abi_smoke.c), compiled with gcc
against include/ggarray.h and the in-tree _ggarray.so -- the binding a caller
in another language would write."""
import os
import subprocess

import pytest

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def test_c_program_end_to_end(tmp_path):
    exe = str(tmp_path / "abi_smoke")
    pkg = os.path.join(ROOT, "paper_2209_00103_b200")
    cmd = ["gcc", "-std=c11", "-O1", os.path.join(ROOT, "tests", "c", "abi_smoke.c"), "-o", exe,
           "-I", os.path.join(ROOT, "include"), "-I", os.path.join(CUDA, "include"),
           os.path.join(pkg, "_ggarray.so"), "-L", os.path.join(CUDA, "lib64"), "-lcudart",
           "-Wl,-rpath," + pkg + ":" + os.path.join(CUDA, "lib64")]
    subprocess.run(cmd, check=True, capture_output=True, text=True)
    r = subprocess.run([exe], capture_output=True, text=True, timeout=300)
    assert r.returncode == 0 and r.stdout.strip() == "OK", r.stderr
