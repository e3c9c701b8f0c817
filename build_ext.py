"""Build the in-tree CUDA library paper_2209_00103_b200/_ggarray.so for sm_100a.

Used by __graft_entry__.build(); runnable directly: python build_ext.py
"""
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.abspath(__file__))
PKG = os.path.join(ROOT, "paper_2209_00103_b200")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

FLAGS = ["-std=c++17", "-O3", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
         "-Xcompiler", "-fPIC", "-Xcompiler", "-O3", "-shared", "-cudart", "static",
         "-I", os.path.join(ROOT, "include")]


def build(verbose: bool = False) -> str:
    src = os.path.join(PKG, "csrc", "ggarray.cu")
    out = os.path.join(PKG, "_ggarray.so")
    import glob
    deps = [src, __file__] + glob.glob(os.path.join(ROOT, "include", "*")) + \
        glob.glob(os.path.join(PKG, "csrc", "*"))
    if os.path.exists(out) and all(os.path.getmtime(out) >= os.path.getmtime(d) for d in deps):
        return out
    cmd = [NVCC, *FLAGS, "-o", out + ".tmp", src]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building _ggarray.so")
    os.replace(out + ".tmp", out)
    return out


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
