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


def install_reference(force: bool = False) -> str | None:
    """pip-install the UNMODIFIED reference (/root/reference/pkg, pure Python,
    numpy only) into baseline/_ref for bench.py --impl reference, from a /tmp
    copy (the reference tree is read-only) with --no-deps (numpy is in the
    image, the wheelhouse has no numpy wheel).  No-op when already installed
    or when /root/reference is absent (GPU box)."""
    import shutil
    import tempfile
    ref_src = "/root/reference/pkg"
    target = os.path.join(ROOT, "baseline", "_ref")
    if os.path.isfile(os.path.join(target, "growarray", "__init__.py")) and not force:
        return target
    if not os.path.isdir(ref_src):
        return None
    with tempfile.TemporaryDirectory() as tmp:
        copy = os.path.join(tmp, "pkg")
        shutil.copytree(ref_src, copy, ignore=shutil.ignore_patterns(".hypothesis", "__pycache__"))
        shutil.rmtree(target, ignore_errors=True)
        res = subprocess.run([sys.executable, "-m", "pip", "install", "--no-index", "--no-build-isolation",
                              "--no-deps", "--find-links", "/opt/wheelhouse", "--target", target, copy],
                             capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout[-2000:] + res.stderr[-2000:])
        return None
    return target


if __name__ == "__main__":
    print(build(verbose="-v" in sys.argv))
