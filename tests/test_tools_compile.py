"""The measurement scripts in tools/ and bench.py at least compile (they only
run on a GPU box)."""
import glob
import os
import py_compile

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
SCRIPTS = sorted(glob.glob(os.path.join(ROOT, "tools", "*.py")) + glob.glob(os.path.join(ROOT, "tools", "probe", "*.py"))
                 + [os.path.join(ROOT, "bench.py"), os.path.join(ROOT, "build_ext.py"),
                    os.path.join(ROOT, "__graft_entry__.py")])


@pytest.mark.parametrize("path", SCRIPTS, ids=lambda p: os.path.relpath(p, ROOT))
def test_compiles(path, tmp_path):
    py_compile.compile(path, cfile=str(tmp_path / "x.pyc"), doraise=True)
