"""Drop-in check: every public name of the reference package exists in ours,
classes expose the reference's public members, and functions / methods take
the reference's parameters in the same order (ours may add trailing
extension parameters).  Only where the reference is mounted (build
container); CPU-only (introspection, no GPU calls)."""
import inspect
import os
import sys

import pytest

REF = "/root/reference/pkg/src"
pytestmark = pytest.mark.skipif(not os.path.isdir(REF), reason="reference not mounted")

CLASSES = ("GrowableArray", "ShardVector", "BucketTable", "StaticArray", "DoublingArray",
           "ChunkTableArray", "AtomicCounter", "AtomicReserver", "ScanReserver", "LanePlan",
           "ReservedRange", "MemoryModelParams", "MemoryReport")


@pytest.fixture(scope="module")
def mods():
    sys.path.insert(0, REF)
    import growarray as R
    import paper_2209_00103_b200 as G
    return R, G


def _params(f):
    try:
        return list(inspect.signature(f).parameters)
    except (TypeError, ValueError):
        return None


def test_public_names(mods):
    R, G = mods
    assert [n for n in R.__all__ if not hasattr(G, n)] == []


@pytest.mark.parametrize("cls", CLASSES)
def test_class_members_and_signatures(mods, cls):
    R, G = mods
    r, g = getattr(R, cls), getattr(G, cls)
    instance_attrs = {"size_counter"}          # set per instance in both packages
    missing = sorted(a for a in dir(r) if not a.startswith("_") and not hasattr(g, a)
                     and a not in instance_attrs)
    assert missing == []
    for a in ["__init__"] + [a for a in dir(r) if not a.startswith("_")]:
        ra, ga = getattr(r, a, None), getattr(g, a, None)
        if callable(ra) and callable(ga):
            rp, gp = _params(ra), _params(ga)
            if rp is not None and gp is not None:
                assert gp[:len(rp)] == rp, (cls, a, rp, gp)


def test_function_signatures(mods):
    R, G = mods
    for n in R.__all__:
        r = getattr(R, n)
        if inspect.isfunction(r):
            rp, gp = _params(r), _params(getattr(G, n))
            assert gp[:len(rp)] == rp, (n, rp, gp)
