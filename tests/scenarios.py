"""Operation scripts replayed through three implementations of the GGArray API:

* the unmodified reference ``growarray`` (to generate ``tests/golden/golden.json``),
* the CPU oracle ``oracle.ggoracle`` (pinned against those goldens),
* the B200 drop-in ``paper_2209_00103_b200`` (the parity tests proper).

A scenario is a list of JSON ops; after every op the runner records the
observable state (per-shard sizes, capacities, allocated-bucket flags, the
committed prefix, counter ops, allocator calls, the flattened bytes and a
few ``get_global`` samples) plus the exception raised, if any.  The ops and
their semantics follow the reference tests they are drawn from
(``pkg/tests/test_sharded_array.py``, ``test_bucket_vector.py``,
``test_baselines.py``) and the bench workloads (``bench_cli.py:298-376``).
"""

from __future__ import annotations

import hashlib

import numpy as np

RANDOM_DTYPES = ["int32", "int64", "float32", "float64", "int8", "int16", "uint8",
                 "uint16", "uint32", "uint64", "float16"]


# ------------------------------------------------------------------ scenario set

def _random_scenario(seed: int) -> list[dict]:
    rng = np.random.default_rng(1000 + seed)
    S = int(rng.choice([1, 2, 3, 5, 8, 17, 32, 40]))
    fb = int(rng.choice([1, 2, 4, 8, 32, 1024]))
    dtype = str(rng.choice(RANDOM_DTYPES))
    ops: list[dict] = [{"op": "new", "shards": S, "fb": fb, "dtype": dtype, "max_buckets": 58}]
    tag = 0
    for _ in range(int(rng.integers(4, 10))):
        kind = rng.choice(["insert", "insert", "insert", "dup", "grow", "add", "set",
                           "push", "commit", "reserve"])
        if kind == "insert":
            sizes = rng.integers(0, 3 * fb + 70, size=S)
            sizes[rng.random(S) < 0.3] = 0
            ops.append({"op": "insert", "sizes": [int(x) for x in sizes], "base": tag})
            tag += int(sizes.sum())
        elif kind == "dup":
            ops.append({"op": "dup"})
        elif kind == "grow":
            if rng.random() < 0.5:
                ops.append({"op": "grow", "target": int(rng.integers(0, 4000)), "dist": None})
            else:
                ops.append({"op": "grow", "target": 0,
                            "dist": [int(x) for x in rng.integers(0, 500, size=S)]})
        elif kind == "add":
            ops.append({"op": "add", "c": int(rng.integers(1, 4)), "passes": int(rng.integers(1, 4))})
        elif kind == "set":
            ops.append({"op": "set_frac", "f": float(rng.random()), "v": int(rng.integers(0, 100))})
        elif kind == "push":
            ops.append({"op": "push", "s": int(rng.integers(0, S)),
                        "n": int(rng.integers(0, 2 * fb + 9)), "base": tag})
            tag += 1000
        elif kind == "reserve":
            ops.append({"op": "reserve", "s": int(rng.integers(0, S)), "cap": int(rng.integers(0, 900))})
        else:
            ops.append({"op": "commit"})
    ops.append({"op": "commit"})
    ops.append({"op": "add", "c": 1, "passes": 1})
    return ops


def scenarios() -> dict[str, list[dict]]:
    sc: dict[str, list[dict]] = {}
    sc["kat_prefix"] = [
        {"op": "new", "shards": 3, "fb": 2, "dtype": "int64"},
        {"op": "push", "s": 0, "n": 4, "base": 0},
        {"op": "push", "s": 2, "n": 5, "base": 4},
        {"op": "commit"},
        {"op": "get", "g": 4},
        {"op": "get", "g": 9},
        {"op": "get", "g": -1},
    ]
    sc["kat_insert_sizes"] = [
        {"op": "new", "shards": 4, "fb": 2, "dtype": "int64"},
        {"op": "insert", "sizes": [2, 0, 3, 1], "base": 1},
        {"op": "insert_wrong_count"},
    ]
    sc["kat_fb1_boundary"] = [
        {"op": "new", "shards": 1, "fb": 1, "dtype": "int64"},
        {"op": "push", "s": 0, "n": 1, "base": 0},
        {"op": "push", "s": 0, "n": 4, "base": 1},
        {"op": "push", "s": 0, "n": 0, "base": 0},
        {"op": "commit"},
    ]
    sc["kat_fb2_boundary"] = [
        {"op": "new", "shards": 1, "fb": 2, "dtype": "int64"},
        {"op": "push", "s": 0, "n": 1, "base": 0},
        {"op": "push", "s": 0, "n": 4, "base": 1},
        {"op": "commit"},
    ]
    sc["capacity_exhausted"] = [
        {"op": "new", "shards": 1, "fb": 1, "dtype": "int64", "max_buckets": 3},
        {"op": "push", "s": 0, "n": 7, "base": 0},
        {"op": "push", "s": 0, "n": 1, "base": 7},
        {"op": "reserve", "s": 0, "cap": 8},
    ]
    sc["partial_failure"] = [
        {"op": "new", "shards": 3, "fb": 1, "dtype": "int64", "max_buckets": 3},
        {"op": "insert", "sizes": [1, 1, 1], "base": 1},
        {"op": "insert", "sizes": [1, 20, 1], "base": 10},
        {"op": "insert", "sizes": [1, 0, 1], "base": 50},
    ]
    sc["alloc_fail_hole"] = [
        {"op": "new", "shards": 2, "fb": 4, "dtype": "int32", "fail_calls": [3]},
        {"op": "insert", "sizes": [10, 10], "base": 100},
        {"op": "insert", "sizes": [1, 1], "base": 500},
        {"op": "new_bucket", "s": 1, "b": 0},
        {"op": "add", "c": 2, "passes": 1},
    ]
    sc["alloc_fail_midrange"] = [
        {"op": "new", "shards": 3, "fb": 2, "dtype": "int64", "fail_calls": [4, 9]},
        {"op": "insert", "sizes": [5, 13, 3], "base": 0},
        {"op": "insert", "sizes": [30, 2, 7], "base": 100},
        {"op": "grow", "target": 300, "dist": None},
        {"op": "grow", "target": 300, "dist": None},
    ]
    sc["grow_cases"] = [
        {"op": "new", "shards": 2, "fb": 4, "dtype": "int64", "count_alloc": True},
        {"op": "grow", "target": 100, "dist": None},
        {"op": "grow", "target": 100, "dist": None},
        {"op": "grow", "target": 0, "dist": [10, 0]},
        {"op": "grow", "target": 10, "dist": [5]},
        {"op": "new", "shards": 1, "fb": 32, "dtype": "int64", "count_alloc": True},
        {"op": "grow", "target": 33, "dist": None},
        {"op": "grow", "target": 66, "dist": None},
        {"op": "new", "shards": 3, "fb": 2, "dtype": "int64"},
        {"op": "grow", "target": 0, "dist": [10, 0, 3]},
        {"op": "new", "shards": 32, "fb": 32, "dtype": "int64"},
        {"op": "grow", "target": 1000000, "dist": None},
    ]
    sc["grow_capacity_error"] = [
        {"op": "new", "shards": 3, "fb": 1, "dtype": "int64", "max_buckets": 3},
        {"op": "grow", "target": 0, "dist": [7, 8, 3]},
        {"op": "grow", "target": 0, "dist": [0, 7, 3]},
    ]
    sc["new_bucket"] = [
        {"op": "new", "shards": 2, "fb": 32, "dtype": "int64", "fail_calls": [2]},
        {"op": "new_bucket", "s": 0, "b": 0},
        {"op": "new_bucket", "s": 0, "b": 0},
        {"op": "new_bucket", "s": 1, "b": 3},
        {"op": "new_bucket", "s": 1, "b": 3},
        {"op": "new_bucket", "s": 1, "b": 58},
        {"op": "push", "s": 1, "n": 40, "base": 0},
    ]
    sc["set_get"] = [
        {"op": "new", "shards": 4, "fb": 2, "dtype": "int64"},
        {"op": "insert", "sizes": [6, 0, 2, 9], "base": 0},
    ] + [{"op": "set", "g": int(g), "v": int(v)} for g, v in
         zip(np.random.default_rng(17).integers(0, 17, 60),
             np.random.default_rng(18).integers(-1000, 1000, 60))] + [
        {"op": "set", "g": 17, "v": 0},
        {"op": "get", "g": 17},
        {"op": "get", "g": 16},
    ]
    sc["add30"] = [
        {"op": "new", "shards": 3, "fb": 2, "dtype": "int64"},
        {"op": "insert", "sizes": [5, 0, 11], "base": 0},
        {"op": "add", "c": 1, "passes": 30},
    ]
    sc["uncommitted_tail"] = [
        {"op": "new", "shards": 1, "fb": 2, "dtype": "int64"},
        {"op": "insert", "sizes": [4], "base": 0},
        {"op": "push", "s": 0, "n": 2, "base": 99},
        {"op": "add", "c": 5, "passes": 1},
        {"op": "commit"},
    ]
    sc["locate_shard"] = [
        {"op": "new", "shards": 7, "fb": 2, "dtype": "int64"},
        {"op": "insert", "sizes": [3, 0, 0, 17, 1, 0, 9], "base": 0},
    ] + [{"op": "get", "g": g} for g in range(30)]
    sc["dup_rounds"] = [{"op": "from_flat", "n": 32, "shards": 8, "fb": 4, "dtype": "int64"}] + \
        [{"op": "dup"} for _ in range(6)]
    sc["from_flat_cases"] = [
        {"op": "from_flat", "n": 5, "shards": 3, "fb": 2, "dtype": "int64"},
        {"op": "from_flat", "n": 0, "shards": 4, "fb": 32, "dtype": "int64"},
        {"op": "from_flat", "n": 9, "shards": 2, "fb": 32, "dtype": "int32"},
        {"op": "from_flat", "n": 1000, "shards": 7, "fb": 8, "dtype": "float32"},
        {"op": "from_flat", "n": 300, "shards": 9, "fb": 1, "dtype": "int8"},
        {"op": "from_flat", "n": 777, "shards": 16, "fb": 4, "dtype": "float64"},
        {"op": "from_flat", "n": 2, "shards": 4, "fb": 2, "dtype": "uint16"},
    ]
    sc["empty_ops"] = [
        {"op": "new", "shards": 4, "fb": 32, "dtype": "int64"},
        {"op": "insert", "sizes": [0, 0, 0, 0], "base": 0},
        {"op": "dup"},
        {"op": "add", "c": 1, "passes": 2},
        {"op": "commit"},
    ]
    sc["config1_2p20"] = [
        {"op": "new", "shards": 512, "fb": 32, "dtype": "int32"},
        {"op": "insert_split", "n": 1 << 20, "base": 0},
        {"op": "add", "c": 1, "passes": 1},
    ]
    cfg2 = [{"op": "from_flat", "n": 1 << 14, "shards": 64, "fb": 32, "dtype": "int32"}]
    for _ in range(6):
        cfg2 += [{"op": "grow_double"}, {"op": "dup"}, {"op": "add", "c": 1, "passes": 1}]
    sc["config2_small"] = cfg2
    for k in range(16):
        sc[f"random_{k:02d}"] = _random_scenario(k)
    return sc


def baseline_scenarios() -> dict[str, list[dict]]:
    sc: dict[str, list[dict]] = {}
    sc["static_overflow"] = [
        {"op": "b_new", "kind": "static", "cap": 10, "dtype": "int64"},
        {"op": "b_insert", "n": 10, "base": 0},
        {"op": "b_insert", "n": 1, "base": 99},
        {"op": "b_set", "i": 0, "v": 5},
        {"op": "b_get", "i": 0},
        {"op": "b_get", "i": 10},
    ]
    sc["doubling_resize"] = [
        {"op": "b_new", "kind": "doubling", "cap": 4, "dtype": "int64"},
        {"op": "b_insert", "n": 4, "base": 1},
        {"op": "b_resize", "cap": 5},
        {"op": "b_resize", "cap": 3},
        {"op": "b_insert", "n": 4, "base": 10},
        {"op": "b_insert", "n": 1, "base": 10},
        {"op": "b_resize", "cap": 100},
        {"op": "b_insert", "n": 50, "base": 20},
    ]
    sc["doubling_schedule"] = [{"op": "b_new", "kind": "doubling", "cap": 64, "dtype": "int32"},
                               {"op": "b_insert", "n": 64, "base": 0}]
    for _ in range(3):
        sc["doubling_schedule"] += [{"op": "b_resize_double"}, {"op": "b_dup"}]
    sc["chunk_table"] = [
        {"op": "b_new", "kind": "chunktable", "cap": 4, "dtype": "int64"},
        {"op": "b_resize", "cap": 10},
        {"op": "b_insert", "n": 10, "base": 0},
        {"op": "b_insert", "n": 3, "base": 0},
        {"op": "b_resize", "cap": 13},
        {"op": "b_insert", "n": 3, "base": 50},
        {"op": "b_set", "i": 11, "v": -7},
        {"op": "b_get", "i": 11},
    ]
    sc["static_float"] = [
        {"op": "b_new", "kind": "static", "cap": 1000, "dtype": "float32"},
        {"op": "b_insert", "n": 333, "base": 0},
        {"op": "b_dup"},
        {"op": "b_add", "c": 3, "passes": 2},
    ]
    return sc


# ------------------------------------------------------------------ runner

class FailingAllocator:
    """Counting allocator hook; raises MemoryError on the listed (1-based) calls
    (the reference tests' CountingAllocator, test_bucket_vector.py:38-51)."""

    def __init__(self, dtype, fail_calls=()):
        self.dtype = np.dtype(dtype)
        self.fail_calls = set(fail_calls)
        self.calls = 0

    def __call__(self, n):
        self.calls += 1
        if self.calls in self.fail_calls:
            raise MemoryError("injected allocation failure")
        return np.zeros(n, dtype=self.dtype)


def _tags(base: int, n: int, dtype) -> np.ndarray:
    return (np.arange(n, dtype=np.int64) + base).astype(np.dtype(dtype))


def _bytes_digest(a: np.ndarray) -> str:
    b = np.ascontiguousarray(a).tobytes()
    return b.hex() if len(b) <= 2048 else "sha256:" + hashlib.sha256(b).hexdigest()


def _err(exc: BaseException | None):
    if exc is None:
        return None
    out = {"type": type(exc).__name__}
    if hasattr(exc, "failures"):
        out["failures"] = {str(k): type(v).__name__ for k, v in sorted(exc.failures.items())}
    if hasattr(exc, "succeeded"):
        out["succeeded"] = sorted(int(x) for x in exc.succeeded)
    return out


def _state(arr, alloc) -> dict:
    if hasattr(arr, "_parity_state"):
        st = dict(arr._parity_state())
    else:
        st = {
            "sizes": [int(sh.size) for sh in arr.shards],
            "caps": [int(sh.capacity) for sh in arr.shards],
            "flags": [int(sum(1 << b for b, f in enumerate(sh.table.allocated_flags) if f))
                      for sh in arr.shards],
            "prefix": [int(x) for x in arr.prefix],
            "ops": [int(sh.size_counter.op_count) for sh in arr.shards],
        }
    st.pop("alloc_calls", None)
    st["alloc_hook_calls"] = alloc.calls if alloc is not None else None
    try:
        flat = arr.flatten()
        st["flat"] = _bytes_digest(flat)
        st["flat_dtype"] = str(flat.dtype)
    except Exception as exc:  # noqa: BLE001
        st["flat"] = None
        st["flat_err"] = type(exc).__name__
    return st


def _scalar(v):
    v = np.asarray(v)
    return v.item() if v.dtype.kind != "f" else float(v)


def run_scenario(lib, ops: list[dict]) -> list[dict]:
    """Replay ``ops`` through ``lib`` (a module exposing the growarray API)."""
    arr = None
    alloc = None
    out = []
    for op in ops:
        kind = op["op"]
        exc = None
        extra = {}
        try:
            if kind == "new":
                alloc = None
                if "fail_calls" in op or op.get("count_alloc"):
                    alloc = FailingAllocator(op["dtype"], op.get("fail_calls", ()))
                arr = lib.GrowableArray(op["shards"], op["fb"], dtype=np.dtype(op["dtype"]),
                                        max_buckets=op.get("max_buckets", 58), allocator=alloc)
            elif kind == "from_flat":
                alloc = None
                vals = _tags(op.get("base", 0), op["n"], op["dtype"])
                arr = lib.GrowableArray.from_flat(vals, shards=op["shards"],
                                                  first_bucket_size=op["fb"])
            elif kind == "insert":
                base = op["base"]
                batches = []
                for n in op["sizes"]:
                    batches.append(_tags(base, n, arr.dtype))
                    base += n
                arr.insert_parallel(batches, workers=1)
            elif kind == "insert_split":
                vals = _tags(op["base"], op["n"], arr.dtype)
                arr.insert_parallel(lib.split_batches(vals, arr.shard_count), workers=1)
            elif kind == "insert_wrong_count":
                arr.insert_parallel([np.zeros(1, arr.dtype)] * (arr.shard_count - 1), workers=1)
            elif kind == "dup":
                if hasattr(arr, "insert_duplicate"):
                    arr.insert_duplicate()
                else:
                    arr.insert_parallel([sh.to_numpy(arr.committed_length(s))
                                         for s, sh in enumerate(arr.shards)], workers=1)
            elif kind == "grow":
                arr.grow(op["target"], op["dist"])
            elif kind == "grow_double":
                arr.grow(2 * arr.committed_size)
            elif kind == "add":
                if hasattr(arr, "rw_add"):
                    arr.rw_add(op["c"], op["passes"])
                else:
                    c = np.asarray(op["c"]).astype(arr.dtype)
                    for _ in range(op["passes"]):
                        arr.for_each_shard(lambda v, c=c: np.add(v, c, out=v, casting="unsafe"))
            elif kind == "commit":
                arr.commit()
            elif kind == "push":
                r = arr.shards[op["s"]].push_back_batch(_tags(op["base"], op["n"], arr.dtype))
                extra["ret"] = [int(r[0]), int(r[1])] if isinstance(r, tuple) else [r.start, r.count]
            elif kind == "reserve":
                arr.shards[op["s"]].reserve(op["cap"])
            elif kind == "new_bucket":
                extra["ret"] = bool(arr.shards[op["s"]].new_bucket(op["b"]))
            elif kind == "set":
                arr.set_global(op["g"], np.asarray(op["v"]).astype(arr.dtype))
            elif kind == "set_frac":
                n = arr.committed_size
                if n:
                    arr.set_global(int(op["f"] * n), np.asarray(op["v"]).astype(arr.dtype))
            elif kind == "get":
                extra["ret"] = _scalar(arr.get_global(op["g"]))
            else:
                raise AssertionError(f"unknown op {kind}")
        except (ValueError, IndexError, RuntimeError, MemoryError) as e:
            exc = e
        rec = {"op": kind, "err": _err(exc), **extra}
        if arr is not None:
            rec.update(_state(arr, alloc))
        out.append(rec)
    return out


def run_baseline_scenario(lib, ops: list[dict]) -> list[dict]:
    st = None
    out = []
    kinds = {"static": "StaticArray", "doubling": "DoublingArray", "chunktable": "ChunkTableArray"}
    for op in ops:
        kind = op["op"]
        exc = None
        extra = {}
        try:
            if kind == "b_new":
                cls = getattr(lib, kinds[op["kind"]])
                dt = np.dtype(op["dtype"])
                st = (cls(op["cap"], dtype=dt) if op["kind"] == "static" else
                      cls(op["cap"], dtype=dt))
            elif kind == "b_insert":
                st.insert_batch(_tags(op["base"], op["n"], st.dtype))
            elif kind == "b_dup":
                st.insert_batch(st.to_numpy())
            elif kind == "b_resize":
                st.resize(op["cap"])
            elif kind == "b_resize_double":
                st.resize(2 * st.size)
            elif kind == "b_set":
                st.set(op["i"], op["v"])
            elif kind == "b_get":
                extra["ret"] = _scalar(st.get(op["i"]))
            elif kind == "b_add":
                if hasattr(st, "rw_add"):
                    st.rw_add(op["c"], op["passes"])
                else:
                    v = st.view()
                    for _ in range(op["passes"]):
                        np.add(v, np.asarray(op["c"]).astype(st.dtype), out=v, casting="unsafe")
            else:
                raise AssertionError(kind)
        except (ValueError, IndexError, RuntimeError, MemoryError) as e:
            exc = e
        rec = {"op": kind, "err": _err(exc), **extra}
        if st is not None:
            rec.update({"size": int(st.size), "capacity": int(st.capacity),
                        "copied": int(getattr(st, "elements_copied", 0)),
                        "contents": _bytes_digest(st.to_numpy())})
        out.append(rec)
    return out
