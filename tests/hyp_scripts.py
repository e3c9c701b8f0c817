"""Hypothesis strategy for GGArray op scripts in the scenarios.py JSON format
(the same ops the golden scenarios use): random shard counts, first-bucket
sizes, dtypes, ragged inserts, duplicates, grows (uniform and explicit),
r/w passes, sets, pushes, reserves and commits."""
from hypothesis import strategies as st

import scenarios

DTYPES = ["int32", "int64", "float32", "float64", "int8", "uint16", "uint64", "float16"]


@st.composite
def op_scripts(draw, max_ops=9):
    S = draw(st.sampled_from([1, 2, 3, 7, 16, 33]))
    fb = draw(st.sampled_from([1, 2, 4, 32, 64]))
    dtype = draw(st.sampled_from(DTYPES))
    ops = [{"op": "new", "shards": S, "fb": fb, "dtype": dtype, "max_buckets": 58}]
    tag = 0
    for _ in range(draw(st.integers(1, max_ops))):
        kind = draw(st.sampled_from(["insert", "insert", "dup", "grow", "grow_dist", "add", "set_frac",
                                     "push", "reserve", "commit"]))
        if kind == "insert":
            sizes = draw(st.lists(st.integers(0, 3 * fb + 50), min_size=S, max_size=S))
            ops.append({"op": "insert", "sizes": sizes, "base": tag})
            tag += sum(sizes)
        elif kind == "dup":
            ops.append({"op": "dup"})
        elif kind == "grow":
            ops.append({"op": "grow", "target": draw(st.integers(0, 3000)), "dist": None})
        elif kind == "grow_dist":
            ops.append({"op": "grow", "target": 0,
                        "dist": draw(st.lists(st.integers(0, 400), min_size=S, max_size=S))})
        elif kind == "add":
            ops.append({"op": "add", "c": draw(st.integers(1, 3)), "passes": draw(st.integers(1, 3))})
        elif kind == "set_frac":
            ops.append({"op": "set_frac", "f": draw(st.floats(0, 0.999)), "v": draw(st.integers(0, 99))})
        elif kind == "push":
            ops.append({"op": "push", "s": draw(st.integers(0, S - 1)), "n": draw(st.integers(0, 2 * fb + 9)),
                        "base": tag})
            tag += 1000
        elif kind == "reserve":
            ops.append({"op": "reserve", "s": draw(st.integers(0, S - 1)), "cap": draw(st.integers(0, 700))})
        else:
            ops.append({"op": "commit"})
    ops.append({"op": "commit"})
    ops.append({"op": "add", "c": 1, "passes": 1})
    return ops


run = scenarios.run_scenario
