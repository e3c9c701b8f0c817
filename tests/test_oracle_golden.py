"""Pin the CPU oracle (oracle/ggoracle.py) against golden states recorded from
the unmodified reference package (tests/golden/make_golden.py)."""
import json
import os

import numpy as np
import pytest

from oracle import ggoracle as O
import scenarios

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = json.load(open(os.path.join(ROOT, "tests", "golden", "golden.json")))


@pytest.mark.parametrize("name", sorted(GOLDEN["ggarray"]))
def test_oracle_matches_reference_scenario(name):
    case = GOLDEN["ggarray"][name]
    got = scenarios.run_scenario(O, case["ops"])
    assert len(got) == len(case["states"])
    for k, (g, want) in enumerate(zip(got, case["states"])):
        assert g == want, f"{name} step {k} ({case['ops'][k]['op']})"


@pytest.mark.parametrize("name", sorted(GOLDEN["baselines"]))
def test_oracle_baselines_match_reference(name):
    case = GOLDEN["baselines"][name]
    got = scenarios.run_baseline_scenario(O, case["ops"])
    for k, (g, want) in enumerate(zip(got, case["states"])):
        assert g == want, f"{name} step {k}"


@pytest.mark.parametrize("fb", ["1", "2", "32", "1024"])
def test_locate_tables(fb):
    t = GOLDEN["locate"][fb]
    f = int(fb)
    assert [list(O.locate(i, f)) for i in t["idx"]] == t["loc"]
    b, off = O.locate_many(np.asarray(t["idx"]), f)
    assert [[int(x), int(y)] for x, y in zip(b, off)] == t["loc"]
    assert [O.min_buckets_for(n, f) for n in t["idx"][:300]] == t["min_buckets"]
    assert [O.capacity_of(k, f) for k in range(40)] == t["capacity_of"]


def test_capacity_model():
    cm = GOLDEN["capacity_model"]
    assert [int(x) for x in O.sharded_capacity_elements(cm["demands"], 512, 32)] == cm["S512_fb32"]
    assert [int(x) for x in O.sharded_capacity_elements(cm["demands"], 8, 4)] == cm["S8_fb4"]


def test_spec_known_answers():
    # SPEC.md / test_bucket_vector.py:63-75,116-122 and memory config goldens
    assert O.locate(0, 1) == (0, 0) and O.locate(6, 1) == (2, 3) and O.locate(5, 2) == (1, 3)
    assert [O.min_buckets_for(n, 32) for n in (0, 1, 32, 33, 97)] == [0, 1, 1, 2, 3]
    assert int(O.sharded_capacity_elements([1 << 20], 512, 32)[0]) == 2_080_768
    assert int(O.sharded_capacity_elements([1 << 30], 512, 32)[0]) == 2_147_467_264
    assert list(O.split_offsets(2, 4)) == [0, 1, 2, 2, 2]
    assert O.exclusive_scan([4, 0, 5]) == [0, 4, 4]
