"""Section-5 sizing model (paper_2209_00103_b200/memory_model.py) against rows,
quantiles and CLI text recorded from the reference (tests/golden/
make_memory_model_golden.py), plus the reference's own invariants
(test_memory_model.py in the reference).  CPU only; the device-measured
columns are in tests/test_gpu_memory_model.py."""
import dataclasses
import io
import json
import os

import numpy as np
import pytest

from paper_2209_00103_b200 import memory_model as M

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "memory_model.json")))


@pytest.mark.parametrize("run", GOLD["runs"], ids=lambda r: f"seed{r['seed']}_S{r['shards']}")
def test_run_model_rows_match_reference(run):
    p = M.MemoryModelParams(base_size=run["base"], samples=run["samples"], seed=run["seed"])
    got = M.run_model(p, shards=run["shards"], first_bucket_size=run["fb"])
    assert len(got) == len(run["rows"]) == 21
    for g, w in zip(got, run["rows"]):
        g = dataclasses.asdict(g)
        for k in ("sigma", "element_size", "optimal_bytes", "ggarray_capacity_bytes",
                  "ggarray_worst_bytes", "ggarray_ratio", "ggarray_worst_ratio"):
            assert g[k] == w[k], k                      # same RNG stream, same integer model
        for k in ("static_p_bytes", "static_ratio"):    # quantile: AS241 vs Acklam+Halley
            assert g[k] == pytest.approx(w[k], rel=1e-12), k


def test_normal_quantile_matches_reference():
    for p, want in GOLD["quantile"].items():
        # the reference loses ~1e-11 near p -> 1 (1 - p cancellation); its own bar vs scipy is 1e-8
        assert M.normal_quantile(float(p)) == pytest.approx(want, rel=1e-10, abs=1e-12)
    for bad in (0.0, 1.0, -0.1, 1.1):
        with pytest.raises(ValueError):
            M.normal_quantile(bad)


def test_cli_csv_matches_reference():
    from paper_2209_00103_b200 import bench_cli
    import contextlib
    buf = io.StringIO()
    with contextlib.redirect_stdout(buf):
        assert bench_cli.main(GOLD["cli_csv"]["argv"]) == 0
    got = [l.split(",") for l in buf.getvalue().splitlines()]
    want = [l.split(",") for l in GOLD["cli_csv"]["text"].splitlines()]
    assert got[0] == want[0] == M.CSV_COLUMNS
    for g, w in zip(got[1:], want[1:]):
        assert np.allclose([float(x) for x in g], [float(x) for x in w], rtol=1e-12, atol=0)
    assert len(got) == len(want) == 22


def test_params_validation_and_static_sizing():
    with pytest.raises(ValueError):
        M.MemoryModelParams(failure_prob=0.0)
    with pytest.raises(ValueError):
        M.MemoryModelParams(sigma=-1)
    assert M.static_requirement(M.MemoryModelParams(sigma=0.0, base_size=1000), 4) == pytest.approx(4000.0)
    reqs = [M.static_requirement(M.MemoryModelParams(sigma=s, base_size=1000)) for s in np.linspace(0, 2, 21)]
    assert all(a <= b for a, b in zip(reqs, reqs[1:]))


def test_capacity_bound_sweep():
    S, fb = 32, 32
    d = np.arange(1, 100_001)
    caps = M.sharded_capacity_elements(d, S, fb)
    assert np.all(caps < 2 * d + S * fb) and np.all(caps >= d)
    assert M.ggarray_capacity_for(33, shards=1, first_bucket_size=32, element_size=1) == 96


def test_csv_with_measured_columns_schema():
    p = M.MemoryModelParams(base_size=1000, samples=50, seed=1)
    reps = M.run_model(p, sigma_grid=[0.0, 1.0])
    meas = [{"samples": 2, "capacity_mean": 1.0, "mapped_mean": 2.0, "mapped_ratio": 1.5,
             "mapped_ratio_max": 1.7}] * 2
    buf = io.StringIO()
    M.write_report_csv(reps, buf, measured=meas)
    lines = buf.getvalue().splitlines()
    assert lines[0].split(",") == M.CSV_COLUMNS + M.MEASURED_COLUMNS and len(lines) == 3
