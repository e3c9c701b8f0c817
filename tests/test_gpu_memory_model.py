"""The sizing model's GGArray column realised on the B200: device capacity of
lognormal demands equals the closed form; mapped slab bytes stay near it."""
import pytest

from paper_2209_00103_b200 import memory_model as M

pytestmark = pytest.mark.gpu


def test_measure_device_matches_closed_form():
    p = M.MemoryModelParams(base_size=200_000, samples=100, seed=3)
    rows = M.measure_device(p, 3, shards=32, first_bucket_size=32, sigma_grid=[0.0, 0.7, 1.5])
    assert [r["sigma"] for r in rows] == [0.0, 0.7, 1.5]
    for r in rows:
        assert r["samples"] == 3
        assert r["mapped_mean"] >= r["capacity_mean"] > 0


def test_cli_memory_model_measure(capsys):
    from paper_2209_00103_b200 import bench_cli
    assert bench_cli.main(["memory-model", "--samples", "200", "--base-size", "100000", "--shards", "32",
                           "--measure", "2"]) == 0
    lines = capsys.readouterr().out.splitlines()
    assert lines[0].split(",") == M.CSV_COLUMNS + M.MEASURED_COLUMNS
    assert len(lines) == 22
