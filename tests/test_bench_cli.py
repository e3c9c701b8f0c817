"""GPU benchmark CLI (paper_2209_00103_b200.bench_cli): same subcommands, flags
and CSV schema as the reference harness (pkg/tests/test_bench_cli.py)."""
import io

import pytest

from paper_2209_00103_b200 import bench_cli as B


def test_config_defaults_and_validation():
    B.BenchConfig()
    for kw in ({"structure": "x"}, {"algo": "x"}, {"rw_mode": "x"}, {"shards": 0},
               {"first_bucket": 3}, {"iterations": 0}):
        with pytest.raises(ValueError):
            B.BenchConfig(**kw)


def test_schema_extends_the_reference_columns():
    ref = ["experiment", "structure", "shards", "first_bucket", "workers", "initial_size",
           "iterations", "algo", "rw_mode", "work_passes", "repetitions", "seed", "variant",
           "repetition", "iteration", "phase", "elapsed_ns", "size_after", "counter_ops",
           "copied_elements", "speedup"]
    assert B.CSV_COLUMNS[:len(ref)] == ref


def test_csv_lf_and_header():
    buf = io.StringIO()
    B.write_rows([{"experiment": "x", "elapsed_ns": 5}], buf)
    text = buf.getvalue()
    assert text.startswith("experiment,") and "\r" not in text and text.count("\n") == 2
    buf = io.StringIO()
    B.write_rows([{"experiment": "x"}], buf, header=False)
    assert buf.getvalue().startswith("x,")


def test_parser_and_schedule_guard():
    a = B.build_parser().parse_args(["shard-sweep", "--shards", "1,4"])
    assert a.shards == [1, 4]
    with pytest.raises(ValueError):
        B._final_size(B.BenchConfig(initial_size=1 << 30, iterations=4))


@pytest.mark.gpu
@pytest.mark.parametrize("structure", ["ggarray", "static", "doubling", "chunktable"])
def test_grow_insert_rw_oracle(structure):
    cfg = B.BenchConfig(structure=structure, shards=8, initial_size=1000, iterations=3,
                        work_passes=2, repetitions=1)
    rows = B.bench_grow_insert_rw(cfg)
    assert rows and rows[-1]["size_after"] == 8000
    if structure == "doubling":
        assert sum(r.get("copied_elements", 0) for r in rows) == 1000 + 2000 + 4000
    if structure == "chunktable":
        assert sum(r.get("copied_elements", 0) for r in rows) == 0


@pytest.mark.gpu
def test_insert_algos_counter_ops():
    cfg = B.BenchConfig(initial_size=1000, iterations=2, repetitions=1)
    rows = B.bench_insert_algos(cfg)
    ops = {(r["algo"], r["iteration"]): r["counter_ops"] for r in rows}
    assert ops[("atomic", 0)] == 1000 and ops[("scan", 0)] == -(-1000 // 32)


@pytest.mark.gpu
def test_shard_sweep_and_two_phase():
    cfg = B.BenchConfig(initial_size=500, iterations=2, work_passes=2, repetitions=1)
    assert B.bench_shard_sweep(cfg, [1, 4])
    rows = B.bench_two_phase(B.BenchConfig(shards=4, initial_size=512, iterations=2,
                                           work_passes=2, repetitions=1))
    totals = [r for r in rows if r["phase"] == "total"]
    assert len(totals) == 6 and all(r["size_after"] == 2048 for r in totals)
