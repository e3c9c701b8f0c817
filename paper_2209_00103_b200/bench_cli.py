"""GPU counterpart of the reference harness ``growarray-bench`` (bench_cli.py in
the reference): the same subcommands, flags and CSV schema, run on the B200
structures with CUDA-event phase timing, plus roofline columns.

    python -m paper_2209_00103_b200.bench_cli grow-insert-rw --structure ggarray --shards 512
    python -m paper_2209_00103_b200.bench_cli insert-algos --initial-size 1048576 --iterations 8
    python -m paper_2209_00103_b200.bench_cli shard-sweep --shards 32,512 --initial-size 100000
    python -m paper_2209_00103_b200.bench_cli two-phase --structure ggarray

Every benchmark checks its end state against the sequential oracle of the
reference harness (multiset of tags + passes, bench_cli.py:170-177) before a
row is written; timing columns are informational.  ``memory-model`` is the
reference's section-5 sizing model; ``--measure N`` realises N demands per
sigma as GGArrays on the GPU and appends measured capacity / mapped columns.
"""

from __future__ import annotations

import argparse
import csv
import json
import os
import sys
from dataclasses import dataclass, replace

import numpy as np

STRUCTURES = ("static", "doubling", "chunktable", "ggarray")
ALGOS = ("atomic", "scan", "warp", "block")
RW_MODES = ("global", "per_shard")
BENCH_DTYPE = np.int32
CSV_COLUMNS = [
    "experiment", "structure", "shards", "first_bucket", "workers",
    "initial_size", "iterations", "algo", "rw_mode", "work_passes",
    "repetitions", "seed", "variant", "repetition", "iteration", "phase",
    "elapsed_ns", "size_after", "counter_ops", "copied_elements", "speedup",
    # B200 additions
    "gelem_s", "hbm_gbs", "roofline_frac", "capacity_bytes", "mapped_bytes", "needed_bytes",
]
DEFAULT_SHARD_SWEEP = tuple(2 ** i for i in range(13))
TWO_PHASE_MULTIPLIERS = (1, 3, 10)


class OracleMismatch(RuntimeError):
    """A benchmark end state disagreed with its sequential oracle."""


@dataclass
class BenchConfig:
    structure: str = "ggarray"
    shards: int = 32
    first_bucket: int = 32
    workers: int = 4
    initial_size: int = 100_000
    iterations: int = 10
    algo: str = "scan"
    rw_mode: str = "per_shard"
    work_passes: int = 30
    repetitions: int = 5
    seed: int = 0
    out: str = "-"
    csv_header: bool = True
    rw_grain: int = 65536

    def __post_init__(self):
        if self.structure not in STRUCTURES:
            raise ValueError(f"structure must be one of {STRUCTURES}")
        if self.algo not in ALGOS:
            raise ValueError(f"algo must be one of {ALGOS}")
        if self.rw_mode not in RW_MODES:
            raise ValueError(f"rw_mode must be one of {RW_MODES}")
        for name in ("shards", "workers", "initial_size", "iterations", "work_passes",
                     "repetitions", "rw_grain"):
            if getattr(self, name) < 1:
                raise ValueError(f"{name} must be >= 1")
        fb = self.first_bucket
        if fb < 1 or fb & (fb - 1):
            raise ValueError("first_bucket must be a positive power of two")


def _hbm_peak() -> float:
    try:
        root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
        return float(json.load(open(os.path.join(root, "MEASURED_PEAKS.json")))["hbm_gbs"])
    except (OSError, KeyError, ValueError):
        return 6650.0


class _Timer:
    """CUDA-event timing of one phase on the current stream."""

    def __enter__(self):
        import torch
        self.e0, self.e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        self.e0.record()
        return self

    def __exit__(self, *exc):
        import torch
        self.e1.record()
        torch.cuda.synchronize()
        self.ns = int(self.e0.elapsed_time(self.e1) * 1e6)


def _final_size(config) -> int:
    final = config.initial_size << config.iterations
    if final + config.iterations * config.work_passes >= 2 ** 31:
        raise ValueError(f"schedule reaches {final} elements; too large for 32-bit bench values")
    return final


def _rates(row: dict, elems: int, bytes_per_elem: int = 8) -> dict:
    ns = max(row["elapsed_ns"], 1)
    row["gelem_s"] = round(elems / ns, 3)
    gbs = bytes_per_elem * elems / ns
    row["hbm_gbs"] = round(gbs, 1)
    row["roofline_frac"] = round(gbs / _hbm_peak(), 4)
    return row


def _contents(store):
    import torch
    if hasattr(store, "flatten_device"):
        return store.flatten_device()
    return store.view().clone() if store.size else torch.empty(0, dtype=torch.int32, device="cuda")


def _assert_multiset(actual, expected, context: str) -> None:
    import torch
    a = torch.sort(actual.to(torch.int64)).values
    b = torch.sort(expected.to(torch.int64)).values
    if a.numel() != b.numel() or not torch.equal(a, b):
        raise OracleMismatch(f"{context}: end state disagrees with the sequential oracle")


def _base_record(config, experiment: str) -> dict:
    return {"experiment": experiment, "structure": config.structure, "shards": config.shards,
            "first_bucket": config.first_bucket, "workers": config.workers,
            "initial_size": config.initial_size, "iterations": config.iterations,
            "algo": config.algo, "rw_mode": config.rw_mode, "work_passes": config.work_passes,
            "repetitions": config.repetitions, "seed": config.seed}


def _mem(store) -> dict:
    if hasattr(store, "memory_stats"):
        m = store.memory_stats()
        return {"capacity_bytes": m["capacity_bytes"], "mapped_bytes": m["mapped_bytes"],
                "needed_bytes": m["needed_bytes"]}
    cap = store.capacity * store.dtype.itemsize
    return {"capacity_bytes": cap, "mapped_bytes": getattr(store, "mapped_bytes", cap),
            "needed_bytes": store.size * store.dtype.itemsize}


def _build(config, initial, final):
    import paper_2209_00103_b200 as gg
    if config.structure == "ggarray":
        return gg.GrowableArray.from_flat(initial, config.shards, config.first_bucket)
    if config.structure == "static":
        st = gg.StaticArray(final, dtype=BENCH_DTYPE)
    elif config.structure == "doubling":
        st = gg.DoublingArray(max(1, initial.numel()), dtype=BENCH_DTYPE)
    else:
        st = gg.ChunkTableArray(dtype=BENCH_DTYPE)
        st.resize(initial.numel())
    if initial.numel():
        st.insert_batch(initial)
    return st


def _insert_flat(store, vals, algo: str) -> None:
    # reference algos: atomic (one counter op per element), scan (one per group
    # of 32 lanes = warp aggregation); plus the B200 block-scan variant
    store.insert_batch(vals, algo={"atomic": "atomic", "scan": "warp", "warp": "warp",
                                   "block": "block"}[algo])


def _insert_duplicate(store, config) -> None:
    if hasattr(store, "insert_duplicate"):
        store.insert_duplicate()
    else:
        _insert_flat(store, store.view().clone(), config.algo)


def _grow(store, target: int) -> None:
    if hasattr(store, "grow"):
        store.grow(target)
    else:
        store.resize(target)


def _rw(store, passes: int, mode: str) -> None:
    if hasattr(store, "rw_add"):
        if hasattr(store, "shard_count"):
            store.rw_add(1, passes=passes, mode=mode)
        else:
            store.rw_add(1, passes=passes)


def _flat_rw(t, passes: int) -> None:
    """+1 sweeps over a contiguous device tensor (the two-phase work phase)."""
    import ctypes as C
    import torch
    from . import _lib as L
    one = np.ones(1, BENCH_DTYPE)
    L.check(L.lib.gg_flat_add(C.c_void_p(t.data_ptr()), t.numel(), L.DTYPE_CODES[np.dtype(BENCH_DTYPE)],
                              one.ctypes.data_as(C.c_void_p), int(passes), 0,
                              torch.cuda.current_stream().cuda_stream), "flat_add")


def _ops(store) -> int:
    if hasattr(store, "shards"):
        return int(store._host()["ops"].sum())
    return int(store.size_counter.op_count)


# ---------------------------------------------------------------------------- experiments
def bench_insert_algos(config) -> list:
    """Duplication rounds on the static array under each reservation algorithm
    (bench_cli.py:422-463): one atomic per element vs one per warp (scan) vs one
    per CTA (block); counter traffic recorded; contents must agree."""
    import torch
    import paper_2209_00103_b200 as gg
    final = _final_size(config)
    rows = []
    for algo in ("atomic", "scan", "block"):
        for rep in range(config.repetitions):
            st = gg.StaticArray(final, dtype=BENCH_DTYPE)
            st.insert_batch(torch.arange(config.initial_size, dtype=torch.int32, device="cuda"))
            tag = config.initial_size
            for it in range(config.iterations):
                n = st.size
                vals = torch.arange(tag, tag + n, dtype=torch.int32, device="cuda")
                ops0 = st.size_counter.op_count
                with _Timer() as t:
                    _insert_flat(st, vals, algo)
                tag += n
                r = _base_record(config, "insert-algos")
                r.update(structure="static", algo=algo, variant=algo, repetition=rep, iteration=it,
                         phase="insert", elapsed_ns=t.ns, size_after=st.size,
                         counter_ops=st.size_counter.op_count - ops0, **_mem(st))
                rows.append(_rates(r, n))
            _assert_multiset(st.view(), torch.arange(final, device="cuda"), f"insert-algos[{algo}]")
    return rows


def bench_shard_sweep(config, s_list=None) -> list:
    """Grow + duplicate-insert rounds and rw in both modes per shard count
    (bench_cli.py:466-505)."""
    import torch
    import paper_2209_00103_b200 as gg
    s_list = list(s_list if s_list is not None else DEFAULT_SHARD_SWEEP)
    if not s_list:
        raise ValueError("s_list must be non-empty")
    _final_size(config)
    rows = []
    for S in s_list:
        for rep in range(config.repetitions):
            init = torch.arange(config.initial_size, dtype=torch.int32, device="cuda")
            arr = gg.GrowableArray.from_flat(init, S, config.first_bucket)
            oracle = init.to(torch.int64)
            for it in range(config.iterations):
                base = _base_record(config, "shard-sweep")
                base.update(structure="ggarray", shards=S, variant=f"S={S}", repetition=rep, iteration=it)
                with _Timer() as t:
                    arr.grow(2 * arr.committed_size)
                rows.append(dict(base, phase="grow", elapsed_ns=t.ns, size_after=arr.committed_size,
                                 **_mem(arr)))
                n = arr.committed_size
                with _Timer() as t:
                    arr.insert_duplicate()
                rows.append(_rates(dict(base, phase="insert", elapsed_ns=t.ns,
                                        size_after=arr.committed_size, **_mem(arr)), n))
                oracle = torch.cat([oracle, oracle])
                for mode in ("global", "per_shard"):
                    with _Timer() as t:
                        arr.rw_add(1, passes=config.work_passes, mode=mode)
                    rows.append(_rates(dict(base, phase="rw", rw_mode=mode, elapsed_ns=t.ns,
                                            size_after=arr.committed_size),
                                       arr.committed_size * config.work_passes))
                oracle += 2 * config.work_passes
            _assert_multiset(arr.flatten_device(), oracle, f"shard-sweep[S={S}]")
    return rows


def bench_grow_insert_rw(config) -> list:
    """Per duplication round: grow, insert one element per existing element, rw
    passes -- for the configured structure (bench_cli.py:508-543)."""
    import torch
    final = _final_size(config)
    rows = []
    for rep in range(config.repetitions):
        init = torch.arange(config.initial_size, dtype=torch.int32, device="cuda")
        store = _build(config, init, final)
        oracle = init.to(torch.int64)
        for it in range(config.iterations):
            base = _base_record(config, "grow-insert-rw")
            base.update(variant=config.structure, repetition=rep, iteration=it)
            size = store.committed_size if hasattr(store, "committed_size") else store.size
            if config.structure != "static":
                c0 = getattr(store, "elements_copied", 0)
                with _Timer() as t:
                    _grow(store, 2 * size)
                rows.append(dict(base, phase="grow", elapsed_ns=t.ns, size_after=size,
                                 copied_elements=getattr(store, "elements_copied", 0) - c0, **_mem(store)))
            ops0 = _ops(store)
            with _Timer() as t:
                _insert_duplicate(store, config)
            after = store.committed_size if hasattr(store, "committed_size") else store.size
            rows.append(_rates(dict(base, phase="insert", elapsed_ns=t.ns, size_after=after,
                                    counter_ops=_ops(store) - ops0, **_mem(store)), size))
            oracle = torch.cat([oracle, oracle])
            with _Timer() as t:
                _rw(store, config.work_passes, config.rw_mode)
            rows.append(_rates(dict(base, phase="rw", rw_mode=config.rw_mode, elapsed_ns=t.ns,
                                    size_after=after), after * config.work_passes))
            oracle += config.work_passes
        _assert_multiset(_contents(store), oracle, f"grow-insert-rw[{config.structure}]")
    return rows


def _two_phase_run(config, kind: str, start: int, k: int, final: int):
    import torch
    from paper_2209_00103_b200.sharded_array import split_offsets
    store = _build(replace(config, structure=kind), torch.arange(start, dtype=torch.int32, device="cuda"), final)
    oracle = torch.arange(start, dtype=torch.int64, device="cuda")
    tag, total, phases = start, 0, []
    for it in range(config.iterations):
        size = store.committed_size if hasattr(store, "committed_size") else store.size
        m = final - size if it == config.iterations - 1 else min(k * size, final - size)
        vals = torch.arange(tag, tag + m, dtype=torch.int32, device="cuda")
        tag += m
        with _Timer() as t:
            if kind == "ggarray":
                S = store.shard_count
                chunk = -(-m // S) if m else 0
                off = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(chunk), np.uint64(m))
                store.insert_csr(vals, off)
            else:
                if kind != "static":
                    store.resize(size + m)
                _insert_flat(store, vals, config.algo)
        total += t.ns
        after = store.committed_size if hasattr(store, "committed_size") else store.size
        phases.append(dict(iteration=it, phase="insert", elapsed_ns=t.ns, size_after=after))
        oracle = torch.cat([oracle, vals.to(torch.int64)])
        if kind == "ggarray":
            with _Timer() as t:
                flat = store.flatten_device()
            f_ns = t.ns
            with _Timer() as t:
                _flat_rw(flat, config.work_passes)
            w_ns = t.ns
            with _Timer() as t:
                # rebuild (from_flat's re-sharding, sharded_array.py:259-282) into
                # the same handle: the reset keeps its buckets mapped, so the
                # rebuild is one planned insert, no VMM driver call
                store.shrink(0, release=False)
                store.insert_csr(flat, split_offsets(int(flat.numel()), store.shard_count))
            f_ns += t.ns
            total += f_ns + w_ns
            phases.append(dict(iteration=it, phase="flatten", elapsed_ns=f_ns, size_after=after))
            phases.append(dict(iteration=it, phase="work", elapsed_ns=w_ns, size_after=after))
        else:
            with _Timer() as t:
                _rw(store, config.work_passes, config.rw_mode)
            total += t.ns
            phases.append(dict(iteration=it, phase="work", elapsed_ns=t.ns, size_after=after))
        oracle += config.work_passes
    end = store.committed_size if hasattr(store, "committed_size") else store.size
    if end != final:
        raise OracleMismatch(f"two-phase[{kind}, k={k}]: ended at {end}, expected {final}")
    _assert_multiset(_contents(store), oracle, f"two-phase[{kind}, k={k}]")
    return phases, total, end


def bench_two_phase(config) -> list:
    """Insertion phases alternating with work phases; the dynamic structure
    flattens before each work phase and rebuilds after it (bench_cli.py:546-643,
    paper Fig. 6), compared against the chunk-table (memMap) baseline."""
    final = _final_size(config)
    kinds = ["chunktable"] + ([config.structure] if config.structure != "chunktable" else [])
    rows = []
    for k in TWO_PHASE_MULTIPLIERS:
        start = max(1, final // (1 + k) ** config.iterations)
        base_tot = {}
        for kind in kinds:
            role = "baseline" if kind == "chunktable" else "candidate"
            for rep in range(config.repetitions):
                phases, total, end = _two_phase_run(config, kind, start, k, final)
                base = _base_record(config, "two-phase")
                base.update(structure=kind, variant=f"mult={k}:{role}", repetition=rep)
                rows += [dict(base, **ph) for ph in phases]
                tr = dict(base, iteration="", phase="total", elapsed_ns=total, size_after=end)
                if role == "baseline":
                    base_tot[rep] = total
                    if len(kinds) == 1:
                        tr["speedup"] = 1.0
                else:
                    tr["speedup"] = round(base_tot[rep] / max(total, 1), 4)
                rows.append(tr)
    return rows


def write_rows(rows, out, header: bool = True) -> None:
    def emit(fh):
        w = csv.DictWriter(fh, fieldnames=CSV_COLUMNS, restval="", lineterminator="\n")
        if header:
            w.writeheader()
        w.writerows(rows)
    if out in ("-", None):
        emit(sys.stdout)
    elif hasattr(out, "write"):
        emit(out)
    else:
        with open(out, "w", encoding="utf-8", newline="") as fh:
            emit(fh)


def _parse_shards(text: str) -> list:
    try:
        vals = [int(p) for p in str(text).split(",") if p.strip()]
    except ValueError as exc:
        raise argparse.ArgumentTypeError(f"bad shard list {text!r}") from exc
    if not vals or any(v < 1 for v in vals):
        raise argparse.ArgumentTypeError(f"shard counts must be >= 1, got {text!r}")
    return vals


def build_parser() -> argparse.ArgumentParser:
    p = argparse.ArgumentParser(prog="ggarray-bench",
                                description="B200 GGArray benchmark harness (growarray-bench schema).")
    sub = p.add_subparsers(dest="command", required=True)
    c = argparse.ArgumentParser(add_help=False)
    c.add_argument("--structure", choices=STRUCTURES, default="ggarray")
    c.add_argument("--shards", type=_parse_shards, default=[32])
    c.add_argument("--first-bucket", type=int, default=32)
    c.add_argument("--workers", type=int, default=4)
    c.add_argument("--initial-size", type=int, default=100_000)
    c.add_argument("--iterations", type=int, default=10)
    c.add_argument("--algo", choices=ALGOS, default="scan")
    c.add_argument("--rw-mode", choices=RW_MODES, default="per_shard")
    c.add_argument("--work-passes", type=int, default=30)
    c.add_argument("--repetitions", type=int, default=5)
    c.add_argument("--seed", type=int, default=0)
    c.add_argument("--out", default="-")
    c.add_argument("--csv-header", action=argparse.BooleanOptionalAction, default=True)
    c.add_argument("--rw-grain", type=int, default=65536)
    for name in ("insert-algos", "shard-sweep", "grow-insert-rw", "two-phase"):
        sub.add_parser(name, parents=[c])
    mm = sub.add_parser("memory-model", parents=[c])
    mm.add_argument("--samples", type=int, default=100_000)
    mm.add_argument("--base-size", type=int, default=1_000_000)
    mm.add_argument("--element-size", type=int, default=4)
    mm.add_argument("--measure", type=int, default=0,
                    help="demands per sigma realised as GGArrays on the GPU (0 = model only)")
    return p


def main(argv=None) -> int:
    args = build_parser().parse_args(argv)
    if args.command != "shard-sweep" and len(args.shards) != 1:
        raise SystemExit(f"{args.command}: --shards takes a single value")
    if args.command == "memory-model":          # bench_cli.py:725-738 in the reference
        from . import memory_model as mmod
        params = mmod.MemoryModelParams(base_size=args.base_size, samples=args.samples, seed=args.seed)
        reports = mmod.run_model(params, shards=args.shards[0], first_bucket_size=args.first_bucket,
                                 element_size=args.element_size)
        measured = None
        if args.measure:
            measured = mmod.measure_device(params, args.measure, shards=args.shards[0],
                                           first_bucket_size=args.first_bucket,
                                           element_size=args.element_size)
        mmod.write_report_csv(reports, sys.stdout if args.out == "-" else args.out,
                              header=args.csv_header, measured=measured)
        return 0
    cfg = BenchConfig(structure=args.structure, shards=args.shards[0], first_bucket=args.first_bucket,
                      workers=args.workers, initial_size=args.initial_size,
                      iterations=args.iterations, algo=args.algo, rw_mode=args.rw_mode,
                      work_passes=args.work_passes, repetitions=args.repetitions, seed=args.seed,
                      out=args.out, csv_header=args.csv_header, rw_grain=args.rw_grain)
    fn = {"insert-algos": bench_insert_algos, "grow-insert-rw": bench_grow_insert_rw,
          "two-phase": bench_two_phase}.get(args.command)
    rows = bench_shard_sweep(cfg, args.shards) if args.command == "shard-sweep" else fn(cfg)
    write_rows(rows, cfg.out, header=cfg.csv_header)
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
