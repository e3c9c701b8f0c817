"""Generate tests/golden/memory_model.json from the UNMODIFIED reference
memory model (imported read-only from /root/reference/pkg/src): run_model
rows for a few (seed, shards, base) settings, normal_quantile values and the
CLI's CSV text.  Run here:  python tests/golden/make_memory_model_golden.py
"""
import dataclasses
import io
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, "/root/reference/pkg/src")

from growarray import memory_model as M  # noqa: E402
from growarray import bench_cli  # noqa: E402


def main():
    out = {"generator": "tests/golden/make_memory_model_golden.py", "runs": [], "quantile": {}}
    for seed, shards, fb, base, samples in [(0, 32, 32, 1_000_000, 4000), (3, 512, 32, 1 << 20, 3000),
                                            (7, 8, 4, 777, 2500)]:
        p = M.MemoryModelParams(base_size=base, samples=samples, seed=seed)
        reps = M.run_model(p, shards=shards, first_bucket_size=fb)
        out["runs"].append({"seed": seed, "shards": shards, "fb": fb, "base": base, "samples": samples,
                            "rows": [dataclasses.asdict(r) for r in reps]})
    for p in [1e-9, 1e-4, 0.01, 0.02425, 0.3, 0.5, 0.9, 0.975, 0.99, 1 - 1e-6]:
        out["quantile"][repr(p)] = M.normal_quantile(p)
    buf = io.StringIO()
    sys.stdout, old = buf, sys.stdout
    try:
        bench_cli.main(["memory-model", "--samples", "500", "--base-size", "5000", "--shards", "16",
                        "--seed", "5"])
    finally:
        sys.stdout = old
    out["cli_csv"] = {"argv": ["memory-model", "--samples", "500", "--base-size", "5000", "--shards",
                               "16", "--seed", "5"], "text": buf.getvalue()}
    with open(os.path.join(HERE, "memory_model.json"), "w") as fh:
        json.dump(out, fh, indent=0)
    print("wrote memory_model.json")


if __name__ == "__main__":
    main()
