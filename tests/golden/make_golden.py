"""Generate tests/golden/golden.json by replaying tests/scenarios.py through the
UNMODIFIED reference package (imported read-only from /root/reference/pkg/src).

Run here (the reference is not on the GPU box):  python tests/golden/make_golden.py
The JSON stores each scenario's ops next to the recorded states, so the
fixture is self-contained; tests replay the stored ops.
"""
import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))            # tests/
sys.path.insert(0, "/root/reference/pkg/src")

import growarray  # noqa: E402
import scenarios  # noqa: E402


def main():
    out = {"generator": "tests/golden/make_golden.py",
           "reference": "growarray " + growarray.__version__ + " @ /root/reference/pkg/src",
           "ggarray": {}, "baselines": {}, "locate": {}}
    for name, ops in scenarios.scenarios().items():
        out["ggarray"][name] = {"ops": ops, "states": scenarios.run_scenario(growarray, ops)}
    for name, ops in scenarios.baseline_scenarios().items():
        out["baselines"][name] = {"ops": ops, "states": scenarios.run_baseline_scenario(growarray, ops)}
    # layout known-answer tables (bucket_vector.py:48-79)
    import numpy as np
    rng = np.random.default_rng(7)
    for fb in (1, 2, 32, 1024):
        idx = list(range(0, 2000)) + [int(x) for x in rng.integers(0, 1 << 40, 200)]
        out["locate"][str(fb)] = {
            "idx": idx,
            "loc": [list(growarray.locate(i, fb)) for i in idx],
            "min_buckets": [growarray.min_buckets_for(n, fb) for n in idx[:300]],
            "capacity_of": [growarray.capacity_of(k, fb) for k in range(40)],
        }
    demands = [0, 1, 31, 32, 33, 1000, 99999, 1 << 20, (1 << 20) + 5, 1 << 30]
    out["capacity_model"] = {
        "demands": demands,
        "S512_fb32": [int(x) for x in growarray.sharded_capacity_elements(demands, 512, 32)],
        "S8_fb4": [int(x) for x in growarray.sharded_capacity_elements(demands, 8, 4)],
    }
    with open(os.path.join(HERE, "golden.json"), "w") as fh:
        json.dump(out, fh, separators=(",", ":"))
    print("wrote", os.path.join(HERE, "golden.json"), os.path.getsize(os.path.join(HERE, "golden.json")))


if __name__ == "__main__":
    main()
