"""Is the CPU arm (the oracle port) a fair stand-in for the reference's own
CPU path?  Times the config-2 doubling schedule (2^20 -> 2^27, S=512 int32)
through the unmodified reference package (this container only: it reads
/root/reference) and through oracle.doubling_schedule_cpu, at 1 and all
threads, best of 3 each."""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, "/root/reference/pkg/src")
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import growarray as G  # noqa: E402
from oracle import ggoracle as O  # noqa: E402

N0, S, FB, R = 1 << 20, 512, 32, 7
cores = len(os.sched_getaffinity(0))


def ref_sched(workers):
    t0 = time.perf_counter()
    arr = G.GrowableArray.from_flat(np.arange(N0, dtype=np.int32), S, FB, np.int32)
    ins = N0
    for _ in range(R):
        n = arr.committed_size
        arr.grow(2 * n)
        snaps = [arr.shards[s].to_numpy(arr.committed_length(s)) for s in range(S)]
        arr.insert_parallel(snaps, workers=workers)
        ins += n
    return ins / (time.perf_counter() - t0) / 1e9


def port(threads):
    t0 = time.perf_counter()
    _, ins, _, _ = O.doubling_schedule_cpu(N0, R, S, FB, np.int32, threads)
    return ins / (time.perf_counter() - t0) / 1e9


res = {"cores": cores, "schedule": "S=512 int32 2^20 -> 2^27, Gelem/s, best of 3"}
for w in (1, cores):
    res[f"reference_workers_{w}"] = round(max(ref_sched(w) for _ in range(3)), 4)
    res[f"port_threads_{w}"] = round(max(port(w) for _ in range(3)), 4)
print(json.dumps(res))
