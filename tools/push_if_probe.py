"""push_if (the device push_back API from a user kernel, paper Alg. 1/2)
throughput at 2^28 candidates over 512 LFVectors, predicate density 1/2:
events around the public call (host view prepare / finish inside) for block
and warp aggregation and every element size, with the multiset check.
Bytes = values + predicates read + kept values written.  A/B builds via
GG_LIB_PATH; PROBE_GRID overrides the grid (0 = the library's default)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_00103_b200 as gg

S, FB = 512, 32
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
PEAK = json.load(open(os.path.join(ROOT, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6548.5) \
    if os.path.exists(os.path.join(ROOT, "MEASURED_PEAKS.json")) else 6548.5
dev = torch.device("cuda", 0)
TD = {1: torch.int8, 2: torch.int16, 4: torch.int32, 8: torch.int64}
ND = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}
GRID = int(os.environ.get("PROBE_GRID", "0"))
out = {"peak": PEAK, "grid": GRID}


CHAIN = 4


def run(esz, mode, N=1 << 28, density=0.5, reps=5, chained=True):
    vals = (torch.arange(N, device=dev) % 100003).to(TD[esz])
    g = torch.Generator(device=dev).manual_seed(7)
    pred = (torch.rand(N, device=dev, generator=g) < density).to(torch.uint8)
    tot = int(pred.sum())
    a = gg.GrowableArray(S, FB, dtype=ND[esz])
    a.push_if(vals, pred, mode=mode, grid=GRID, commit=False)
    best = 1e9
    for _ in range(reps):
        a.shrink(0, release=False)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record()
        a.push_if(vals, pred, mode=mode, grid=GRID, commit=False)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    a.commit()
    kept = torch.sort(vals[pred.bool()])[0]
    ok = bool(torch.equal(torch.sort(a.flatten_device())[0], kept))
    nbytes = (esz + 1) * N + esz * tot
    res = {"candidates": N, "appended": tot, "ms": round(best, 4),
           "gbs": round(nbytes / (best * 1e-3) / 1e9, 1),
           "frac": round(nbytes / (best * 1e-3) / 1e9 / PEAK, 4),
           "gelem_s": round(tot / (best * 1e-3) / 1e9, 2), "multiset_ok": ok}
    if chained and N >= 1 << 24:
        # CHAIN back-to-back calls between two events: each plans on the
        # previous calls' upper bounds instead of waiting for their readback
        best_c = 1e9
        for _ in range(3):
            a.shrink(0, release=False)
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
            e0.record()
            for _ in range(CHAIN):
                a.push_if(vals, pred, mode=mode, grid=GRID, commit=False)
            e1.record()
            torch.cuda.synchronize()
            best_c = min(best_c, e0.elapsed_time(e1) / CHAIN)
        a.commit()
        okc = bool(torch.equal(torch.sort(a.flatten_device())[0], torch.sort(kept.repeat(CHAIN))[0]))
        res["chained"] = {"calls": CHAIN, "ms_per_call": round(best_c, 4),
                          "frac": round(nbytes / (best_c * 1e-3) / 1e9 / PEAK, 4), "multiset_ok": okc}
    a.close()
    return res


ONLY = os.environ.get("PROBE_ONLY")           # e.g. "block_e4": one config (ncu)
if ONLY:
    mode, e = ONLY.split("_e")
    out[ONLY] = run(int(e), mode, reps=1)
    print(json.dumps(out))
    sys.exit(0)
out["block_e4_2p20"] = run(4, "block", N=1 << 20)
for esz in (4, 1, 2, 8):
    for mode in ("block", "warp"):
        out[f"{mode}_e{esz}"] = run(esz, mode)
        torch.cuda.empty_cache()
out["block_e4_d0.05"] = run(4, "block", density=0.05)
out["block_e4_d0.95"] = run(4, "block", density=0.95)
print(json.dumps(out))
