"""GGArray benchmark (BASELINE.json config 2 is the headline; configs 3-5 are
reported beside it).

A *step* is the config-2 insertion phase on one GPU: reset the array (all
buckets back to the arena free lists), insert 2^20 int32 over 512 LFVectors
(from a device-resident batch), then 10 doubling rounds of {grow(2n);
every LFVector appends a copy of its committed contents; commit} up to 2^30
elements.  ``value`` = elements inserted / device time of the K timed steps
(Gelem/s, whole job = sum over ranks / max-over-ranks time).

Usage: python bench.py [--gpus N] [--steps K] [--warmup W] [--impl reference]
Under torchrun (N>1) every rank owns its own 512 LFVectors (weak scaling) and
the only cross-GPU step is the all-gather of the per-GPU committed sizes that
forms the global directory.
"""

from __future__ import annotations

import argparse
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

S, FB, N0, ROUNDS = 512, 32, 1 << 20, 10
METRIC = "GGArray insert Gelem/s"
UNIT = "Gelem/s"
WORKLOAD = "config2: GGArray-512 doubling 2^20->2^30 int32 (grow + duplicate-insert per round)"


def config_dict(world: int) -> dict:
    """The workload both arms (GPU and --impl reference) run, per GPU."""
    return {"workload": WORKLOAD, "shards_per_gpu": S, "first_bucket_size": FB,
            "initial_elements": N0, "rounds": ROUNDS, "final_elements_per_gpu": 1 << 30,
            "parallelism": f"lfvector-sharded x{world}",
            "l2": "inputs larger than L2 (4 GiB live, 8 GiB capacity per GPU)"}


def _ncu_traffic():
    """dram read+write bytes of the dominant kernel's largest launch, from the
    newest committed ncu summary (profiles/rNN_ncu_summary.json)."""
    import glob
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_ncu_summary.json")))
    for f in reversed(files):
        try:
            for e in json.load(open(f))["full_capture"]:
                if "W_DUP" in e.get("label", ""):
                    return {"bytes_per_launch": e["traffic_bytes"], "algorithmic_bytes": e["algorithmic_bytes"],
                            "ratio": e["traffic_over_algorithmic"], "source": os.path.relpath(f, ROOT),
                            "launch": "last doubling round, 2^29 elements"}
        except (OSError, KeyError, ValueError):
            continue
    return None


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            return json.load(fh), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0}, "fallback"


# --------------------------------------------------------------------------- clocks
class ClockSampler:
    """Polls NVML (SM clock + throttle reasons) every 1 ms on a thread while the
    timed region runs (the headline region is ~13 ms); falls back to nothing
    if NVML is unavailable."""

    def __init__(self, index: int, period_s: float = 0.001):
        self.index, self.period, self.rows, self._stop = index, period_s, [], None

    def __enter__(self):
        import threading
        try:
            import pynvml as N
            N.nvmlInit()
            self._N, self._h = N, N.nvmlDeviceGetHandleByIndex(self.index)
            self.max_mhz = N.nvmlDeviceGetMaxClockInfo(self._h, N.NVML_CLOCK_SM)
        except Exception:  # noqa: BLE001
            self._N = None
            return self
        self._stop = threading.Event()

        def poll():
            while not self._stop.is_set():
                self._sample()
                self._stop.wait(self.period)
        self._t = threading.Thread(target=poll, daemon=True)
        self._t.start()
        return self

    def _sample(self):
        N, h = self._N, self._h
        try:
            self.rows.append((N.nvmlDeviceGetClockInfo(h, N.NVML_CLOCK_SM),
                              N.nvmlDeviceGetCurrentClocksEventReasons(h)))
        except Exception:  # noqa: BLE001
            pass

    def sample_now(self):
        """One synchronous sample (call while the device is still busy)."""
        if self._stop is not None:
            self._sample()

    def __exit__(self, *exc):
        if self._stop is not None:
            self._stop.set()
            self._t.join()

    def summary(self) -> dict:
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": getattr(self, "max_mhz", None),
                    "reasons": ["unsampled"], "samples": 0}
        N = self._N
        bits = {"hw_slowdown": N.nvmlClocksEventReasonHwSlowdown,
                "hw_thermal_slowdown": N.nvmlClocksEventReasonHwThermalSlowdown,
                "sw_thermal_slowdown": N.nvmlClocksEventReasonSwThermalSlowdown,
                "sw_power_cap": N.nvmlClocksEventReasonSwPowerCap}
        sm = sorted(r[0] for r in self.rows)
        reasons = sorted({k for _, m in self.rows for k, bit in bits.items() if m & bit})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.rows), "source": "nvml (1 ms poll thread + host polling while the queued replays run)"}


# --------------------------------------------------------------------------- device legs
def _events(torch):
    return torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)


class Step:
    """One config-2 schedule on a persistent array; per-phase CUDA events."""

    def __init__(self, gg, torch, device, dtype=np.int32):
        self.gg, self.torch = gg, torch
        self.arr = gg.GrowableArray(S, FB, dtype=dtype, device=device)
        tdt = {np.int32: torch.int32, np.float32: torch.float32, np.int64: torch.int64}[dtype]
        self.vals = torch.arange(N0, dtype=tdt, device=device)
        self.offsets = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(N0 // S), N0)
        self.dup_ms, self.grow_ms, self.dup_elems = [], [], 0

    def run(self, timed_phases: bool):
        a, torch = self.arr, self.torch
        a.shrink(0, release=False)                    # reset: buckets cached in place
        a.insert_csr(self.vals, self.offsets)         # 2^20 initial elements
        ev = []
        for _ in range(ROUNDS):
            n = a.committed_size
            if timed_phases:
                e0, e1, e2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
                e0.record()
                a.grow(2 * n)
                e1.record()
                a.insert_duplicate()
                e2.record()
                ev.append((e0, e1, e2, n))
            else:
                a.grow(2 * n)
                a.insert_duplicate()
        return ev

    def collect(self, ev):
        for e0, e1, e2, n in ev:
            self.grow_ms.append(e0.elapsed_time(e1))
            self.dup_ms.append(e1.elapsed_time(e2))
            self.dup_elems += n


def run_device(args, rank, world, local_rank):
    import torch
    import paper_2209_00103_b200 as gg
    from paper_2209_00103_b200 import _lib
    dist = None
    if world > 1:
        import torch.distributed as dist
    device = torch.device("cuda", local_rank)
    torch.cuda.set_device(device)
    peaks, peaks_kind = _peaks()
    hbm = float(peaks.get("hbm_gbs", 6650.0))

    # once per process and device: CUDA context + the library's kernel image
    # (gg_create would do it at the first construction); reported, not in any step
    i0 = time.perf_counter()
    _lib.check(_lib.lib.gg_init(local_rank), "init")
    init_ms = (time.perf_counter() - i0) * 1e3
    gg.pool_trim(local_rank)
    c0 = time.perf_counter()
    step = Step(gg, torch, device)
    construct_ms = (time.perf_counter() - c0) * 1e3
    # the very first step on a fresh array also maps its 8 GiB of slab chunks
    # (driver work the steady-state steps reuse): reported, not in `value`
    torch.cuda.synchronize()
    c0 = time.perf_counter()
    step.run(False)
    torch.cuda.synchronize()
    sl = step.arr.slab_stats()
    cold = {"ms": round((time.perf_counter() - c0) * 1e3, 3),
            "map_ms": round(sl["map_ns"] / 1e6, 3), "extents_mapped": sl["chunks_mapped"],
            "driver_handles_created": sl["handles_created"],
            "library_init_ms": round(init_ms, 3), "array_construct_ms": round(construct_ms, 3),
            "note": "first step of a fresh array in a fresh process (pool trimmed), wall clock, incl. "
                    "cuMemCreate/Map/SetAccess of its 8 GiB of slab extents; the once-per-process "
                    "library init (CUDA context + kernel image load, gg_init) and the array "
                    "construction are reported beside it"}
    for _ in range(args.warmup):
        step.run(False)
    torch.cuda.synchronize()
    # eager, host-driven steps with per-phase events (phases, dominant kernel)
    e0, e1 = _events(torch)
    e0.record()
    h0 = time.perf_counter()
    evs = [step.run(True) for _ in range(args.steps)]
    host_ms = (time.perf_counter() - h0) * 1e3
    e1.record()
    torch.cuda.synchronize()
    eager_ms = e0.elapsed_time(e1)
    for ev in evs:
        step.collect(ev)
    # the same step captured once in a CUDA graph (host planning done at capture;
    # every kernel of the step runs on each replay)
    graph = step.arr.capture(lambda: step.run(False))
    for _ in range(args.warmup):
        graph.replay()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    launches0 = _lib.lib.gg_kernel_launches()
    sampler = ClockSampler(local_rank)
    with sampler:
        t0, t1 = _events(torch)
        torch.cuda.synchronize()
        t0.record()
        for _ in range(args.steps):
            graph.replay()
        t1.record()
        while not t1.query():            # the replays are queued: sample while they run
            sampler.sample_now()
            time.sleep(0.001)
        torch.cuda.synchronize()
    # graph replays do not pass through the launch counter: count the kernels
    # the captured step launches (same as one eager step) per replay
    launches = launches_per_step(step) * args.steps
    ms = t0.elapsed_time(t1)
    check_state(step, torch)
    if dist:
        t = torch.tensor([ms], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        # global directory: all-gather of per-GPU committed sizes (the one exchange)
        sizes = [torch.zeros(1, dtype=torch.int64, device=device) for _ in range(world)]
        dist.all_gather(sizes, torch.tensor([step.arr.committed_size], device=device))
    inserted_per_step = 1 << 30                        # 2^20 initial + sum of duplicates
    value = world * inserted_per_step * args.steps / (ms * 1e-3) / 1e9
    eager_value = world * inserted_per_step * args.steps / (eager_ms * 1e-3) / 1e9

    a = step.arr
    assert a.committed_size == 1 << 30
    traffic = _ncu_traffic()
    mem = a.memory_stats()
    dup_bytes = 8 * step.dup_elems                     # read 4 + write 4 per element
    dup_ms = sum(step.dup_ms)
    achieved = dup_bytes / (dup_ms * 1e-3) / 1e9
    last_round = [m for i, m in enumerate(step.dup_ms) if i % ROUNDS == ROUNDS - 1]
    last_gbs = (8 * (1 << 29)) / (np.mean(last_round) * 1e-3) / 1e9
    out = {
        "metric": METRIC, "value": round(value, 3), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms / args.steps, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
        "data": "synthetic (np.arange tags, as bench_cli.py)",
        "config": config_dict(world),
        "gpu_launches": int(launches),
        "roofline": {"bound": "hbm", "kernel": "k_walk<4,W_DUP> (duplicate insert, all 10 rounds)",
                     "achieved": round(achieved, 1), "peak": hbm, "unit": "GB/s",
                     "frac": round(achieved / hbm, 4), "peak_kind": peaks_kind,
                     "traffic": (traffic or {}).get("bytes_per_launch"),
                     "traffic_detail": traffic, "algorithmic_bytes_per_elem": 8,
                     "achieved_def": "sum of 8 B x elements duplicated / sum of CUDA-event times around "
                                     "the insert_duplicate calls of the K eager steps (the planned "
                                     "copy walk k_walk<W_DUP> with its metadata CTA, which also "
                                     "publishes the deferred grow)",
                     "last_round_2p29_gbs": round(float(last_gbs), 1),
                     "last_round_frac": round(float(last_gbs) / hbm, 4)},
        "phases": {"insert_ms_per_step": round(dup_ms / args.steps, 4),
                   "insert_ms_by_round": [round(float(np.mean(step.dup_ms[r::ROUNDS])), 4)
                                          for r in range(ROUNDS)],
                   "grow_ms_per_step": round(sum(step.grow_ms) / args.steps, 4),
                   "insert_only_gelem_s": round(step.dup_elems / (dup_ms * 1e-3) / 1e9, 2)},
        "footprint": {"needed_bytes": mem["needed_bytes"], "capacity_bytes": mem["capacity_bytes"],
                      "mapped_bytes": mem["mapped_bytes"],
                      "capacity_over_needed": round(mem["capacity_over_needed"], 6),
                      "mapped_over_needed": round(mem["mapped_over_needed"], 6)},
        "clocks": sampler.summary(),
        "timing": "value: K replays of the step captured once as a CUDA graph; "
                  "eager: the same K steps issued op by op from Python",
        "eager": {"value": round(eager_value, 3), "ms_per_step": round(eager_ms / args.steps, 4),
                  "host_enqueue_ms_per_step": round(host_ms / args.steps, 4)},
        "cold_first_step": {**cold, "x_warm_step": round(cold["ms"] / (ms / args.steps), 2)},
    }
    if dist:
        out["gather_flatten"] = gather_leg(args, torch, device, step, dist, world)
    if not args.quick:
        _between_legs(gg)
        out["cold_steps"] = cold_leg(args, gg, torch, device, ms / args.steps)
        _between_legs(gg)
        out.update(secondary(args, gg, torch, device, step, hbm))
        _between_legs(gg)
        out["config2_dtypes"] = dtype_variants(args, gg, torch, device, hbm)
        _between_legs(gg)
        out["phased_config4"] = phased_leg(args, gg, torch, device)
        _between_legs(gg)
        out["insert_paths"] = insert_paths_leg(args, gg, torch, device, hbm)
        _between_legs(gg)
        out["config5_per_gpu"] = config5_leg(args, gg, torch, device, hbm)
        _between_legs(gg)
        out["config1"] = config1_leg(args, gg, torch, device, rank == 0 and world == 1 and not args.no_cpu)
        _between_legs(gg)
        out["e2e"] = e2e_leg(args, gg, torch, device, world, dist)
    if rank == 0 and world == 1 and not args.no_cpu:
        out["cpu_baseline"] = cpu_baseline(args)
    return out


def gather_leg(args, torch, device, step, dist, world):
    """Config 5's exchange step: every GPU's 2^30-element array gathered into
    rank 0 by the fused flatten into peer memory (CUDA IPC over NVLink /
    NVSwitch, multigpu.PeerGather).  Device time = max over ranks of the
    flatten launch; bytes over NVLink = all slices but the root's own."""
    try:
        from paper_2209_00103_b200.multigpu import DistributedGrowableArray, PeerGather
        d = DistributedGrowableArray(step.arr, device=device)
        ok_peer, why = d.peer_topology()
        pre = d.global_prefix()
        # bytes each rank moves into the root's buffer (the root's own slice stays local)
        per_rank = [0 if r == 0 else (pre[r + 1] - pre[r]) * 4 for r in range(world)]
        if not ok_peer:
            return fallback_gather_leg(torch, device, d, dist, pre, per_rank, why)
        g = PeerGather(d, 0)
        g.run(); g.wait()
        k = 3
        e0, e1 = _events(torch)
        dist.barrier()
        e0.record()
        for _ in range(k):
            g.run()
        e1.record()
        g.wait()
        t = torch.tensor([e0.elapsed_time(e1) / k], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
        total = g.prefix[-1] * 4
        nvlink = total - (g.prefix[1] - g.prefix[0]) * 4
        ok = True
        if dist.get_rank() == 0:
            flat = g.result()
            per = step.arr.committed_size
            ok = bool(torch.equal(flat[:per], step.arr.flatten_device()))
            del flat
        g.close()
        del g
        torch.cuda.empty_cache()
        nccl = None
        if dist.get_backend() == "nccl":
            # the library baseline for the same exchange: local K-flatten into
            # a staging buffer, then NCCL gather to the root
            local = step.arr.flatten_device()
            glist = [torch.empty_like(local) for _ in range(world)] if dist.get_rank() == 0 else None

            def nccl_gather():
                step.arr.flatten_device(out=local)
                dist.gather(local, glist, dst=0)
            nccl_gather()
            torch.cuda.synchronize()
            dist.barrier()
            e0.record()
            for _ in range(k):
                nccl_gather()
            e1.record()
            torch.cuda.synchronize()
            t = torch.tensor([e0.elapsed_time(e1) / k], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            nms = float(t.item())
            nccl = {"ms": round(nms, 4), "nvlink_gbs_into_root": round(nvlink / (nms * 1e-3) / 1e9, 1),
                    "method": "flatten_device + torch.distributed.gather (NCCL)"}
            if dist.get_rank() == 0:
                nccl["root_slice_ok"] = bool(torch.equal(glist[0], local))
            del local, glist
            torch.cuda.empty_cache()
        # even rebalance: every rank ends with N/G of the global flat array
        d.rebalance_flat_peer()
        dist.barrier()
        e0.record()
        part, (lo, hi) = d.rebalance_flat_peer()
        e1.record()
        torch.cuda.synchronize()
        t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        rb_ms = float(t.item())
        del part
        torch.cuda.empty_cache()
        return {"ms": round(ms, 4), "bytes_total": total, "bytes_over_nvlink": nvlink,
                "bytes_over_nvlink_per_rank": per_rank, "peer_topology": "ok",
                "nvlink_gbs_into_root": round(nvlink / (ms * 1e-3) / 1e9, 1),
                "root_slice_ok": ok, "method": "fused K-flatten into the root buffer (CUDA IPC)",
                "rebalance_ms_incl_setup": round(rb_ms, 3),
                "rebalance": "even slices N/G per rank, K-flatten ranges into the owners' buffers",
                "nccl_baseline": nccl}
    except Exception as exc:                          # report, never lose the bench line
        return {"error": repr(exc)[:300]}


def fallback_gather_leg(torch, device, d, dist, pre, per_rank, why):
    """No peer access between the ranks' GPUs (multigpu.peer_topology): the
    same gather through DistributedGrowableArray.flatten_global's NCCL path
    (local K-flatten + point-to-point into the root), with the reason."""
    e0, e1 = _events(torch)
    d.flatten_global(0, method="nccl")
    torch.cuda.synchronize()
    dist.barrier()
    e0.record()
    out = d.flatten_global(0, method="nccl")
    e1.record()
    torch.cuda.synchronize()
    t = torch.tensor([e0.elapsed_time(e1)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms = float(t.item())
    ok = True
    if dist.get_rank() == 0:
        n0 = pre[1] - pre[0]
        ok = bool(torch.equal(out[:n0].to(device), d.local.flatten_device()))
    del out
    torch.cuda.empty_cache()
    moved = sum(per_rank)
    return {"ms": round(ms, 4), "bytes_total": pre[-1] * 4, "bytes_over_nvlink": moved,
            "bytes_over_nvlink_per_rank": per_rank, "gbs_into_root": round(moved / (ms * 1e-3) / 1e9, 1),
            "root_slice_ok": ok, "method": f"fallback: {d.last_method} (local K-flatten + point-to-point)",
            "peer_topology": "unavailable", "fallback_reason": why}


def _between_legs(gg):
    """Outside every timed region: collect garbage (the collector is off
    during the run, so no teardown lands inside a timed loop) and free what
    dropped arrays left behind."""
    import gc
    gc.collect()
    gg.reclaim(True)


def cold_leg(args, gg, torch, device, warm_ms):
    """The first config-2 step of a FRESH array, wall clock (host planning,
    driver calls, kernels): (1) after pool_trim, every slab extent comes from
    cuMemCreate; (2) after that array was destroyed, a new same-shape array
    adopts its slab from the process slab cache (the two-phase / rebuild
    pattern: no driver call)."""
    out = {}
    gg.pool_trim(device.index)
    for tag in ("driver", "adopted_slab"):
        st = Step(gg, torch, device)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st.run(False)
        torch.cuda.synchronize()
        ms = (time.perf_counter() - t0) * 1e3
        sl = st.arr.slab_stats()
        check_state(st, torch)
        out[tag] = {"ms": round(ms, 3), "x_warm_step": round(ms / warm_ms, 2),
                    "map_ms": round(sl["map_ns"] / 1e6, 3), "extents_mapped": sl["chunks_mapped"],
                    "driver_handles_created": sl["handles_created"],
                    "handles_from_pool": sl["handles_from_pool"]}
        st.arr.close()
        del st
        gg.reclaim(True)
    out["note"] = "wall clock of one full step on a new GrowableArray, array construction excluded"
    return out


def launches_per_step(step) -> int:
    from paper_2209_00103_b200 import _lib
    import torch
    c0 = _lib.lib.gg_kernel_launches()
    step.run(False)
    torch.cuda.synchronize()
    return int(_lib.lib.gg_kernel_launches() - c0)


def check_state(step, torch) -> None:
    """After the replays: device state == host mirror, and the contents equal
    the closed form of the schedule (element g = (g // 2^21) * 2048 + g % 2048)."""
    a = step.arr
    dev, host = a.device_state(), a._host()
    for k in ("sizes", "caps", "flags", "prefix"):      # ops counts replays: not a fixed point
        assert np.array_equal(dev[k], host[k]), f"device/host mismatch in {k} after replays"
    assert int(dev["prefix"][-1]) == 1 << 30
    idx = torch.randint(0, 1 << 30, (1 << 16,), device="cuda", dtype=torch.int64)
    got = a.get_many(idx).to(torch.int64)
    per = (N0 // S) << ROUNDS
    exp = (idx // per) * (N0 // S) + idx % (N0 // S)
    assert torch.equal(got, exp), "schedule contents differ from the closed form"


def _time(torch, fn, reps=1):
    e0, e1 = _events(torch)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def dtype_variants(args, gg, torch, device, hbm):
    """The config-2 schedule for the other element types of SURVEY 8(d)
    (float32 = same values cast; int64 = 2x the bytes), graph-replayed like
    the headline and checked against the closed form."""
    res = {}
    for name, dt, esz in (("float32", np.float32, 4), ("int64", np.int64, 8)):
        st = Step(gg, torch, device, dtype=dt)
        st.run(False)
        g = st.arr.capture(lambda: st.run(False))
        for _ in range(max(3, args.warmup)):
            g.replay()
        reps = max(3, args.steps)
        ms = _time(torch, lambda: [g.replay() for _ in range(reps)]) / reps
        check_state(st, torch)
        res[name] = {"ms_per_step": round(ms, 4), "gelem_s": round((1 << 30) / ms / 1e6, 2),
                     "gbs": round(2 * esz * (1 << 30) / ms / 1e6, 1),
                     "frac": round(2 * esz * (1 << 30) / ms / 1e6 / hbm, 4), "contents_ok": True}
        del g
        st.arr.close()
        del st
    return res


def secondary(args, gg, torch, device, step, hbm):
    """Configs 3 (r/w), flatten, and the static / semi-static / memMap baselines."""
    a = step.arr
    n = a.committed_size
    passes = args.rw_passes
    res = {}
    # --- config 3: 100 x (+1) sweeps over 2^30 elements
    rw = {}
    for mode in ("per_shard", "global"):
        p = passes if mode == "per_shard" else max(1, passes // 10)
        a.rw_add(1, passes=1, mode=mode)
        ms = _time(torch, lambda: a.rw_add(1, passes=p, mode=mode)) / p
        rw[f"ggarray_{mode}"] = {"ms_per_pass": round(ms, 4), "gbs": round(8 * n / ms / 1e6, 1),
                                 "frac": round(8 * n / ms / 1e6 / hbm, 4), "passes": p}
    ms = _time(torch, lambda: a.rw_add(1, passes=passes, mode="fused"))
    rw["ggarray_fused_100_in_registers"] = {"ms": round(ms, 4)}
    # every +1 above landed exactly once per element: sample against the closed form
    adds = (1 + passes) + (1 + max(1, passes // 10)) + passes
    idx = torch.randint(0, n, (1 << 16,), device=device, dtype=torch.int64)
    per = (N0 // S) << ROUNDS
    exp = (idx // per) * (N0 // S) + idx % (N0 // S) + adds
    rw["contents_ok_after_passes"] = bool(torch.equal(a.get_many(idx).to(torch.int64), exp))
    a.rw_add(-adds)                                  # back to the schedule's contents
    flat = a.flatten_device()
    fl_ms = _time(torch, lambda: a.flatten_device(out=flat), reps=5)
    res["flatten"] = {"ms": round(fl_ms, 4), "gbs": round(8 * n / fl_ms / 1e6, 1),
                      "frac": round(8 * n / fl_ms / 1e6 / hbm, 4)}
    from paper_2209_00103_b200 import _lib
    import ctypes as C
    one = np.ones(1, np.int32)
    fl = lambda: _lib.lib.gg_flat_add(C.c_void_p(flat.data_ptr()), n, 4, one.ctypes.data_as(C.c_void_p),
                                      passes, 0, torch.cuda.current_stream().cuda_stream)
    ms = _time(torch, fl) / passes
    rw["flattened_contiguous"] = {"ms_per_pass": round(ms, 4), "gbs": round(8 * n / ms / 1e6, 1),
                                  "frac": round(8 * n / ms / 1e6 / hbm, 4)}
    res["rw_config3"] = rw
    # --- two-phase usage (paper section 6): grow -> flatten -> static work -> rebuild.
    # from_flat re-shards the flat array into a fresh GGArray (one planned CSR
    # insert); the first build maps new slabs, the second reuses the chunk pool.
    flat.sub_(passes)                                # flat_add put +passes on the copy: back to a's contents
    tp = {"flatten_ms": res["flatten"]["ms"], "static_rw_ms_per_pass": rw["flattened_contiguous"]["ms_per_pass"]}
    for tag in ("rebuild_cold", "rebuild_pooled"):
        if tag == "rebuild_cold":
            gg.pool_trim(device.index)               # fresh driver memory: no cached handles or slabs
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        w0 = time.perf_counter()
        e0.record()
        b = gg.GrowableArray.from_flat(flat, shards=S, first_bucket_size=FB, dtype=np.int32, device=device)
        e1.record()
        torch.cuda.synchronize()
        wall = (time.perf_counter() - w0) * 1e3
        sl = b.slab_stats()
        tp[tag] = {"wall_ms": round(wall, 3), "device_ms": round(e0.elapsed_time(e1), 3),
                   "gelem_s": round(n / wall / 1e6, 2), "driver_handles_created": sl["handles_created"],
                   "handles_from_pool": sl["handles_from_pool"], "extents_mapped": sl["chunks_mapped"],
                   "adopted_slab_bytes": int(b.memory_stats(settle=False)["mapped_bytes"]) if not sl["chunks_mapped"] else 0}
        if tag == "rebuild_pooled":
            tp["roundtrip_ok"] = bool(torch.equal(b.flatten_device(), flat))
            # steady two-phase loop: reuse the GGArray (reset keeps its buckets mapped)
            from paper_2209_00103_b200.sharded_array import split_offsets
            offs = split_offsets(n, S)

            def reuse():
                b.shrink(0, release=False)
                b.insert_csr(flat, offs)
            reuse()
            ms = _time(torch, reuse, reps=5)
            tp["rebuild_reuse"] = {"device_ms": round(ms, 4), "gelem_s": round(n / ms / 1e6, 2),
                                   "gbs": round(8 * n / ms / 1e6, 1)}
            tp["reuse_roundtrip_ok"] = bool(torch.equal(b.flatten_device(), flat))
        b.close()
        del b
        gg.reclaim(True)                             # b's slab -> the slab cache (same shape next)
    tp["note"] = ("rebuild = GrowableArray.from_flat(flat) into a FRESH array: rebuild_cold after "
                  "pool_trim (cuMemCreate/Map/SetAccess of 8 GiB), rebuild_pooled adopts the slab the "
                  "destroyed cold array left (no driver call); rebuild_reuse = shrink(0) + insert_csr "
                  "into the same array")
    res["two_phase"] = tp
    del flat
    # --- baselines: the last doubling step 2^29 -> 2^30 (paper Table II)
    half = 1 << 29
    src = torch.arange(half, dtype=torch.int32, device=device)
    base = {}
    st = gg.StaticArray(1 << 30, dtype=np.int32, device=device)
    st.insert_batch(src)
    for algo in ("atomic", "warp", "block", None):
        def ins(algo=algo):
            st._count = half
            st._d_count.fill_(half)
            st.insert_batch(src, algo=algo)
        ins()
        ms = _time(torch, ins, reps=3)
        base[f"static_insert_{algo or 'batch'}"] = {
            "ms": round(ms, 4), "gelem_s": round(half / ms / 1e6, 2),
            "gbs": round(8 * half / ms / 1e6, 1), "frac": round(8 * half / ms / 1e6 / hbm, 4)}
    assert bool(torch.equal(st.view()[half:], src)), "static insert_batch contents"
    base["static_insert_batch"]["kernel"] = "k_flat_append (one reservation, 16 B vector copy)"
    base["static_insert_block"]["kernel"] = "k_flat_insert_block (one atomicAdd per 32 KiB tile, 16 B stores)"
    ms = _time(torch, lambda: st.rw_add(1, passes=passes)) / passes
    base["static_rw"] = {"ms_per_pass": round(ms, 4), "gbs": round(8 * (1 << 30) / ms / 1e6, 1)}
    del st
    torch.cuda.empty_cache()
    # semi-static doubling: resize (new + D2D copy + free), then insert
    g_ms, i_ms = [], []
    for _ in range(3):
        d = gg.DoublingArray(half, dtype=np.int32, device=device)
        d.insert_batch(src)
        torch.cuda.synchronize()
        g_ms.append(_time(torch, lambda: d.resize(1 << 30)))
        i_ms.append(_time(torch, lambda: d.insert_batch(src)))
        del d
    base["doubling"] = {"grow_ms": round(min(g_ms), 4), "insert_ms": round(min(i_ms), 4),
                        "insert_gelem_s": round(half / min(i_ms) / 1e6, 2),
                        "insert": "insert_batch (one reservation + k_flat_append)",
                        "grow": "cudaMallocAsync(2^30) + zero + D2D copy of 2^29 + free (host-resized)"}
    # memMap (VMM append, no copy)
    g_ms, i_ms = [], []
    for _ in range(3):
        c = gg.ChunkTableArray(dtype=np.int32, device=device)
        c.resize(half)
        c.insert_batch(src)
        torch.cuda.synchronize()
        g_ms.append(_time(torch, lambda: c.resize(1 << 30)))
        i_ms.append(_time(torch, lambda: c.insert_batch(src)))
        del c
    base["memmap"] = {"grow_ms": round(min(g_ms), 4), "insert_ms": round(min(i_ms), 4),
                      "insert_gelem_s": round(half / min(i_ms) / 1e6, 2),
                      "insert": "insert_batch (one reservation + k_flat_append)",
                      "grow": "cuMemCreate/Map/SetAccess of 2 GiB more (64 MiB pieces) + zero"}
    # GGArray's grow of the same step from FRESH driver memory, like memMap's
    # (the steady-state step below grows into chunks its reset kept mapped)
    from paper_2209_00103_b200.sharded_array import split_offsets
    g_ms, mapped = [], 0
    for _ in range(3):
        gg.pool_trim(device.index)
        e = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
        e.insert_csr(src, split_offsets(half, S))
        e.flush()
        torch.cuda.synchronize()
        m0 = e.memory_stats(settle=False)["mapped_bytes"]
        g_ms.append(_time(torch, lambda: (e.grow(1 << 30), e.flush())))
        mapped = e.memory_stats(settle=False)["mapped_bytes"] - m0
        e.close()
        del e
        gg.reclaim(True)
    base["ggarray512_cold_grow"] = {"grow_ms": round(min(g_ms), 4), "mapped_bytes": int(mapped),
                                    "grow": "grow(2^30) on a fresh array after pool_trim: cuMemCreate/Map/"
                                            "SetAccess of the new bucket class (one extent) + k_grow"}
    # ggarray, same last step
    last = step.dup_ms[ROUNDS - 1::ROUNDS]
    lastg = step.grow_ms[ROUNDS - 1::ROUNDS]
    base["ggarray512"] = {"grow_ms": round(float(np.mean(lastg)), 4),
                          "insert_ms": round(float(np.mean(last)), 4),
                          "insert_gelem_s": round(half / float(np.mean(last)) / 1e6, 2)}
    res["baselines_last_doubling_2p29"] = base
    del src
    torch.cuda.empty_cache()
    res["baselines_full_schedule"] = full_schedule_baselines(gg, torch, device, step, args)
    return res


def insert_paths_leg(args, gg, torch, device, hbm):
    """The insert paths beside config 2's uniform doubling, at 2^28 int32 over
    512 LFVectors (inputs and arrays far larger than L2):
      * ragged CSR insert: per-LFVector batch sizes uniform in [0, 2 x mean]
        (BASELINE config 4's distribution), then the duplicate of that ragged
        array (every LFVector's source and destination start at another
        offset mod 16 B), its flatten and a +1 r/w pass -- the shard-grid walk
        (k_walk_shard); 8 B algorithmic per element;
      * paper Alg. 1 with per-lane counts (insert_lanes): lanes of K values,
        counts uniform in [0, K]; algorithmic bytes = counts (4 B / lane) +
        the [lanes x K] value block the counts select from + the compacted
        output (the layout the API takes), the useful bytes (counts + kept
        values read + written) beside it; `chained`: 4 back-to-back calls per
        event pair (each planned on the previous calls' upper bounds);
      * push_if (the device push_back API from a kernel): 2^28 candidates,
        predicate density 1/2; bytes = values + predicates read + kept written.
    Eager timings are CUDA events around the public call (host planning and
    the deferred metadata pass, flushed, inside); graph timings replay the
    reset + insert captured once (device time)."""
    from paper_2209_00103_b200.sharded_array import split_offsets  # noqa: F401
    N = 1 << 28
    rng = np.random.default_rng(0)
    out = {"elements": N, "shards": S}

    def rec(name, ms, nbytes, elems, extra=None):
        gbs = nbytes / (ms * 1e-3) / 1e9
        out[name] = {"ms": round(ms, 4), "gbs": round(gbs, 1), "frac": round(gbs / hbm, 4),
                     "gelem_s": round(elems / (ms * 1e-3) / 1e9, 2), **(extra or {})}

    def best(fn, reset, reps=5):
        ms = 1e9
        for _ in range(reps):
            reset()
            torch.cuda.synchronize()
            e0, e1 = _events(torch)
            e0.record()
            fn()
            e1.record()
            torch.cuda.synchronize()
            ms = min(ms, e0.elapsed_time(e1))
        return ms

    counts = rng.integers(0, 2 * (N // S) + 1, S).astype(np.int64)
    counts = (counts * (N / counts.sum())).astype(np.int64)
    counts[-1] += N - counts.sum()
    off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
    src = torch.arange(N, dtype=torch.int32, device=device)
    a = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
    a.insert_csr(src, off)
    a.insert_duplicate()
    reset = lambda: a.shrink(0, release=False)
    rec("ragged_insert_csr", best(lambda: (a.insert_csr(src, off), a.flush()), reset), 8 * N, N)

    def chained_csr(calls=4):
        # back-to-back public calls between two events: each call's host
        # planning overlaps the previous call's kernel (no readback between)
        for _ in range(calls):
            a.insert_csr(src, off)
        a.flush()
    ms4 = best(chained_csr, reset)
    out["ragged_insert_csr"]["chained"] = {
        "calls": 4, "ms_per_call": round(ms4 / 4, 4),
        "frac": round(8 * N / (ms4 / 4 * 1e-3) / 1e9 / hbm, 4),
        "gelem_s": round(N / (ms4 / 4 * 1e-3) / 1e9, 2)}

    def graph_ms(fn, reps=10):
        g = a.capture(fn)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        e0, e1 = _events(torch)
        e0.record()
        for _ in range(reps):
            g.replay()
        e1.record()
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps
    rec("ragged_insert_csr_graph", graph_ms(lambda: (a.shrink(0, release=False), a.insert_csr(src, off))),
        8 * N, N, {"note": "reset + insert captured once, replayed (device time)"})

    def reset_dup():
        a.shrink(0, release=False)
        a.insert_csr(src, off)
    rec("ragged_duplicate", best(lambda: (a.insert_duplicate(), a.flush()), reset_dup), 8 * N, N)
    exp = torch.cat([torch.cat([src[int(off[s]):int(off[s + 1])]] * 2) for s in range(S)])
    got = a.flatten_device()
    out["ragged_contents_ok"] = bool(torch.equal(got, exp))
    rec("ragged_flatten", best(lambda: a.flatten_device(out=got), lambda: None), 16 * N, 2 * N)
    rec("ragged_rw_per_shard", best(lambda: a.rw_add(1), lambda: None), 16 * N, 2 * N)
    out["ragged_rw_contents_ok"] = bool(torch.equal(a.flatten_device(out=got), exp + 5))
    a.close()
    del a, exp, got, src
    torch.cuda.empty_cache()
    _between_legs(gg)
    # paper Alg. 1 with per-lane counts
    for K in (8, 1):
        L = N // max(1, K // 2)                      # expected appended elements ~ N (K = 8) / N / 2 (K = 1)
        lo = np.arange(S + 1, dtype=np.uint64) * np.uint64(L // S)
        g = torch.Generator(device=device).manual_seed(K)
        cnt = torch.randint(0, K + 1, (L,), dtype=torch.int32, device=device, generator=g)
        vals = torch.arange(L * K, dtype=torch.int32, device=device)
        tot = int(cnt.sum())
        b = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
        b.insert_lanes(vals, cnt, lo, K, commit=False)
        ms = best(lambda: b.insert_lanes(vals, cnt, lo, K, commit=False), lambda: b.shrink(0, release=False))
        layout = 4 * L + 4 * L * K + 4 * tot
        useful = 4 * L + 8 * tot
        rec(f"lanes_K{K}", ms, layout, tot,
            {"lanes": L, "appended": tot, "algorithmic_bytes": layout, "useful_bytes": useful,
             "useful_frac": round(useful / (ms * 1e-3) / 1e9 / hbm, 4),
             "kernels": ("k_lanes_bulk (one pass: chunk count sums, decoupled look-back per LFVector, value tiles "
                         "streamed by TMA bulk copies into a 2-stage shared-memory ring)" if K == 8 else
                         "k_lanes_chunk (one pass: chunk count sums, decoupled look-back per LFVector, "
                         "register-resident tile walk)")})
        b.commit()
        mask = torch.arange(K, device=device)[None, :] < cnt[:, None]
        comp = vals.view(-1, K)[mask]
        out[f"lanes_K{K}"]["contents_ok"] = bool(torch.equal(b.flatten_device(), comp))
        # 4 back-to-back calls between two events: each plans on the previous
        # calls' upper bounds instead of waiting for their sizes (chained)
        ms4 = best(lambda: [b.insert_lanes(vals, cnt, lo, K, commit=False) for _ in range(4)],
                   lambda: b.shrink(0, release=False), reps=3) / 4
        b.commit()
        ends = torch.cumsum(cnt.to(torch.int64), 0)
        bnd = [0] + [int(ends[int(x) - 1]) for x in lo[1:]]
        exp = torch.cat([comp[bnd[s]:bnd[s + 1]].repeat(4) for s in range(S)])
        out[f"lanes_K{K}"]["chained"] = {
            "calls": 4, "ms_per_call": round(ms4, 4), "frac": round(layout / (ms4 * 1e-3) / 1e9 / hbm, 4),
            "gelem_s": round(tot / (ms4 * 1e-3) / 1e9, 2),
            "contents_ok": bool(torch.equal(b.flatten_device(), exp))}
        del comp, exp
        b.close()
        del b, vals, cnt, mask
        torch.cuda.empty_cache()
        _between_legs(gg)
    # push_if (device push_back API)
    vals = torch.arange(N, dtype=torch.int32, device=device)
    g = torch.Generator(device=device).manual_seed(7)
    pred = (torch.rand(N, device=device, generator=g) < 0.5).to(torch.uint8)
    tot = int(pred.sum())
    for mode in ("block", "warp"):
        c = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
        c.push_if(vals, pred, mode=mode, commit=False)
        ms = best(lambda: c.push_if(vals, pred, mode=mode, commit=False), lambda: c.shrink(0, release=False))
        rec(f"push_if_{mode}", ms, 5 * N + 4 * tot, tot,
            {"candidates": N, "appended": tot, "kernel": f"k_push_if ({mode}_push_back_staged, 8 rounds per thread)"})
        c.commit()
        kept = vals[pred.bool()]
        out[f"push_if_{mode}"]["multiset_ok"] = bool(torch.equal(torch.sort(c.flatten_device())[0], kept))
        # 4 back-to-back calls between two events (chained: each plans on the
        # previous calls' upper bounds instead of waiting for their readback)
        ms4 = best(lambda: [c.push_if(vals, pred, mode=mode, commit=False) for _ in range(4)],
                   lambda: c.shrink(0, release=False), reps=3) / 4
        c.commit()
        out[f"push_if_{mode}"]["chained"] = {
            "calls": 4, "ms_per_call": round(ms4, 4),
            "frac": round((5 * N + 4 * tot) / (ms4 * 1e-3) / 1e9 / hbm, 4),
            "multiset_ok": bool(torch.equal(torch.sort(c.flatten_device())[0], torch.sort(kept.repeat(4))[0]))}
        c.close()
        del c
    del vals, pred
    torch.cuda.empty_cache()
    return out


def full_schedule_baselines(gg, torch, device, step, args):
    """The whole config-2 schedule (2^20 -> 2^30 by doubling: grow, then append
    a copy of the current contents) on the static array (capacity 2^30
    allocated up front), the host-resized doubling array and the memMap
    array, insert_batch (one reservation + vectorised copy, the reference's
    semantics and the baselines' fastest), CUDA events over
    the 10 rounds; next to the GGArray's eager step (same schedule + reset)."""
    out = {}
    n0, final = N0, N0 << ROUNDS

    def schedule(arr, grow):
        n = n0
        e0, e1 = _events(torch)
        torch.cuda.synchronize()
        e0.record()
        for _ in range(ROUNDS):
            grow(arr, 2 * n)
            arr.insert_batch(arr.view()[:n])
            n *= 2
        e1.record()
        torch.cuda.synchronize()
        assert arr.size == final
        return e0.elapsed_time(e1)

    src = torch.arange(n0, dtype=torch.int32, device=device)
    for name, make, grow in [
            ("static_batch", lambda: gg.StaticArray(final, dtype=np.int32, device=device), lambda a, m: None),
            ("doubling_batch", lambda: gg.DoublingArray(n0, dtype=np.int32, device=device), lambda a, m: a.resize(m)),
            ("memmap_batch", lambda: gg.ChunkTableArray(dtype=np.int32, device=device), lambda a, m: a.resize(m))]:
        try:
            ts = []
            for _ in range(2):
                a = make()
                grow(a, n0)
                a.insert_batch(src)
                ts.append(schedule(a, grow))
                del a
                torch.cuda.empty_cache()
            out[name] = {"ms": round(min(ts), 3), "gelem_s": round((final - n0) / min(ts) / 1e6, 2)}
        except Exception as exc:
            out[name] = {"error": repr(exc)[:200]}
    ins = (sum(step.dup_ms) + sum(step.grow_ms)) / args.steps
    out["ggarray512_eager"] = {"ms": round(ins, 3), "gelem_s": round((final - n0) / ins / 1e6, 2),
                               "note": "grow + duplicate-insert phases of the eager steps (events)"}
    return out


def phased_leg(args, gg, torch, device):
    """Config 4: 100 rounds; each draws a total size uniform in [0, 2] x the
    base size (2^26), spread evenly over 512 LFVectors, and inserts or shrinks
    to it; footprint sampled after every round.  Shrink has no reference
    semantics (parity unpinned).  Three release policies of shrink: 2.0 (the
    default: unmap emptied chunks only while more than 2x the needed bytes are
    mapped), True (unmap every emptied chunk) and False (cache them all)."""
    n0 = 1 << 26
    cap_elems = 1 << 28
    src = torch.arange(cap_elems, dtype=torch.int32, device=device)

    def run(release):
        rng = np.random.default_rng(0)
        a = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
        a.insert_csr(src[:n0], split_off(n0))
        n = n0
        cap_ratio, map_ratio, moved = [], [], 0
        sl0 = a.slab_stats()
        torch.cuda.synchronize()
        e0, e1 = _events(torch)
        e0.record()
        for _ in range(100):
            target = int(min(cap_elems, round(rng.uniform(0, 2) * n0)))
            q, r = divmod(target, S)
            new = np.full(S, q, np.int64)
            new[:r] += 1
            cur = a._host()["sizes"].astype(np.int64)
            if target >= n:
                delta = new - cur
                off = np.concatenate([[0], np.cumsum(delta)]).astype(np.uint64)
                a.insert_csr(src[:int(off[-1])], off)
                moved += int(off[-1])
            else:
                a.shrink(new, release=release)
            n = target
            ms = a.memory_stats()
            if target >= n0 // 8:          # ratios of near-empty arrays are dominated by S*fb
                cap_ratio.append(ms["capacity_bytes"] / ms["needed_bytes"])
                map_ratio.append(ms["mapped_bytes"] / ms["needed_bytes"])
        e1.record()
        torch.cuda.synchronize()
        ms_tot = e0.elapsed_time(e1)
        sl = a.slab_stats()
        a.close()
        return {"ms": round(ms_tot, 3), "inserted_elements": moved,
                "capacity_over_needed_max": round(max(cap_ratio), 4),
                "capacity_over_needed_mean": round(float(np.mean(cap_ratio)), 4),
                "mapped_over_needed_max": round(max(map_ratio), 4),
                "mapped_over_needed_mean": round(float(np.mean(map_ratio)), 4),
                "mapped_over_needed_final": round(map_ratio[-1], 4),
                "slab": {"chunks_mapped": sl["chunks_mapped"] - sl0["chunks_mapped"],
                         "chunks_unmapped": sl["chunks_unmapped"] - sl0["chunks_unmapped"],
                         "map_ms": round((sl["map_ns"] - sl0["map_ns"]) / 1e6, 3),
                         "unmap_ms": round((sl["unmap_ns"] - sl0["unmap_ns"]) / 1e6, 3)}}

    out = {"rounds": 100, "seed": 0, "start_elements": n0, "max_elements": cap_elems,
           "ratios_over": "rounds with total >= base/8"}
    # the default policy three times, the median run reported: the driver's
    # map / unmap cost can spike for ~0.2 s while it is still releasing an
    # earlier process's or leg's memory (tools/phased_order_probe.py: 130 ms
    # then 28-30 ms for the same run in one process)
    runs = sorted((run(2.0) for _ in range(3)), key=lambda r: r["ms"])
    out.update(runs[1])
    out["default_policy_runs_ms"] = [r["ms"] for r in runs]
    out["release_all_policy"] = run(True)
    out["cached_policy"] = run(False)
    out["note"] = ("capacity = allocated buckets (reference semantics, <= 2x + fb per shard); "
                   "mapped = physical slab chunks; default policy unmaps emptied chunks only "
                   "down to 2x needed, release_all unmaps every emptied chunk, cached keeps "
                   "them; map/unmap driver cost (incl. page scrubbing) is inside ms")
    del src
    torch.cuda.empty_cache()
    return out


def config1_leg(args, gg, torch, device, with_cpu):
    """Config 1 (BASELINE configs[0], the reference's CPU-runnable case): 512
    LFVectors, one batch insert of 2^20 int32 split like split_batches, one +1
    pass, flatten.  Latency-bound on a B200 (8 MiB); reported as time per
    sequence through the reference-style API (numpy batches in, numpy out:
    H2D + kernels + D2H, wall clock) and device-resident (CUDA events), next
    to the oracle port on the CPU."""
    vals = np.arange(1 << 20, dtype=np.int32)
    batches = gg.split_batches(vals, S)
    dvals = torch.from_numpy(vals).to(device)
    offs = split_off(1 << 20)

    def host_api():
        a = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
        a.insert_parallel(batches)
        a.rw_add(1)
        return a.flatten()

    ref = vals + 1
    assert host_api().tobytes() == ref.tobytes()
    ts = []
    for _ in range(15):
        t0 = time.perf_counter()
        host_api()
        ts.append(time.perf_counter() - t0)
    a = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
    flat = torch.empty(1 << 20, dtype=torch.int32, device=device)

    def dev_seq():
        a.shrink(0, release=False)
        a.insert_csr(dvals, offs)
        a.rw_add(1)
        a.flatten_device(out=flat)

    dev_seq()
    dev_ms = _time(torch, dev_seq, reps=20)
    assert torch.equal(flat.cpu(), torch.from_numpy(ref))
    res = {"elements": 1 << 20, "host_api_ms": round(1e3 * float(np.median(ts)), 3),
           "device_resident_us": round(1e3 * dev_ms, 2),
           "host_api": "GrowableArray(512) + insert_parallel(split_batches(numpy)) + rw_add(1) + "
                       "flatten() -> numpy, median of 15 (includes array construction)",
           "device_resident": "shrink(0) + insert_csr(device batch) + rw_add(1) + flatten_device, "
                              "CUDA events, mean of 20"}
    if with_cpu:
        G = load_reference()
        if G is not None:
            # the reference itself (baseline/_ref): GrowableArray + insert_parallel +
            # for_each_shard(v += 1) + flatten, one worker (its fastest at this size)
            tr = []
            for _ in range(5):
                t0 = time.perf_counter()
                r = G.GrowableArray(S, FB, dtype=np.int32)
                r.insert_parallel(G.split_batches(vals, S), workers=1)
                r.for_each_shard(lambda v: np.add(v, 1, out=v))
                got = r.flatten()
                tr.append(time.perf_counter() - t0)
            assert got.tobytes() == ref.tobytes()
            res["cpu_reference_ms"] = round(1e3 * min(tr), 3)
            res["cpu_reference"] = "growarray (baseline/_ref), same sequence, workers=1, best of 5"
        from oracle import ggoracle as O
        tc = []
        for _ in range(5):
            t0 = time.perf_counter()
            o = O.OracleGGArray(S, FB, dtype=np.int32)
            o.insert_parallel(O.split_batches(vals, S))
            o.rw_add(1)
            o.flatten()
            tc.append(time.perf_counter() - t0)
        res["cpu_port_ms"] = round(1e3 * min(tc), 3)
    return res


def config5_leg(args, gg, torch, device, hbm):
    """Config 5's per-GPU part at BASELINE's ~2^34: 512 LFVectors grown by
    doubling from 2^20 to 2^34 int32 on this GPU (64 GiB live, 128 GiB
    capacity), then flattened in 8 GiB slices (flatten_range) into one staging
    buffer -- an out-of-place flatten of 2^34 does not fit next to the array
    in 180 GB (SURVEY 8e caveat), a streamed one does.  Contents checked in
    full against the closed form of the schedule.  Falls back to 2^33 if the
    GPU cannot hold 2^34 next to the rest of the bench."""
    out = {"device_free_gib_at_entry": round(torch.cuda.mem_get_info(device)[0] / 2**30, 1)}
    # the process slab cache may still hold earlier legs' slabs: hand them
    # back to the driver first (2^34 needs 128 GiB next to the rest)
    gg.pool_trim(device.index)
    torch.cuda.empty_cache()
    out["device_free_gib_after_trim"] = round(torch.cuda.mem_get_info(device)[0] / 2**30, 1)
    for rounds in (14, 13):
        a = None
        try:
            a = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
            src = torch.arange(N0, dtype=torch.int32, device=device)

            def schedule():
                a.shrink(0, release=False)
                a.insert_csr(src, split_off(N0))
                torch.cuda.synchronize()
                e0, e1 = _events(torch)
                e0.record()
                for _ in range(rounds):
                    a.grow(2 * a.committed_size)
                    a.insert_duplicate()
                e1.record()
                torch.cuda.synchronize()
                return e0.elapsed_time(e1)

            cold_ms = schedule()          # first growth maps the slab chunks (driver time)
            sl = a.slab_stats()
            grow_ms = schedule()          # chunks cached in place: the copy work alone
            n = a.committed_size
            sl_elems = 1 << 31
            stage = torch.empty(min(n, sl_elems), dtype=torch.int32, device=device)

            def streamed_flatten():
                for lo in range(0, n, sl_elems):
                    a.flatten_range_to(lo, min(n, lo + sl_elems), stage.data_ptr())

            streamed_flatten()
            fl_ms = _time(torch, streamed_flatten, reps=2)
            per, base = (N0 // S) << rounds, N0 // S
            ok = True
            chunk = 1 << 28
            for c in range(0, n, chunk):
                m = min(chunk, n - c)
                a.flatten_range_to(c, c + m, stage.data_ptr())
                g = torch.arange(c, c + m, dtype=torch.int64, device=device)
                ok &= bool(torch.equal(stage[:m].to(torch.int64), (g // per) * base + g % base))
                del g
            mem = a.memory_stats()
            moved = n - N0
            out.update({"elements": n, "rounds": rounds, "grow_insert_ms": round(grow_ms, 3),
                        "first_growth_ms_incl_mapping": round(cold_ms, 3),
                        "first_growth_map_ms": round(sl["map_ns"] / 1e6, 3),
                        "chunks_mapped": sl["chunks_mapped"],
                        "insert_gelem_s": round(moved / (grow_ms * 1e-3) / 1e9, 2),
                        "insert_frac": round(8 * moved / (grow_ms * 1e-3) / 1e9 / hbm, 4),
                        "flatten_streamed_ms": round(fl_ms, 3), "flatten_slice_elems": sl_elems,
                        "flatten_gbs": round(8 * n / fl_ms / 1e6, 1),
                        "flatten_frac": round(8 * n / fl_ms / 1e6 / hbm, 4), "contents_ok": ok,
                        "capacity_over_needed": round(mem["capacity_over_needed"], 6),
                        "mapped_over_needed": round(mem["mapped_over_needed"], 6),
                        "mapped_gib": round(mem["mapped_bytes"] / 2**30, 2)})
            a.close()
            del stage, a
            gg.pool_trim(device.index)     # 128 GiB back to the driver before the next legs
            torch.cuda.empty_cache()
            return out
        except Exception as exc:                      # report, never lose the bench line
            out[f"error_2p{20 + rounds}"] = repr(exc)[:300]
            if a is not None:
                a.close()
            del a
            gg.pool_trim(device.index)
            torch.cuda.empty_cache()
    return out


def split_off(n):
    return np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(-(-n // S)), np.uint64(n))


def e2e_leg(args, gg, torch, device, world, dist):
    """The same schedule through the public API with HOST input: a fresh pinned
    host batch is copied H2D inside the timed region every step, and the
    per-shard sizes are read back D2H at its end."""
    host = torch.arange(N0, dtype=torch.int32).pin_memory()
    arr = gg.GrowableArray(S, FB, dtype=np.int32, device=device)
    offs = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(N0 // S), N0)
    res = torch.empty(S, dtype=torch.int64).pin_memory()

    def one():
        arr.shrink(0, release=False)
        arr.insert_csr(host.to(device, non_blocking=True), offs)
        for _ in range(ROUNDS):
            arr.grow(2 * arr.committed_size)
            arr.insert_duplicate()
        return arr

    for _ in range(2):
        one()
    torch.cuda.synchronize()
    if dist:
        dist.barrier()
    k = max(2, args.steps)
    pre_d = torch.empty(S + 1, dtype=torch.int64, device=device)
    pre_h = torch.empty(S + 1, dtype=torch.int64).pin_memory()

    def trial():
        t0 = time.perf_counter()
        for _ in range(k):
            one()
            pre_h.copy_(arr.prefix_device(out=pre_d), non_blocking=True)   # D2H of the step's result
            torch.cuda.current_stream().synchronize()
            assert int(pre_h[-1]) == 1 << 30
        return time.perf_counter() - t0

    # pipelined: step j+1's batch is copied H2D on a copy stream (double buffer)
    # while step j's doubling rounds run; every step still copies its own
    # batch inside the timed region and reads its result back before the next
    cs = torch.cuda.Stream(device)
    bufs = [torch.empty(N0, dtype=torch.int32, device=device) for _ in range(2)]
    ready = [torch.cuda.Event() for _ in range(2)]

    def h2d(j):
        with torch.cuda.stream(cs):
            bufs[j % 2].copy_(host, non_blocking=True)   # buf last read by step j-2 (synced)
            ready[j % 2].record(cs)

    def ptrial():
        t0 = time.perf_counter()
        h2d(0)
        cur = torch.cuda.current_stream()
        for j in range(k):
            cur.wait_event(ready[j % 2])
            arr.shrink(0, release=False)
            arr.insert_csr(bufs[j % 2], offs)
            if j + 1 < k:
                h2d(j + 1)
            for _ in range(ROUNDS):
                arr.grow(2 * arr.committed_size)
                arr.insert_duplicate()
            pre_h.copy_(arr.prefix_device(out=pre_d), non_blocking=True)
            cur.synchronize()
            assert int(pre_h[-1]) == 1 << 30
        return time.perf_counter() - t0

    # one step in flight: step j's result (the committed directory) is copied
    # D2H into its own pinned buffer and checked once step j+1 is enqueued, so
    # the host plans step j+1 while the device runs step j.  Every step still
    # copies its batch H2D and its result D2H inside the timed region.
    consumed = [torch.cuda.Event() for _ in range(2)]
    done = [torch.cuda.Event() for _ in range(2)]
    pre_ds = [torch.empty(S + 1, dtype=torch.int64, device=device) for _ in range(2)]
    pre_hs = [torch.empty(S + 1, dtype=torch.int64).pin_memory() for _ in range(2)]

    def h2d_after(j):
        with torch.cuda.stream(cs):
            if j >= 2:
                cs.wait_event(consumed[j % 2])           # step j-2's insert has read this buffer
            bufs[j % 2].copy_(host, non_blocking=True)
            ready[j % 2].record(cs)

    def atrial():
        t0 = time.perf_counter()
        h2d_after(0)
        cur = torch.cuda.current_stream()
        for j in range(k):
            cur.wait_event(ready[j % 2])
            arr.shrink(0, release=False)
            arr.insert_csr(bufs[j % 2], offs)
            consumed[j % 2].record(cur)
            if j + 1 < k:
                h2d_after(j + 1)
            for _ in range(ROUNDS):
                arr.grow(2 * arr.committed_size)
                arr.insert_duplicate()
            pre_hs[j % 2].copy_(arr.prefix_device(out=pre_ds[j % 2]), non_blocking=True)
            done[j % 2].record(cur)
            if j >= 1:
                done[(j - 1) % 2].synchronize()
                assert int(pre_hs[(j - 1) % 2][-1]) == 1 << 30
        done[(k - 1) % 2].synchronize()
        assert int(pre_hs[(k - 1) % 2][-1]) == 1 << 30
        return time.perf_counter() - t0

    def wall_max(fn):
        sec = sorted(fn() for _ in range(3))[1]        # wall clock: median of 3 trials of K steps
        if dist:
            t = torch.tensor([sec], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item())
        return sec

    ptrial()
    atrial()
    serial_sec = wall_max(trial)
    sync_sec = wall_max(ptrial)
    sec = wall_max(atrial)
    # context for the host-side numbers: this box's pinned H2D bandwidth for the step's batch
    dev_tmp = torch.empty(N0, dtype=torch.int32, device=device)
    h2d = []
    for _ in range(10):
        e0, e1 = _events(torch)
        e0.record()
        dev_tmp.copy_(host, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d.append(e0.elapsed_time(e1))
    del dev_tmp
    out = {"value": round(world * (1 << 30) * k / sec / 1e9, 3), "unit": UNIT,
           "h2d_gbs_of_4mib_batch": round(N0 * 4 / float(np.median(h2d)) / 1e6, 1),
           "wall_ms_per_step": round(sec * 1e3 / k, 4),
           "h2d_bytes_per_step": N0 * 4, "d2h_bytes_per_step": (S + 1) * 8,
           "api": "GrowableArray.insert_csr(host batch) + grow + insert_duplicate + prefix_device "
                  "(committed directory D2H into pinned memory), op by op; the next step's host "
                  "batch is copied H2D on a side stream while this step's rounds run, and each "
                  "step's result is checked on the host once the next step is enqueued (one step "
                  "in flight); the last step's result is synchronised inside the timed region",
           "timing": "wall clock, median of 3 trials of K steps (max over ranks)",
           "prefetch_sync_each_step": {"value": round(world * (1 << 30) * k / sync_sec / 1e9, 3),
                                       "wall_ms_per_step": round(sync_sec * 1e3 / k, 4),
                                       "api": "same with the host waiting for each step's result "
                                              "before enqueuing the next"},
           "serial": {"value": round(world * (1 << 30) * k / serial_sec / 1e9, 3),
                      "wall_ms_per_step": round(serial_sec * 1e3 / k, 4),
                      "api": "same, H2D on the compute stream before each step"}}
    # the same end-to-end step captured once through the public API
    # (GrowableArray.capture_mode + torch.cuda.graph): every replay copies the
    # pinned host batch H2D and the committed directory D2H, then syncs
    try:
        dev_in = torch.empty(N0, dtype=torch.int32, device=device)
        res_h = torch.empty(S + 1, dtype=torch.int64).pin_memory()
        pre_d = torch.empty(S + 1, dtype=torch.int64, device=device)

        def one_graph():
            arr.shrink(0, release=False)
            dev_in.copy_(host, non_blocking=True)
            arr.insert_csr(dev_in, offs)
            for _ in range(ROUNDS):
                arr.grow(2 * arr.committed_size)
                arr.insert_duplicate()
            arr.prefix_device(out=pre_d)
            res_h.copy_(pre_d, non_blocking=True)

        g = arr.capture(one_graph)
        for _ in range(3):
            g.replay()
        torch.cuda.synchronize()
        if dist:
            dist.barrier()
        def gtrial():
            t0 = time.perf_counter()
            for _ in range(k):
                g.replay()
                torch.cuda.current_stream().synchronize()
                assert int(res_h[-1]) == 1 << 30
            return time.perf_counter() - t0

        sec = sorted(gtrial() for _ in range(3))[1]
        if dist:
            t = torch.tensor([sec], dtype=torch.float64, device=device)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            sec = float(t.item())
        out["graph"] = {"value": round(world * (1 << 30) * k / sec / 1e9, 3),
                        "h2d_bytes_per_step": N0 * 4, "d2h_bytes_per_step": (S + 1) * 8,
                        "api": "GrowableArray.capture of the same step (host batch H2D + "
                               "directory D2H + sync in every replay)"}
    except Exception as exc:
        out["graph"] = {"error": repr(exc)[:300]}
    return out


# --------------------------------------------------------------------------- CPU legs
REF_DIR = os.path.join(ROOT, "baseline", "_ref")


def load_reference():
    """The UNMODIFIED reference package ``growarray``, pip-installed into
    baseline/_ref (git-ignored; it travels to the GPU box with the snapshot),
    or None when it is absent."""
    if not os.path.isfile(os.path.join(REF_DIR, "growarray", "__init__.py")):
        return None
    if REF_DIR not in sys.path:
        sys.path.insert(0, REF_DIR)
    import growarray
    assert os.path.dirname(os.path.abspath(growarray.__file__)) == os.path.join(REF_DIR, "growarray")
    return growarray


def reference_step(G, workers: int, rounds: int = ROUNDS):
    """One config-2 step through growarray's own harness code path
    (bench_cli.py:508-543 with structure=ggarray): from_flat(arange(2^20), 512,
    32, int32) (_build_structure, :239-244), then per round _grow(2n) (:310-314)
    and _insert_duplicate (:298-307: per-shard to_numpy + insert_parallel with
    ``workers`` threads).  Returns the array (2^(20+rounds) elements)."""
    from growarray import bench_cli as B
    cfg = B.BenchConfig(structure="ggarray", shards=S, first_bucket=FB, workers=workers,
                        initial_size=N0, iterations=rounds)
    store = B._build_structure(cfg, np.arange(N0, dtype=B.BENCH_DTYPE), N0 << rounds)
    for _ in range(rounds):
        B._grow(store, 2 * B._committed_size(store))
        B._insert_duplicate(store, cfg)
    return store


def _check_reference_state(store, rounds: int = ROUNDS) -> None:
    """Sizes / capacity and sampled contents of the reference's end state
    against the closed form of the schedule (element g = (g // per) * 2048 +
    g % 2048)."""
    n = N0 << rounds
    assert store.committed_size == n and store.total_size == n
    per, base = (N0 // S) << rounds, N0 // S
    for g in (0, 1, base - 1, base, per - 1, per, n // 2 + 12345, n - 1):
        assert int(store.get_global(g)) == (g // per) * base + g % base, g


def _time_reference_steps(G, steps: int, workers: int, rounds: int = ROUNDS):
    """Wall time of each step (array construction included); the previous
    step's array is torn down outside the timed window."""
    import gc
    secs = []
    for _ in range(steps):
        gc.collect()
        t0 = time.perf_counter()
        store = reference_step(G, workers, rounds)
        secs.append(time.perf_counter() - t0)
        _check_reference_state(store, rounds)
        del store
    gc.collect()
    return secs


def _port_steps(steps: int, cores: int, rounds: int):
    from oracle import ggoracle as O
    secs = []
    for _ in range(steps):
        t0 = time.perf_counter()
        O.doubling_schedule_cpu(N0, rounds, S, FB, np.int32, cores)
        secs.append(time.perf_counter() - t0)
    return secs


def cpu_baseline(args):
    """The reference's own CPU path (growarray from baseline/_ref) on this
    host's cores, on the full config-2 step (2^20 -> 2^30); a bounded sample
    of 2 timed steps after one warm-up (~10-30 s).  Without baseline/_ref:
    the oracle port (kind "port")."""
    cores = len(os.sched_getaffinity(0))
    G = load_reference()
    if G is not None:
        _time_reference_steps(G, 1, cores)
        secs = _time_reference_steps(G, 2, cores)
        v = 2 * (1 << 30) / sum(secs) / 1e9
        return {"value": round(v, 5), "unit": UNIT, "cores": cores, "kind": "reference",
                "sample": f"growarray (unmodified, baseline/_ref) bench_cli grow-insert-rw path, "
                          f"structure=ggarray: from_flat(arange(2^20), 512, 32, int32) + 10 x "
                          f"(grow(2n) + per-shard to_numpy + insert_parallel(workers={cores})) "
                          f"-> 2^30, 2 steps after 1 warm-up, wall clock",
                "step_s": [round(x, 3) for x in secs]}
    rounds = args.cpu_rounds
    secs = _port_steps(2, cores, rounds)
    return {"value": round(2 * (1 << (20 + rounds)) / sum(secs) / 1e9, 5), "unit": UNIT, "cores": cores,
            "kind": "port",
            "sample": f"baseline/_ref absent: oracle.ggoracle doubling_schedule_cpu S=512 int32 "
                      f"2^20 -> 2^{20 + rounds}, 2 steps"}


def run_reference(args, rank, world):
    """bench.py --impl reference: the reference's CPU implementation of the
    path on this host's cores, same workload, metric and config as the GPU arm
    (one config-2 step = 2^30 elements inserted).  Rank 0 alone runs."""
    if rank != 0:
        return None
    cores = len(os.sched_getaffinity(0))
    G = load_reference()
    if G is not None:
        rounds = args.ref_rounds                      # tests shorten the schedule; default = config 2
        _time_reference_steps(G, args.warmup, cores, rounds)
        secs = _time_reference_steps(G, args.steps, cores, rounds)
        per_step = 1 << (20 + rounds)
        kind = "reference"
        sample = (f"growarray (unmodified, pip-installed into baseline/_ref) through its bench_cli "
                  f"grow-insert-rw code path (structure=ggarray, workers={cores}): from_flat(arange(2^20), "
                  f"512, 32, int32) + 10 x (grow(2n) + per-shard to_numpy + insert_parallel) -> 2^30 per "
                  f"step, end state checked against the closed form")
        cfg_extra = {} if rounds == ROUNDS else {"rounds": rounds, "final_elements_per_gpu": per_step}
    else:
        rounds = args.cpu_rounds
        _port_steps(min(args.warmup, 1), cores, rounds)
        secs = _port_steps(args.steps, cores, rounds)
        per_step = 1 << (20 + rounds)
        kind = "port"
        sample = f"baseline/_ref absent: oracle port S=512 int32 2^20 -> 2^{20 + rounds} per step"
        cfg_extra = {"cpu_sample_final_elements": per_step}
    sec = sum(secs)
    v = args.steps * per_step / sec / 1e9
    return {"metric": METRIC, "value": round(v, 5), "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3 / args.steps, 2),
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "int32",
            "data": "synthetic (np.arange tags, as bench_cli.py)", "impl": "reference",
            "config": {**config_dict(world), **cfg_extra},
            "cpu_baseline": {"value": round(v, 5), "unit": UNIT, "cores": cores, "kind": kind,
                             "sample": sample, "workers": cores, "step_s": [round(x, 3) for x in secs]},
            "e2e": {"value": round(v, 5), "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=10)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ggarray", choices=["ggarray", "reference"])
    ap.add_argument("--rw-passes", type=int, default=100)
    ap.add_argument("--cpu-rounds", type=int, default=7, help="oracle-port fallback sample (no baseline/_ref)")
    ap.add_argument("--ref-rounds", type=int, default=ROUNDS, help="reference arm schedule (tests only)")
    ap.add_argument("--quick", action="store_true", help="headline only")
    ap.add_argument("--no-cpu", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    import gc
    gc.collect()
    gc.disable()      # arrays hold no reference cycles; collections happen between legs only
    if args.impl == "reference":
        out = run_reference(args, rank, world)
        if out is not None:
            print(json.dumps(out), flush=True)
        return
    if os.environ.get("GG_BENCH_SAME_GPU") == "1":
        # test hook: run the N > 1 code path with every rank on GPU 0 (gloo
        # control plane; NCCL refuses two ranks on one GPU)
        local_rank = 0
    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        if os.environ.get("GG_BENCH_SAME_GPU") == "1":
            dist.init_process_group("gloo")
        else:
            dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = run_device(args, rank, world, local_rank)
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
