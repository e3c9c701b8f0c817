"""Launch every gg:: kernel the library has, leg by leg, for one ncu metrics
pass (tools/profile_r02.sh) that records per launch: duration, DRAM bytes read
+ written, L2 atomic / reduction requests, grid / block / registers.

Legs are separated by ``torch.cuda._sleep`` markers (torch's ``spin_kernel``,
a name no library kernel has); ``gpurun_out/prof_all_legs.json`` lists the
legs in order with their algorithmic bytes (the bytes the operation must move:
8 B per copied int32 element = read + write), so
tools/summarize_all.py can pair each leg's launches with its label.  Only the
region inside the NVTX range "profiled" is captured.
"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import paper_2209_00103_b200 as gg

S, FB, E = 512, 32, 4
dev = torch.device("cuda", 0)
torch.cuda.set_device(dev)
OUT = os.environ.get("PROF_OUT", "gpurun_out")
os.makedirs(OUT, exist_ok=True)
legs = []


def leg(label, algo_bytes, elems, dominant, note=""):
    """Start a leg: marker kernel, then the caller launches the leg's ops."""
    torch.cuda.synchronize()
    torch.cuda._sleep(100)
    legs.append({"label": label, "algorithmic_bytes": int(algo_bytes), "elements": int(elems),
                 "dominant": dominant, "note": note})


# ---------------------------------------------------------------- setup (not profiled)
a = gg.GrowableArray.from_flat(torch.arange(1 << 20, dtype=torch.int32, device=dev), S, FB)
for _ in range(9):
    a.grow(2 * a.committed_size)
    a.insert_duplicate()
n29 = a.committed_size                                            # 2^29
N28 = 1 << 28
src28 = torch.arange(N28, dtype=torch.int32, device=dev)
uni_off = np.minimum(np.arange(S + 1, dtype=np.uint64) * np.uint64(N28 // S), N28)
rng = np.random.default_rng(0)
counts = rng.integers(0, 2 * (N28 // S) + 1, S).astype(np.int64)
counts = (counts * (N28 / counts.sum())).astype(np.int64)
counts[-1] += N28 - counts.sum()
rag_off = np.concatenate([[0], np.cumsum(counts)]).astype(np.uint64)
b = gg.GrowableArray(S, FB, dtype=np.int32)
b.insert_csr(src28, uni_off)                                      # map its slabs before the region
b.shrink(0, release=False)
r = gg.GrowableArray(S, FB, dtype=np.int32)
r.insert_csr(src28, rag_off)
r.insert_duplicate()
r.shrink(0, release=False)
NI = 1 << 24
idx = torch.randint(0, 1 << 30, (NI,), dtype=torch.int64, device=dev)
vals_i = torch.arange(NI, dtype=torch.int32, device=dev)
lanes_in = {}
for K in (8, 1):
    Ln = N28 // max(1, K // 2)
    g = torch.Generator(device=dev).manual_seed(K)
    cnt = torch.randint(0, K + 1, (Ln,), dtype=torch.int32, device=dev, generator=g)
    lanes_in[K] = (torch.arange(Ln * K, dtype=torch.int32, device=dev), cnt,
                   np.arange(S + 1, dtype=np.uint64) * np.uint64(Ln // S), int(cnt.sum()))
lanes_arr = gg.GrowableArray(S, FB, dtype=np.int32)
v8, c8, lo8, _ = lanes_in[8]
lanes_arr.insert_lanes(v8, c8, lo8, 8, commit=False)
lanes_arr.shrink(0, release=False)
pred = (torch.rand(N28, generator=torch.Generator(device=dev).manual_seed(7), device=dev) < 0.5).to(torch.uint8)
kept = int(pred.sum())
pa = gg.GrowableArray(S, FB, dtype=np.int32)
pa.push_if(src28, pred, mode="block", commit=False)
pa.shrink(0, release=False)
st = gg.StaticArray(1 << 30, dtype=np.int32)
st_src = torch.arange(1 << 29, dtype=torch.int32, device=dev)
dbl = gg.DoublingArray(1 << 29, dtype=np.int32)
ct = gg.ChunkTableArray(dtype=np.int32)
ct.resize(1 << 29)
big = gg.GrowableArray(8192, FB, dtype=np.int32)                 # S > 4096: store-only metadata kernels
big.insert_csr(src28, np.minimum(np.arange(8193, dtype=np.uint64) * np.uint64(N28 // 8192), N28))
big.shrink(0, release=False)
calls = []


def hook(n):                                                     # host allocator hook -> exact paths
    calls.append(n)


hk = gg.GrowableArray(64, FB, dtype=np.int32, allocator=hook)
small = torch.arange(1 << 16, dtype=torch.int32, device=dev)
torch.cuda.synchronize()

# ---------------------------------------------------------------- profiled legs
torch.cuda.nvtx.range_push("profiled")
leg("grow 2^29 -> 2^30, uniform (k_grow / k_meta_grow, deferred pass flushed)", 0, 0, "k_grow|k_meta_grow",
    "metadata only: S x buckets flags")
a.grow(2 * n29)
a.flush()
leg("duplicate insert 2^29 -> 2^30 (uniform directory)", 8 * n29, n29, "k_walk")
a.insert_duplicate()
n30 = 2 * n29
leg("r/w +1 per LFVector, 2^30 (rw_b)", 8 * n30, n30, "k_walk")
a.rw_add(1)
leg("r/w +1 global index space, 2^30 (rw_g)", 8 * n30, n30, "k_rw_global")
a.rw_add(1, mode="global")
flat = torch.empty(n30, dtype=torch.int32, device=dev)
leg("flatten 2^30", 8 * n30, n30, "k_walk")
a.flatten_device(out=flat)
leg("flatten_range 2^28 from the middle", 8 * N28, N28, "k_walk")
a.flatten_range_to(n29 - N28 // 2, n29 + N28 // 2, flat.data_ptr())
outi = torch.empty(NI, dtype=torch.int32, device=dev)
leg("get_many 2^24 random global indices", NI * (8 + 4 + 32), NI, "k_gather",
    "index 8 B + value 4 B written + one 32 B sector read per random element")
gvals = a.get_many(idx)
leg("set_many 2^24 random global indices", NI * (8 + 4 + 32), NI, "k_gather",
    "index 8 B + value 4 B read + one 32 B sector written per random element")
a.set_many(idx, vals_i)
leg("shrink uniform 2^30 -> 2^29 (k_shrink_uniform)", 0, 0, "k_shrink_uniform", "metadata only")
a.shrink(n29 // S, release=False)
leg("shrink ragged (k_shrink)", 0, 0, "k_shrink", "metadata only")
a.shrink(np.arange(S, dtype=np.uint64) * 1024, release=False)
leg("insert CSR 2^28, uniform batches (fused metadata CTA)", 8 * N28, N28, "k_walk")
b.insert_csr(src28, uni_off)
leg("insert CSR 2^28, ragged batches (shard-grid walk)", 8 * N28, N28, "k_walk_shard")
r.insert_csr(src28, rag_off)
r.flush()
leg("duplicate 2^28, ragged (shard-grid walk)", 8 * N28, N28, "k_walk_shard")
r.insert_duplicate()
r.flush()
rflat = torch.empty(2 * N28, dtype=torch.int32, device=dev)
leg("flatten 2^29, ragged (shard-grid walk)", 16 * N28, 2 * N28, "k_walk_shard")
r.flatten_device(out=rflat)
leg("r/w +1 per LFVector 2^29, ragged", 16 * N28, 2 * N28, "k_walk_shard")
r.rw_add(1)
leg("commit without a fused walk (k_commit)", 0, 0, "k_commit", "prefix scan over S")
r.insert_duplicate(commit=False)
r.flush()
r.commit()
for K in (8, 1):
    v, cnt, lo, tot = lanes_in[K]
    Ln = cnt.numel()
    dst = lanes_arr if K == 8 else gg.GrowableArray(S, FB, dtype=np.int32)
    leg(f"insert_lanes K={K} ({Ln} lanes, paper Alg. 1)", 4 * Ln + 4 * Ln * K + 4 * tot, tot,
        "k_lanes_chunk", "counts + the [lanes x K] value block + compacted output")
    dst.insert_lanes(v, cnt, lo, K, commit=False)
for mode in ("block", "warp"):
    dst = pa if mode == "block" else gg.GrowableArray(S, FB, dtype=np.int32)
    leg(f"push_if {mode} 2^28 candidates, density 1/2", 5 * N28 + 4 * kept, kept, "k_push_if",
        "values 4 B + predicate 1 B read per candidate + kept values written")
    dst.push_if(src28, pred, mode=mode, commit=False)
leg("uniform insert at S = 8192 (store-only metadata kernel)", 8 * N28, N28, "k_walk|k_meta_uniform")
big.insert_csr(src28, np.minimum(np.arange(8193, dtype=np.uint64) * np.uint64(N28 // 8192), N28))
leg("insert_parallel, host batches 2^16 with an allocator hook (k_reserve / k_planned_meta / k_zero_buckets)",
    8 * (1 << 16), 1 << 16, "k_walk|k_reserve|k_planned_meta")
hk.insert_parallel(gg.split_batches(small.cpu().numpy(), 64))
leg("insert_lanes exact two-pass path (allocator hook: k_lanes_count + k_lanes_insert)",
    4 * 4096 + 4 * 4096 * 4 + 4 * 8192, 8192, "k_lanes_insert")
hk.insert_lanes(torch.arange(4096 * 4, dtype=torch.int32, device=dev),
                torch.full((4096,), 2, dtype=torch.int32, device=dev),
                np.arange(65, dtype=np.uint64) * 64, 4)
leg("size_counter.fetch_add (k_fetch_add)", 0, 0, "k_fetch_add")
hk.shards[3].size_counter.fetch_add(5)
leg("new_bucket (k_new_bucket + k_zero_buckets)", 0, 0, "k_new_bucket")
hk.shards[5].new_bucket(12)
leg("ShardVector.reserve (k_reserve)", 0, 0, "k_reserve|k_grow")
hk.shards[7].reserve(1 << 20)
leg("static insert, one atomicAdd per element, 2^24 (paper 3-B)", 8 * NI, NI, "k_flat_insert")
st.insert_batch(st_src[:NI], algo="atomic")
leg("static insert, one atomicAdd per warp, 2^26", 8 * (1 << 26), 1 << 26, "k_flat_insert")
st.insert_batch(st_src[:1 << 26], algo="warp")
NB = (1 << 29) - NI - (1 << 26)
leg(f"static insert, one atomicAdd per 32 KiB tile, {NB} elements", 8 * NB, NB, "k_flat_insert_block")
st.insert_batch(st_src[:NB], algo="block")
st2 = gg.StaticArray(1 << 30, dtype=np.int32)
leg("static insert_batch (one reservation, k_flat_append), 2^29", 8 * (1 << 29), 1 << 29, "k_flat_append")
st2.insert_batch(st_src)
leg("static r/w +1, 2^29 (k_flat_add)", 8 * (1 << 29), 1 << 29, "k_flat_add")
st2.rw_add(1)
leg("doubling insert_batch 2^29 (k_flat_append)", 8 * (1 << 29), 1 << 29, "k_flat_append")
dbl.insert_batch(st_src)
leg("memMap insert_batch 2^29 (k_flat_append)", 8 * (1 << 29), 1 << 29, "k_flat_append")
ct.insert_batch(st_src)
leg("capture with an odd number of fused walks (k_copy_db restores the buffer parity)", 0, 0, "k_copy_db")
g = b.capture(lambda: b.insert_duplicate())
g.replay()
leg("end", 0, 0, "")
torch.cuda.synchronize()
torch.cuda.nvtx.range_pop()
json.dump(legs, open(os.path.join(OUT, "prof_all_legs.json"), "w"), indent=1)
print("prof_all done:", len(legs) - 1, "legs")
