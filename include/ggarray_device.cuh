/*
 * ggarray_device.cuh -- device-side GGArray API for user kernels (sm_100a).
 *
 * The paper's point (arXiv 2209.00103 Alg. 1/2): threads of a running kernel
 * append to an LFVector, the block computing per-thread offsets with a
 * warp-shuffle / shared-memory scan, reserving with ONE atomicAdd on the
 * LFVector size and allocating the buckets its range touches on the fly (CAS
 * once-flag; the winner allocates, losers wait for publication).  This header
 * exposes exactly that to any kernel:
 *
 *   gg::gg_device_view v = ...;          // from gg_device_view_get() (host)
 *   gg::warp_push_back(v, shard, pred, value);        // one atomicAdd per warp
 *   gg::warp_push_back_n<T, K>(v, shard, count, vals); // per-lane counts, one per warp
 *   gg::warp_push_back_mask<T, K>(v, shard, mask, vals);        // K candidates, bitmask
 *   gg::warp_push_back_staged<T, K>(v, shard, mask, vals, stage); // 16 B stores
 *   gg::block_push_back_mask<BLOCK, T, K>(v, shard, mask, vals, scratch);
 *   gg::block_push_back_staged<BLOCK, T, K>(v, shard, mask, vals, scratch, stage); // 16 B stores
 *   gg::block_push_back<BLOCK>(v, shard, count, vals, scratch);  // one per block
 *
 * Device code cannot map memory, so the host backs the slots a launch may
 * need before it (gg_device_view_get with per-shard worst-case sizes);
 * allocations of unbacked slots fail, set status[shard] |= GG_ENOMEM, and the
 * reservation is kept, like a failing allocator in the reference
 * (bucket_vector.py:194-201).  After the kernel, gg_device_view_sync()
 * refreshes the host's mirrors from the device tables and unmaps the
 * headroom no bucket took.
 *
 * The same structures and allocator back the library's own kernels
 * (paper_2209_00103_b200/csrc/gg_device.cuh), so there is one implementation.
 */
#ifndef GGARRAY_DEVICE_CUH
#define GGARRAY_DEVICE_CUH

#include <cstdint>

namespace gg {

// Device tables of one GGArray (all pointers are device memory).
//
// Bucket storage is a slab per bucket class: class b owns a region of S
// slots of bucket_bytes(b), slot s belonging to shard s, so bucket (s, b)
// lives at cbase[b] + s * bucket_bytes(b) for its whole life (address
// stability, bucket_vector.py:249-255).  Allocation is the CAS once-flag plus
// that address computation -- no device malloc, no bump pointer.  The host
// backs slots with physical memory (CUDA VMM chunks, refcounted by live
// buckets) before any kernel can publish them, and unmaps chunks whose
// buckets were all released by a shrink.
struct gg_device_view {
  uint64_t *size, *cap, *ops, *start, *count, *prefix, *offsets;
  uint32_t *ctl, *flag, *status;
  char **ptr;                 // [S*MB] bucket base pointers (0 = unallocated)
  unsigned long long *pmask;  // [S] published-bucket bitmask per shard
  unsigned long long *amask;  // [S] slots the host has backed; nullptr = every
                              // allocation of the launch was planned (and backed)
  char **cbase;               // [MB] base of class b's slot region
  unsigned long long *misc;   // alloc count, OOM count, launch counters
  uint32_t S, log2fb, MB, esz;
};

constexpr uint32_t kFlagPublished = 2;   // once-flag states: 0 free, 1 allocating, 2 published
constexpr uint32_t kStatusNoMem = 4;     // == GG_ENOMEM

// launch-coordination counters live on their own 128 B lines, away from the
// allocator's bump top (pollers would otherwise contend with its atomics)
enum { MISC_ALLOCS = 1, MISC_OOM = 2,
       MISC_N = 64 };

// bucket_vector.py:48-59: b = hibit(i/fb + 1), off = i - fb*(2^b - 1)
__device__ __forceinline__ void locate(uint64_t i, uint32_t log2fb, uint32_t &b, uint64_t &off) {
  uint64_t q = (i >> log2fb) + 1;
  b = 63u - (uint32_t)__clzll((long long)q);
  off = i - (((1ull << b) - 1ull) << log2fb);
}

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t *p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint64_t ld_acquire64(const uint64_t *p) {
  uint64_t v;
  asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t *p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ uint64_t bucket_bytes(const gg_device_view &t, uint32_t b) {
  return ((1ull << (t.log2fb + b)) * t.esz + 15) & ~15ull;
}
// the fixed slot of bucket (s, b) in class b's slab
__device__ __forceinline__ char *bucket_slot(const gg_device_view &t, uint32_t s, uint32_t b) {
  return t.cbase[b] + (uint64_t)s * bucket_bytes(t, b);
}
// the same address for a bucket the caller knows is published (ensure_buckets
// succeeded for its range): slots never move, so no pointer load is needed --
// only the class base, a read-only (L1-cached) load
__device__ __forceinline__ char *bucket_known(const gg_device_view &t, uint32_t s, uint32_t b) {
  return (char *)__ldg(reinterpret_cast<const unsigned long long *>(t.cbase) + b) + (uint64_t)s * bucket_bytes(t, b);
}

// Paper Alg. 2 (new_bucket): CAS the once-flag; the winner takes the shard's
// slot of class b (if the host backed it) and publishes it with release
// order; losers wait for the publication (or retry after a rollback).
// Returns 1 if this caller allocated, 0 if the bucket was already there, -1 if
// the slot has no physical memory behind it (flag rolled back, like
// bucket_vector.py:196-201).
__device__ inline int alloc_bucket(const gg_device_view &t, uint32_t s, uint32_t b) {
  uint32_t *f = t.flag + (size_t)s * t.MB + b;
  for (;;) {
    uint32_t cur = ld_acquire(f);
    if (cur == kFlagPublished) return 0;
    if (cur == 0 && atomicCAS(f, 0u, 1u) == 0u) break;
    __nanosleep(64);
  }
  if (t.amask && !((t.amask[s] >> b) & 1ull)) {
    atomicAdd(&t.misc[MISC_OOM], 1ull);
    st_release(f, 0);
    return -1;
  }
  t.ptr[(size_t)s * t.MB + b] = bucket_slot(t, s, b);
  atomicAdd((unsigned long long *)&t.cap[s], 1ull << (t.log2fb + b));
  atomicAdd(&t.misc[MISC_ALLOCS], 1ull);
  st_release(f, kFlagPublished);   // orders the pointer (and counters) before the flag
  // release RMW: the pmask bit never becomes visible before the flag
  asm volatile("red.release.gpu.global.or.b64 [%0], %1;" ::"l"(t.pmask + s), "l"(1ull << b) : "memory");
  return 1;
}

// Allocate every bucket covering local indices [start, start + n) of shard s
// (bucket_vector.py:207-214).  Returns false if a bucket could not be had.
__device__ inline bool ensure_buckets(const gg_device_view &t, uint32_t s, uint64_t start,
                                      uint64_t n) {
  if (!n) return true;
  uint32_t b0, b1;
  uint64_t o;
  locate(start, t.log2fb, b0, o);
  locate(start + n - 1, t.log2fb, b1, o);
  bool ok = b1 < t.MB;
  // fast path: one acquire load of the shard's published-bucket mask (a pmask
  // bit is set only after its flag was released as published).  A missing
  // bit proves nothing -- the bucket may be mid-publication -- so the
  // once-flag is the authority below: a bucket another warp is still
  // allocating (flag 1) is waited for, a rolled-back one (no backing) fails
  if (ok) {
    const unsigned long long want = (b1 >= 63 ? ~0ull : ((2ull << b1) - 1ull)) & ~((1ull << b0) - 1ull);
    if ((ld_acquire64(reinterpret_cast<const uint64_t *>(t.pmask + s)) & want) == want) return true;
  }
  for (uint32_t b = b0; ok && b <= b1; ++b)
    if (ld_acquire(t.flag + (size_t)s * t.MB + b) != kFlagPublished && alloc_bucket(t, s, b) < 0) ok = false;
  if (!ok) atomicOr(&t.status[s], kStatusNoMem);
  return ok;
}

// The reservation of one append (insert_index.py:118-143): ONE atomicAdd of
// n on the LFVector size, then the buckets of [start, start + n).  The
// shard's published-bucket mask is loaded BEFORE the atomic so both round
// trips overlap; when it already covers the range (the common case: a bucket
// is published once per doubling) no further load is needed -- a set pmask
// bit can only mean a published bucket, however stale the read.
__device__ inline bool reserve_ensure(const gg_device_view &t, uint32_t s, uint64_t n,
                                      unsigned long long &start) {
  unsigned long long pm;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(pm) : "l"(t.pmask + s) : "memory");
  start = atomicAdd((unsigned long long *)&t.size[s], (unsigned long long)n);
  atomicAdd((unsigned long long *)&t.ops[s], 1ull);
  if (!n) return true;
  uint32_t b0, b1;
  uint64_t o;
  locate(start, t.log2fb, b0, o);
  locate(start + n - 1, t.log2fb, b1, o);
  if (b1 < t.MB) {
    const unsigned long long want = (b1 >= 63 ? ~0ull : ((2ull << b1) - 1ull)) & ~((1ull << b0) - 1ull);
    if ((pm & want) == want) return true;
  }
  return ensure_buckets(t, s, start, n);
}

// Warp-cooperative ensure_buckets: lane k takes buckets b0 + k, b0 + k + 32,
// ... so the (rare) appends that open several buckets allocate them in
// parallel instead of one CAS / publish chain after another.  Called by all 32
// lanes with the same arguments; the result is in every lane.
__device__ inline bool warp_ensure_buckets(const gg_device_view &t, uint32_t s, uint64_t start,
                                           uint64_t n) {
  if (!n) return true;
  const uint32_t lane = threadIdx.x & 31;
  uint32_t b0, b1;
  uint64_t o;
  locate(start, t.log2fb, b0, o);
  locate(start + n - 1, t.log2fb, b1, o);
  bool ok = b1 < t.MB;
  if (ok)
    for (uint32_t b = b0 + lane; b <= b1; b += 32)
      if (ld_acquire(t.flag + (size_t)s * t.MB + b) != kFlagPublished && alloc_bucket(t, s, b) < 0) ok = false;
  ok = __all_sync(0xffffffffu, ok);
  if (!ok && lane == 0) atomicOr(&t.status[s], kStatusNoMem);
  return ok;
}

// reserve_ensure by a whole warp (same arguments in every lane): lane 0 makes
// the reservation, the warp allocates what the published mask does not cover.
// start and the result are returned in every lane.
__device__ inline bool warp_reserve_ensure(const gg_device_view &t, uint32_t s, uint64_t n,
                                           unsigned long long &start) {
  const uint32_t lane = threadIdx.x & 31;
  unsigned long long pm = 0, st = 0;
  if (lane == 0) {
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(pm) : "l"(t.pmask + s) : "memory");
    st = atomicAdd((unsigned long long *)&t.size[s], (unsigned long long)n);
    atomicAdd((unsigned long long *)&t.ops[s], 1ull);
  }
  start = __shfl_sync(0xffffffffu, st, 0);
  pm = __shfl_sync(0xffffffffu, pm, 0);
  if (!n) return true;
  uint32_t b0, b1;
  uint64_t o;
  locate(start, t.log2fb, b0, o);
  locate(start + n - 1, t.log2fb, b1, o);
  if (b1 < t.MB) {
    const unsigned long long want = (b1 >= 63 ? ~0ull : ((2ull << b1) - 1ull)) & ~((1ull << b0) - 1ull);
    if ((pm & want) == want) return true;
  }
  return warp_ensure_buckets(t, s, start, n);
}

// Bucket base of (s, b) read with acquire order: the flag load synchronises
// with the allocator's release, so the pointer read after it is current even
// if another SM allocated the bucket (plain loads could hit a stale L1 line).
// For user kernels that read buckets they did not reserve themselves; the
// append paths above use bucket_known (their reservation already proved the
// bucket published).
__device__ __forceinline__ char *bucket_acquire(const gg_device_view &t, uint32_t s, uint32_t b) {
  if (b >= t.MB || ld_acquire(t.flag + (size_t)s * t.MB + b) != kFlagPublished) return nullptr;
  char *p;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(p) : "l"(t.ptr + (size_t)s * t.MB + b) : "memory");
  return p;
}

// Element store that bypasses L1 (st.global.cg): appended data must survive
// other warps' acquire loads on this SM, which invalidate its L1.
template <typename T>
__device__ __forceinline__ void store_cg(T *p, const T &v) {
  if constexpr (sizeof(T) == 1) { unsigned char x; memcpy(&x, &v, 1); __stcg((unsigned char *)p, x); }
  else if constexpr (sizeof(T) == 2) { unsigned short x; memcpy(&x, &v, 2); __stcg((unsigned short *)p, x); }
  else if constexpr (sizeof(T) == 4) { unsigned int x; memcpy(&x, &v, 4); __stcg((unsigned int *)p, x); }
  else { unsigned long long x; memcpy(&x, &v, 8); __stcg((unsigned long long *)p, x); }
}

// Paper Alg. 1, warp flavour: every lane with `pred` appends `value` to shard s
// (s warp-uniform).  The 0/1 counts are scanned with a ballot (the warp
// shuffle scan of a predicate), the warp reserves with ONE atomicAdd on the
// LFVector size, lane 0 allocates the touched buckets, values land in lane
// order.  Must be called by all 32 lanes.  Returns the lane's local index or
// ~0ull.
template <typename T>
__device__ inline uint64_t warp_push_back(const gg_device_view &t, uint32_t s, bool pred,
                                          const T &value) {
  const unsigned m = __ballot_sync(0xffffffffu, pred);
  if (!m) return ~0ull;
  const uint32_t lane = threadIdx.x & 31, cnt = __popc(m), rank = __popc(m & ((1u << lane) - 1u));
  unsigned long long start = 0;
  if (!warp_reserve_ensure(t, s, cnt, start)) return ~0ull;
  if (!pred) return ~0ull;
  // every bucket of [start, start + cnt) is published (ensure_buckets), so
  // each lane computes its slot address (no pointer load, no shuffle: a
  // full-mask shuffle next to the predicated return can be sunk into a
  // divergent branch by the compiler)
  uint32_t b;
  uint64_t o;
  locate(start + rank, t.log2fb, b, o);
  store_cg(reinterpret_cast<T *>(bucket_known(t, s, b)) + o, value);
  return start + rank;
}

// Paper Alg. 1, warp flavour with per-lane counts: lane j appends vals[0..
// counts_j) (counts_j <= K); a warp shuffle scan gives every lane its offset,
// lane 0 reserves the warp total with ONE atomicAdd and allocates the buckets,
// values land in lane order.  Amortises the reservation over up to 32*K
// values.  Must be called by all 32 lanes; s warp-uniform.
template <typename T, int K>
__device__ inline uint64_t warp_push_back_n(const gg_device_view &t, uint32_t s, uint32_t count,
                                            const T (&vals)[K]) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t x = count;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, x, 31), excl = x - count;
  if (!total) return ~0ull;
  unsigned long long start = 0;
  if (!warp_reserve_ensure(t, s, total, start)) return ~0ull;
  uint32_t cur_b = ~0u;
  char *base = nullptr;
#pragma unroll
  for (int e = 0; e < K; ++e) {
    if ((uint32_t)e < count) {
      uint32_t b;
      uint64_t o;
      locate(start + excl + e, t.log2fb, b, o);
      if (b != cur_b) { base = bucket_known(t, s, b); cur_b = b; }
      store_cg(reinterpret_cast<T *>(base) + o, vals[e]);
    }
  }
  return start + excl;
}

// Paper Alg. 1 with up to K candidate values per lane selected by a bitmask:
// value j of a lane lands at start + excl + popc(mask & ((1 << j) - 1)).  No
// compaction into a dynamically indexed array (which would live in local
// memory): all indexing is static, values stay in registers.  One atomicAdd
// per warp; must be called by all 32 lanes, s warp-uniform.
template <typename T, int K>
__device__ inline uint64_t warp_push_back_mask(const gg_device_view &t, uint32_t s, uint32_t mask,
                                               const T (&vals)[K]) {
  const uint32_t lane = threadIdx.x & 31, count = __popc(mask);
  uint32_t x = count;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, x, 31), excl = x - count;
  if (!total) return ~0ull;
  unsigned long long start = 0;
  if (!warp_reserve_ensure(t, s, total, start)) return ~0ull;
  uint32_t cur_b = ~0u, r = 0;
  char *base = nullptr;
#pragma unroll
  for (int j = 0; j < K; ++j) {
    if ((mask >> j) & 1u) {
      uint32_t b;
      uint64_t o;
      locate(start + excl + r, t.log2fb, b, o);
      if (b != cur_b) { base = bucket_known(t, s, b); cur_b = b; }
      store_cg(reinterpret_cast<T *>(base) + o, vals[j]);
      ++r;
    }
  }
  return start + excl;
}

// Warp flavour of the staged variant: ONE atomicAdd per warp, the warp's run
// staged in its own shared buffer (lane order, shifted congruent with the
// destination mod 16 B) and written as aligned 16 B vector stores through the
// bucket slots -- coalesced, unlike the per-lane element stores of
// warp_push_back_mask.  stage: 32*K + 32/sizeof(T) elements of shared memory,
// 16 B aligned, private to the warp.  Must be called by all 32 lanes; s
// warp-uniform.  Returns the run's start index (or ~0ull).
template <typename T, int K>
__device__ inline uint64_t warp_push_back_staged(const gg_device_view &t, uint32_t s, uint32_t mask,
                                                 const T (&vals)[K], T *stage) {
  static_assert(16 % sizeof(T) == 0, "element size must divide 16 B");
  constexpr uint32_t VE = 16 / sizeof(T);
  const uint32_t lane = threadIdx.x & 31, count = __popc(mask);
  uint32_t x = count;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  const uint32_t total = __shfl_sync(0xffffffffu, x, 31), excl = x - count;
  if (!total) return ~0ull;
  unsigned long long start = 0;
  if (!warp_reserve_ensure(t, s, total, start)) return ~0ull;
  const uint32_t esz_log = sizeof(T) == 1 ? 0 : sizeof(T) == 2 ? 1 : sizeof(T) == 4 ? 2 : 3;
  const bool vec = t.log2fb + esz_log >= 4;               // every bucket is whole 16 B vectors
  const uint32_t shift = vec ? (uint32_t)(start % VE) : 0u;
  uint32_t r = 0;
#pragma unroll
  for (int j = 0; j < K; ++j)
    if ((mask >> j) & 1u) stage[shift + excl + r++] = vals[j];
  __syncwarp();
  if (vec) {
    const uint32_t nv = (shift + total + VE - 1) / VE;
    // the run (warp-uniform) usually lies in ONE bucket: one address
    // computation, each vector an offset from it
    // (4 / 8 B elements; for 1 / 2 B the extra live registers cost more)
    uint32_t bf = 0, bl = 1;
    uint64_t of = 0, ol;
    if (sizeof(T) >= 4) {
      locate(start - shift, t.log2fb, bf, of);
      locate(start + total - 1, t.log2fb, bl, ol);
    }
    T *const rbase = bf == bl ? reinterpret_cast<T *>(bucket_known(t, s, bf)) + of : nullptr;
    for (uint32_t v = lane; v < nv; v += 32) {
      T *dp;
      if (bf == bl) {
        dp = rbase + v * VE;
      } else {
        uint32_t b;
        uint64_t o;
        locate(start - shift + (uint64_t)v * VE, t.log2fb, b, o);
        dp = reinterpret_cast<T *>(bucket_known(t, s, b)) + o;
      }
      const uint32_t k0 = v * VE;
      if (k0 >= shift && k0 + VE <= shift + total) {
        const uint4 q = reinterpret_cast<const uint4 *>(stage)[v];
        asm volatile("st.global.cg.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dp), "r"(q.x), "r"(q.y), "r"(q.z),
                     "r"(q.w) : "memory");
      } else {
        for (uint32_t j = 0; j < VE; ++j)
          if (k0 + j >= shift && k0 + j < shift + total) store_cg(dp + j, stage[k0 + j]);
      }
    }
  } else {
    for (uint32_t k = lane; k < total; k += 32) {
      uint32_t b;
      uint64_t o;
      locate(start + k, t.log2fb, b, o);
      store_cg(reinterpret_cast<T *>(bucket_known(t, s, b)) + o, stage[k]);
    }
  }
  __syncwarp();                                           // the stage is reused by the next call
  return start;
}

// Block flavour of the mask variant: a shared-memory scan of the lanes'
// popcounts, ONE atomicAdd per block, values in thread order.  scratch: 34 u64
// of shared memory; all BLOCK threads must call it.
template <int BLOCK, typename T, int K>
__device__ inline uint64_t block_push_back_mask(const gg_device_view &t, uint32_t s, uint32_t mask,
                                                const T (&vals)[K], unsigned long long *scratch) {
  static_assert(BLOCK % 32 == 0 && BLOCK <= 1024, "BLOCK must be a multiple of 32, <= 1024");
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, count = __popc(mask);
  unsigned long long x = count;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  if (lane == 31) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < BLOCK / 32 ? scratch[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= (uint32_t)d) w += y;
    }
    scratch[lane] = w;
  }
  __syncthreads();
  const unsigned long long excl = x - count + (wid ? scratch[wid - 1] : 0);
  const unsigned long long total = scratch[BLOCK / 32 - 1];
  __syncthreads();
  if (wid == 0 && total) {                 // warp 0 reserves (and allocates in parallel)
    unsigned long long start = 0;
    const bool ok = warp_reserve_ensure(t, s, total, start);
    if (lane == 0) { scratch[32] = start; scratch[33] = ok; }
  } else if (tid == 0) {
    scratch[32] = 0;
    scratch[33] = 1;
  }
  __syncthreads();
  const unsigned long long start = scratch[32];
  const bool ok = scratch[33] != 0;
  __shared__ char *bptr_m[64];
  if (ok && total) {
    uint32_t b0, b1;
    uint64_t o;
    locate(start, t.log2fb, b0, o);
    locate(start + total - 1, t.log2fb, b1, o);
    if (tid <= b1 - b0) bptr_m[b0 + tid] = bucket_known(t, s, b0 + tid);
  }
  __syncthreads();
  if (ok) {
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < K; ++j) {
      if ((mask >> j) & 1u) {
        uint32_t b;
        uint64_t o;
        locate(start + excl + r, t.log2fb, b, o);
        if (bptr_m[b]) store_cg(reinterpret_cast<T *>(bptr_m[b]) + o, vals[j]);
        ++r;
      }
    }
  }
  __syncthreads();
  return start;
}

// Block flavour of the mask variant with the appends leaving as whole
// vectors: after the block scan and the ONE atomicAdd, every thread writes
// its kept values into the shared `stage` (thread order, shifted so that the
// run is congruent with its destination mod 16 B), then the block stores the
// run [start, start + total) with aligned 16 B vector stores through the
// bucket slots (element stores at the run's ends, or everywhere when a
// bucket holds less than 16 B).  stage: BLOCK*K + 32/sizeof(T) elements of
// shared memory, scratch: 34 u64; all BLOCK threads must call it.
template <int BLOCK, typename T, int K>
__device__ inline uint64_t block_push_back_staged(const gg_device_view &t, uint32_t s, uint32_t mask,
                                                  const T (&vals)[K], unsigned long long *scratch, T *stage) {
  static_assert(BLOCK % 32 == 0 && BLOCK <= 1024, "BLOCK must be a multiple of 32, <= 1024");
  static_assert(16 % sizeof(T) == 0, "element size must divide 16 B");
  constexpr uint32_t VE = 16 / sizeof(T);
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, count = __popc(mask);
  uint32_t x = count;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  if (lane == 31) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < BLOCK / 32 ? scratch[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= (uint32_t)d) w += y;
    }
    const unsigned long long total = __shfl_sync(0xffffffffu, w, 31);
    scratch[lane] = w;
    unsigned long long start = 0;
    bool ok = true;
    if (total) ok = warp_reserve_ensure(t, s, total, start);
    if (lane == 0) { scratch[32] = start; scratch[33] = ok; }
  }
  __syncthreads();
  const unsigned long long total = scratch[BLOCK / 32 - 1];
  const unsigned long long start = scratch[32];
  const bool ok = scratch[33] != 0;
  const uint32_t excl = x - count + (wid ? (uint32_t)scratch[wid - 1] : 0u);
  __shared__ char *bptr_s[64];
  const uint32_t esz_log = sizeof(T) == 1 ? 0 : sizeof(T) == 2 ? 1 : sizeof(T) == 4 ? 2 : 3;
  const bool vec = t.log2fb + esz_log >= 4;               // every bucket is whole 16 B vectors
  const uint32_t shift = vec ? (uint32_t)(start % VE) : 0u;
  if (ok && total) {
    uint32_t b0, b1;
    uint64_t o;
    locate(start, t.log2fb, b0, o);
    locate(start + total - 1, t.log2fb, b1, o);
    if (tid <= b1 - b0) bptr_s[b0 + tid] = bucket_known(t, s, b0 + tid);
    uint32_t r = 0;
#pragma unroll
    for (int j = 0; j < K; ++j)
      if ((mask >> j) & 1u) stage[shift + excl + r++] = vals[j];
  }
  __syncthreads();
  if (ok && total) {
    if (vec) {
      const uint32_t nv = (uint32_t)((shift + total + VE - 1) / VE);
      // the run usually lies in ONE bucket: one address computation, each
      // vector an offset from it
      // (4 / 8 B elements; for 1 / 2 B the extra live registers cost more)
      uint32_t bf = 0, bl = 1;
      uint64_t of = 0, ol;
      if (sizeof(T) >= 4) {
        locate(start - shift, t.log2fb, bf, of);
        locate(start + total - 1, t.log2fb, bl, ol);
      }
      T *const rbase = bf == bl && bptr_s[bf] ? reinterpret_cast<T *>(bptr_s[bf]) + of : nullptr;
      for (uint32_t v = tid; v < nv; v += BLOCK) {
        T *dp;
        if (bf == bl) {
          if (!rbase) break;
          dp = rbase + v * VE;
        } else {
          uint32_t b;
          uint64_t o;
          locate(start - shift + (uint64_t)v * VE, t.log2fb, b, o);
          char *base = bptr_s[b];
          if (!base) continue;
          dp = reinterpret_cast<T *>(base) + o;
        }
        const uint32_t k0 = v * VE;
        if (k0 >= shift && k0 + VE <= shift + total) {
          const uint4 q = reinterpret_cast<const uint4 *>(stage)[v];
          asm volatile("st.global.cg.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(dp), "r"(q.x), "r"(q.y), "r"(q.z),
                       "r"(q.w) : "memory");
        } else {
          for (uint32_t j = 0; j < VE; ++j)
            if (k0 + j >= shift && k0 + j < shift + total) store_cg(dp + j, stage[k0 + j]);
        }
      }
    } else {
      for (uint32_t k = tid; k < total; k += BLOCK) {
        uint32_t b;
        uint64_t o;
        locate(start + k, t.log2fb, b, o);
        if (bptr_s[b]) store_cg(reinterpret_cast<T *>(bptr_s[b]) + o, stage[k]);
      }
    }
  }
  __syncthreads();
  return start;
}

// Paper Alg. 1, block flavour: thread j contributes vals[0..count_j); a
// shared-memory scan of the counts gives each thread its offset, thread 0
// reserves the block total with ONE atomicAdd and allocates the buckets, the
// values land in thread order.  `scratch` is 34 u64 of shared memory; BLOCK is
// blockDim.x (multiple of 32).  Returns the block's start index.
template <int BLOCK, typename T>
__device__ inline uint64_t block_push_back(const gg_device_view &t, uint32_t s, uint32_t count,
                                           const T *vals, unsigned long long *scratch) {
  static_assert(BLOCK % 32 == 0 && BLOCK <= 1024, "BLOCK must be a multiple of 32, <= 1024");
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  unsigned long long x = count;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    unsigned long long y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  if (lane == 31) scratch[wid] = x;
  __syncthreads();
  if (wid == 0) {
    unsigned long long w = lane < BLOCK / 32 ? scratch[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      unsigned long long y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= (uint32_t)d) w += y;
    }
    scratch[lane] = w;
  }
  __syncthreads();
  const unsigned long long excl = x - count + (wid ? scratch[wid - 1] : 0);
  const unsigned long long total = scratch[BLOCK / 32 - 1];
  __syncthreads();
  if (wid == 0 && total) {                 // warp 0 reserves (and allocates in parallel)
    unsigned long long start = 0;
    const bool ok = warp_reserve_ensure(t, s, total, start);
    if (lane == 0) { scratch[32] = start; scratch[33] = ok; }
  } else if (tid == 0) {
    scratch[32] = 0;
    scratch[33] = 1;
  }
  __syncthreads();
  const unsigned long long start = scratch[32];
  const bool ok = scratch[33] != 0;
  __shared__ char *bptr[64];
  if (ok && total) {
    uint32_t b0, b1;
    uint64_t o;
    locate(start, t.log2fb, b0, o);
    locate(start + total - 1, t.log2fb, b1, o);
    if (tid <= b1 - b0) bptr[b0 + tid] = bucket_known(t, s, b0 + tid);
  }
  __syncthreads();
  if (ok)
    for (uint32_t e = 0; e < count; ++e) {
      uint32_t b;
      uint64_t o;
      locate(start + excl + e, t.log2fb, b, o);
      if (bptr[b]) store_cg(reinterpret_cast<T *>(bptr[b]) + o, vals[e]);
    }
  __syncthreads();
  return start;
}

}  // namespace gg

#endif  // GGARRAY_DEVICE_CUH
