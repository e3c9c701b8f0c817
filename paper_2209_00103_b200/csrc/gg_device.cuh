// gg_device.cuh -- device side of the B200 GGArray library: bucket
// publication, reservation, commit / shrink / metadata kernels, the streaming
// primitives and the one-tile-per-CTA walker (insert, duplicate, flatten,
// r/w), rw_g, gather/scatter and the static-array baseline kernels.
#ifndef GG_DEVICE_CUH
#define GG_DEVICE_CUH

#include "gg_common.cuh"

namespace gg {

// ------------------------------------------------------------------ device side

template <int ESZ> struct ElemT;
template <> struct ElemT<1> { typedef uint8_t T; };
template <> struct ElemT<2> { typedef uint16_t T; };
template <> struct ElemT<4> { typedef uint32_t T; };
template <> struct ElemT<8> { typedef unsigned long long T; };

// Programmatic dependent launch: every library kernel lets its stream
// successor launch as soon as all its CTAs are running, and waits for its
// predecessor's completion before touching memory (griddepcontrol.wait is a
// no-op when the launch was not programmatic).
__device__ __forceinline__ void pdl_begin() {
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  asm volatile("griddepcontrol.wait;" ::: "memory");
}

__device__ __forceinline__ void stage_cbase(const Tables &t, char **scb) {
  for (uint32_t i = threadIdx.x; i < t.MB; i += blockDim.x) scb[i] = t.cbase[i];
}

// Host-planned allocation of class-b buckets for every lane with `need`
// (each (shard, bucket) is requested by exactly one lane, so the once-flags
// are uncontended and the slot is the shard's own: no address atomics at
// all; one counter update per warp and class).
__device__ __forceinline__ void warp_alloc_class(const Tables &t, bool need, uint32_t s,
                                                 uint32_t b) {
  const unsigned m = __ballot_sync(0xffffffffu, need);
  if (!m) return;
  if ((threadIdx.x & 31) == __ffs(m) - 1) atomicAdd(&t.misc[MISC_ALLOCS], (unsigned long long)__popc(m));
  if (!need) return;
  // plain stores: these launches only publish host-planned buckets and the
  // kernel boundary orders them before any reader
  t.ptr[(size_t)s * t.MB + b] = bucket_slot(t, s, b);
  atomicAdd((unsigned long long *)&t.cap[s], 1ull << (t.log2fb + b));
  t.flag[(size_t)s * t.MB + b] = kFlagPublished;
  atomicOr(&t.pmask[s], 1ull << b);
}

// allocate buckets [lo, hi) of shard s that are not yet published, warp-wide
// loop over classes (lanes without work pass lo = hi)
__device__ __forceinline__ void warp_alloc_range(const Tables &t, uint32_t s, uint32_t lo,
                                                 uint32_t hi) {
  // classes this lane needs = [lo, hi) minus the published ones (one mask load)
  unsigned long long want = 0;
  if (hi > lo) {
    want = (hi >= 64 ? ~0ull : ((1ull << hi) - 1ull)) & ~((1ull << lo) - 1ull);
    want &= ~t.pmask[s];
  }
  unsigned long long any = want;
#pragma unroll
  for (int d = 16; d; d >>= 1) any |= __shfl_xor_sync(0xffffffffu, any, d);
  while (any) {
    const uint32_t b = __ffsll((long long)any) - 1;
    any &= any - 1;
    warp_alloc_class(t, (want >> b) & 1ull, s, b);
  }
}

// Publish buckets (host-planned, slots already backed) for a whole CTA whose
// thread i handles shard base + i with mask `want` (every thread calls it,
// uniform control flow, blockDim <= NT): the shard's pmask (pm = its value at
// kernel start) and capacity, one allocation-count update per warp, then the
// bucket table rows (slot pointer + once-flag per bucket).  A row is t.MB
// entries, so thread-per-shard stores land MB entries apart (one sector per
// store, ~1.3 us per bucket and 512 shards from one SM); instead the CTA ORs
// the masks and writes the [bmin, bmax] window of its rows with consecutive
// threads on consecutive entries.  Plain stores: the kernel boundary orders
// them before any reader.
template <int NT>
__device__ __forceinline__ void publish_buckets_cta(const Tables &t, char *const *scb, uint32_t base,
                                                    unsigned long long pm, unsigned long long want,
                                                    uint32_t lg0) {
  __shared__ unsigned long long w_sh[NT];
  __shared__ unsigned long long or_sh[NT / 32];
  const uint32_t s = base + threadIdx.x, lane = threadIdx.x & 31;
  uint64_t add = 0;
  for (unsigned long long m = want; m; m &= m - 1) add += 1ull << (t.log2fb + __ffsll((long long)m) - 1);
  if (want) {
    t.pmask[s] = pm | want;
    atomicAdd((unsigned long long *)&t.cap[s], (unsigned long long)add);
  }
  const uint32_t tot = __reduce_add_sync(0xffffffffu, (uint32_t)__popcll(want));
  if (lane == 0 && tot) atomicAdd(&t.misc[MISC_ALLOCS], (unsigned long long)tot);
  w_sh[threadIdx.x] = want;
  const uint32_t olo = __reduce_or_sync(0xffffffffu, (uint32_t)want);
  const uint32_t ohi = __reduce_or_sync(0xffffffffu, (uint32_t)(want >> 32));
  if (lane == 0) or_sh[threadIdx.x >> 5] = ((unsigned long long)ohi << 32) | olo;
  __syncthreads();
  unsigned long long u = 0;
  for (uint32_t i = 0; i < (blockDim.x >> 5); ++i) u |= or_sh[i];
  if (u) {
    const uint32_t bmin = __ffsll((long long)u) - 1, bmax = 63 - __clzll((long long)u);
    const uint32_t W = bmax - bmin + 1;
    const uint32_t rows = base < t.S ? min(blockDim.x, t.S - base) : 0u;
    for (uint32_t e = threadIdx.x; e < rows * W; e += blockDim.x) {
      const uint32_t r = e / W, b = bmin + e % W;
      if (w_sh[r] >> b & 1) {
        const uint32_t ss = base + r;
        t.ptr[(size_t)ss * t.MB + b] = scb[b] + ((uint64_t)ss << max(lg0 + b, 4u));
        t.flag[(size_t)ss * t.MB + b] = kFlagPublished;
      }
    }
  }
  __syncthreads();                       // w_sh / or_sh are reused by the next call
}

// Reservation + bucket allocation, one thread per shard: one atomicAdd on the
// shard's size per batch (bucket_vector.py:229 via insert_index.py:118-122),
// then allocate every missing bucket of the reserved range
// (bucket_vector.py:207-214, 234-238).  Count sources:
//   mode 0: CSR offsets (insert); mode 1: committed lengths (duplicate);
//   mode 2: explicit starts + counts already in t.start/t.count (fetch_add'ed)
__device__ __forceinline__ void reserve_shards(const Tables &t, uint32_t s, bool live, int mode) {
  uint64_t c = 0, start = 0;
  uint32_t lo = 0, hi = 0;
  if (live) {
    if (mode == 0) c = t.offsets[s + 1] - t.offsets[s];
    else if (mode == 1) c = t.prefix[s + 1] - t.prefix[s];
    else c = t.count[s];
    const uint32_t ctl = t.ctl ? t.ctl[s] : (kCtlWrite | t.MB);
    if (mode != 2) {
      t.count[s] = c;
      if (c) {
        start = atomicAdd((unsigned long long *)&t.size[s], (unsigned long long)c);
        t.ops[s] += 1;
        t.start[s] = start;
      }
    } else {
      start = t.start[s];
    }
    if (c) {
      uint32_t b0, b1;
      uint64_t o;
      locate(start, t.log2fb, b0, o);
      locate(start + c - 1, t.log2fb, b1, o);
      lo = b0;
      hi = min(ctl & kCtlLimitMask, b1 + 1);
      if (hi < lo) hi = lo;
    }
  }
  warp_alloc_range(t, live ? s : 0, lo, hi);
}

__global__ void k_reserve(Tables t, int mode) {
  pdl_begin();
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  reserve_shards(t, s, s < t.S, mode);
}

// grow: thread per shard, allocate buckets [0, lim[s]); lim comes from the
// ctl words, or (uniform_k != ~0u) is the same for every shard.  Latency
// shaped: every global load (class bases, pmask, ctl) is issued up front, then
// one round of stores (publish_buckets).
__global__ void __launch_bounds__(256) k_grow(Tables t, uint32_t uniform_k) {
  __shared__ char *scb[kMaxBuckets];
  pdl_begin();
  stage_cbase(t, scb);
  const uint32_t s = blockIdx.x * blockDim.x + threadIdx.x;
  const bool live = s < t.S;
  const unsigned long long pm = live ? t.pmask[s] : 0ull;
  const uint32_t lim = !live ? 0u : (uniform_k != ~0u ? uniform_k : (t.ctl[s] & kCtlLimitMask));
  __syncthreads();
  const unsigned long long want = (lim >= 64 ? ~0ull : ((1ull << lim) - 1ull)) & ~pm;
  publish_buckets_cta<256>(t, scb, blockIdx.x * blockDim.x, pm, live ? want : 0ull,
                           t.log2fb + (31u - __clz(t.esz)));
}

__global__ void k_new_bucket(Tables t, uint32_t s, uint32_t b, int *won) {
  *won = alloc_bucket(t, s, b);
}

// view_finish's readback staging: size | cap | ops | pmask (u64 x S each) |
// status (u32 x S, 8 B aligned) | misc (u64 x MISC_N)
__host__ __device__ inline size_t view_pack_bytes(size_t S) { return S * 32 + ((S * 4 + 7) & ~size_t(7)) + MISC_N * 8; }
__global__ void __launch_bounds__(256) k_view_pack(Tables t, char *dst) {
  const size_t S = t.S;
  uint64_t *hs = (uint64_t *)dst, *hc = hs + S, *ho = hc + S, *hp = ho + S;
  uint32_t *hst = (uint32_t *)(hp + S);
  unsigned long long *hm = (unsigned long long *)(dst + S * 32 + ((S * 4 + 7) & ~size_t(7)));
  const uint32_t i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < S) {
    hs[i] = t.size[i]; hc[i] = t.cap[i]; ho[i] = t.ops[i]; hp[i] = t.pmask[i];
    hst[i] = t.status[i];
    t.status[i] = 0;
  }
  if (i < MISC_N) hm[i] = t.misc[i];
}

__global__ void k_fetch_add(Tables t, uint32_t s, uint64_t c) {
  atomicAdd((unsigned long long *)&t.size[s], (unsigned long long)c);
  t.ops[s] += 1;
}

// commit (sharded_array.py:213-222): one CTA, exclusive scan of S sizes.
__global__ void __launch_bounds__(1024) k_commit(Tables t) {
  pdl_begin();
  __shared__ uint64_t warp_tot[32];
  __shared__ uint64_t carry;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  if (tid == 0) carry = 0;
  __syncthreads();
  for (uint32_t base = 0; base < t.S; base += 1024) {
    uint32_t s = base + tid;
    uint64_t v = s < t.S ? t.size[s] : 0;
    uint64_t x = v;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= (uint32_t)d) x += y;
    }
    if (lane == 31) warp_tot[wid] = x;
    __syncthreads();
    if (wid == 0) {
      uint64_t w = warp_tot[lane];
#pragma unroll
      for (int d = 1; d < 32; d <<= 1) {
        uint64_t y = __shfl_up_sync(0xffffffffu, w, d);
        if (lane >= (uint32_t)d) w += y;
      }
      warp_tot[lane] = w;  // inclusive over warps
    }
    __syncthreads();
    uint64_t incl = x + (wid ? warp_tot[wid - 1] : 0) + carry;
    if (s < t.S) {
      t.prefix[s + 1] = incl;
      if (s == 0) t.prefix[0] = 0;
    }
    __syncthreads();
    if (tid == 1023) carry = incl;
    __syncthreads();
  }
}

// block-wide exclusive scan of one u64 per thread (blockDim multiple of 32);
// returns the exclusive prefix, *total gets the block sum.
__device__ __forceinline__ uint64_t block_exclusive_scan(uint64_t v, uint64_t *total,
                                                         uint64_t *warp_sums /* smem[32] */) {
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, nw = blockDim.x >> 5;
  uint64_t x = v;
#pragma unroll
  for (int d = 1; d < 32; d <<= 1) {
    uint64_t y = __shfl_up_sync(0xffffffffu, x, d);
    if (lane >= (uint32_t)d) x += y;
  }
  if (lane == 31) warp_sums[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint64_t w = lane < nw ? warp_sums[lane] : 0;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      uint64_t y = __shfl_up_sync(0xffffffffu, w, d);
      if (lane >= (uint32_t)d) w += y;
    }
    warp_sums[lane] = w;
  }
  __syncthreads();
  uint64_t incl = x + (wid ? warp_sums[wid - 1] : 0);
  *total = warp_sums[nw - 1];
  __syncthreads();
  return incl - v;
}

// Paper Alg. 1 with per-lane counts, pass 1: CTA per shard sums its lanes'
// counts (so the host can map the arena exactly before pass 2).
__global__ void __launch_bounds__(1024) k_lanes_count(Tables t, const uint32_t *counts, uint32_t K) {
  __shared__ uint64_t ws[32];
  const uint32_t s = blockIdx.x;
  const uint64_t lo = t.offsets[s], hi = t.offsets[s + 1];
  uint64_t acc = 0;
  for (uint64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) acc += min(counts[j], K);   // clamped to K
  uint64_t tot;
  block_exclusive_scan(acc, &tot, ws);
  if (threadIdx.x == 0) t.count[s] = tot;
}

// Pass 2 (paper Alg. 1): the CTA of shard s reserves its whole batch with ONE
// atomicAdd on the LFVector size, allocates the buckets the range touches
// (Alg. 2), then block-scans the lane counts chunk by chunk and every lane
// scatters its values to start + carry + exclusive_scan(lane).
template <int ESZ>
__global__ void __launch_bounds__(1024) k_lanes_insert(Tables t, const char *vals,
                                                       const uint32_t *counts, uint32_t K) {
  typedef typename ElemT<ESZ>::T E;
  __shared__ uint64_t ws[32];
  __shared__ char *bptr[64];
  __shared__ uint64_t start_s;
  __shared__ uint32_t ctl_s;
  const uint32_t s = blockIdx.x, tid = threadIdx.x;
  const uint64_t c = t.count[s];
  if (c == 0) return;
  if (tid == 0) {
    const uint32_t ctl = t.ctl ? t.ctl[s] : (kCtlWrite | t.MB);
    const uint64_t start = atomicAdd((unsigned long long *)&t.size[s], (unsigned long long)c);
    t.ops[s] += 1;
    uint32_t b0, b1; uint64_t o;
    locate(start, t.log2fb, b0, o);
    locate(start + c - 1, t.log2fb, b1, o);
    uint32_t lim = min(ctl & kCtlLimitMask, b1 + 1);
    for (uint32_t b = b0; b < lim; ++b)
      if (alloc_bucket(t, s, b) < 0) atomicOr(&t.status[s], (uint32_t)GG_ENOMEM);
    start_s = start;
    ctl_s = ctl;
  }
  __syncthreads();
  if (tid < t.MB) bptr[tid] = t.flag[(size_t)s * t.MB + tid] == kFlagPublished
                                  ? t.ptr[(size_t)s * t.MB + tid] : nullptr;
  __syncthreads();
  const uint64_t start = start_s;
  const uint32_t ctl = ctl_s;
  if (!(ctl & (kCtlWrite | kCtlZero))) return;
  const uint64_t lo = t.offsets[s], hi = t.offsets[s + 1];
  uint64_t carry = 0;
  for (uint64_t base = lo; base < hi; base += blockDim.x) {
    const uint64_t j = base + tid;
    const uint32_t cnt = j < hi ? min(counts[j], K) : 0;
    uint64_t tot;
    const uint64_t ex = block_exclusive_scan(cnt, &tot, ws);
    const E *src = (const E *)vals + j * K;
    for (uint32_t e = 0; e < cnt; ++e) {
      uint32_t b; uint64_t o;
      locate(start + carry + ex + e, t.log2fb, b, o);
      if (bptr[b]) ((E *)bptr[b])[o] = (ctl & kCtlWrite) ? src[e] : E(0);
    }
    carry += tot;
  }
}

// shrink (extension): one CTA; per shard size[s] = new size, buckets
// b >= min_buckets_for(new size) unpublished (their slots stay reserved for
// the shard; the host unmaps chunks that lost their last live bucket), then
// the commit scan over the new sizes.  All loads issued up front.
// new_sizes == nullptr: every shard shrinks to uniform_size (no upload)
// Metadata of a uniform planned append when the walk's metadata CTA is off
// (S > 4096, plain capture, gg_set_fuse(0)): every LFVector appended c at the
// same start with the same buckets, so the host knows every value and the
// kernel only stores, with as many CTAs as the tables need (the one-CTA
// k_planned_meta serialises over S).
__global__ void __launch_bounds__(256) k_meta_uniform(Tables t, uint64_t start, uint64_t c, int commit,
                                                      unsigned long long want, unsigned long long new_pm,
                                                      uint64_t new_cap) {
  pdl_begin();
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  const uint64_t nsz = start + c;
  for (uint64_t s = tid; s < t.S; s += nt) {
    t.size[s] = nsz;
    t.start[s] = start;
    t.count[s] = c;
    t.ops[s] += 1;
    if (want) { t.pmask[s] = new_pm; t.cap[s] = new_cap; }
    if (commit) t.prefix[s + 1] = (s + 1) * nsz;
  }
  if (tid == 0) {
    if (commit) t.prefix[0] = 0;
    if (want) atomicAdd(&t.misc[MISC_ALLOCS], (unsigned long long)__popcll(want) * t.S);
  }
  if (want) {
    char *const *cb = t.cbase;
    const uint32_t lg0 = t.log2fb + (31u - __clz(t.esz));
    const uint32_t bmin = __ffsll((long long)want) - 1, bmax = 63 - __clzll((long long)want);
    const uint32_t W = bmax - bmin + 1;
    for (uint64_t e = tid; e < (uint64_t)t.S * W; e += nt) {
      const uint32_t b = bmin + (uint32_t)(e % W);
      if (want >> b & 1) {
        const uint64_t ss = e / W;
        t.ptr[(size_t)ss * t.MB + b] = cb[b] + (ss << max(lg0 + b, 4u));
        t.flag[(size_t)ss * t.MB + b] = kFlagPublished;
      }
    }
  }
}

// Uniform shrink (every LFVector to the same size, same buckets): the host
// knows the result, so the kernel only stores -- sizes, pmask, capacity and
// the prefix (arithmetic, no scan) per LFVector, and the dropped buckets'
// table entries as one coalesced window over all rows -- with as many CTAs
// as the tables need (the one-CTA k_shrink strides MB entries apart per
// thread and serialises over S).
__global__ void __launch_bounds__(256) k_shrink_uniform(Tables t, uint64_t ns, unsigned long long drop,
                                                        unsigned long long new_pm, uint64_t new_cap) {
  pdl_begin();
  const uint64_t tid = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x, nt = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t s = tid; s < t.S; s += nt) {
    t.size[s] = ns;
    t.prefix[s + 1] = (s + 1) * ns;
    if (drop) { t.pmask[s] = new_pm; t.cap[s] = new_cap; }
  }
  if (tid == 0) t.prefix[0] = 0;
  if (drop) {
    const uint32_t bmin = __ffsll((long long)drop) - 1, bmax = 63 - __clzll((long long)drop);
    const uint32_t W = bmax - bmin + 1;
    for (uint64_t e = tid; e < (uint64_t)t.S * W; e += nt) {
      const uint32_t b = bmin + (uint32_t)(e % W);
      if (drop >> b & 1) {
        const size_t i = (size_t)(e / W) * t.MB + b;
        t.ptr[i] = nullptr;
        t.flag[i] = 0;
      }
    }
  }
}

__global__ void __launch_bounds__(1024) k_shrink(Tables t, const uint64_t *new_sizes,
                                                 uint64_t uniform_size) {
  __shared__ uint64_t ws[32];
  pdl_begin();
  uint64_t carry = 0;
  for (uint32_t base = 0; base < t.S; base += blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    const bool live = s < t.S;
    uint64_t ns = 0, cap = 0;
    unsigned long long m = 0;
    if (live) { ns = new_sizes ? new_sizes[s] : uniform_size; m = t.pmask[s]; cap = t.cap[s]; }
    if (live) {
      const uint32_t keep = ns ? (64u - (uint32_t)__clzll((long long)((ns + (1ull << t.log2fb) - 1) >> t.log2fb))) : 0u;
      const unsigned long long drop = keep < 64 ? (m & ~((1ull << keep) - 1ull)) : 0ull;
      uint64_t freed = 0;
      for (unsigned long long d = drop; d; d &= d - 1) {
        const uint32_t b = __ffsll((long long)d) - 1;
        t.ptr[(size_t)s * t.MB + b] = nullptr;
        t.flag[(size_t)s * t.MB + b] = 0;
        freed += 1ull << (t.log2fb + b);
      }
      if (drop) { t.pmask[s] = m & ~drop; t.cap[s] = cap - freed; }
      t.size[s] = ns;
    }
    uint64_t tot;
    const uint64_t ex = block_exclusive_scan(ns, &tot, ws);
    if (live) t.prefix[s + 1] = carry + ex + ns;
    carry += tot;
  }
  if (threadIdx.x == 0) t.prefix[0] = 0;
}

// ---- streaming primitives: a CTA moves one contiguous piece -------------


__device__ __forceinline__ uint4 ldg_stream(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_rw(const uint4 *p) {
  uint4 r;
  asm volatile("ld.global.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void stg(uint4 *p, const uint4 &v) {
  asm volatile("st.global.L1::no_allocate.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x),
               "r"(v.y), "r"(v.z), "r"(v.w) : "memory");
}

// Cache policy of the streaming loads/stores (selected by the tuning sweep):
// 0 = L2-only (.cg), 1 = read-only path loads (.nc) + default stores,
// 2 = default loads/stores, 3 = evict-first streaming (.cs).
template <int LS> struct LdSt;
template <> struct LdSt<0> {
  template <class V> __device__ __forceinline__ static V ld(const V *p) { return __ldcg(p); }
  template <class V> __device__ __forceinline__ static void st(V *p, const V &v) { __stcg(p, v); }
};
template <> struct LdSt<1> {
  template <class V> __device__ __forceinline__ static V ld(const V *p) { return __ldg(p); }
  template <class V> __device__ __forceinline__ static void st(V *p, const V &v) { *p = v; }
};
template <> struct LdSt<2> {
  template <class V> __device__ __forceinline__ static V ld(const V *p) { return *p; }
  template <class V> __device__ __forceinline__ static void st(V *p, const V &v) { *p = v; }
};
template <> struct LdSt<3> {
  template <class V> __device__ __forceinline__ static V ld(const V *p) { return __ldcs(p); }
  template <class V> __device__ __forceinline__ static void st(V *p, const V &v) { __stcs(p, v); }
};
constexpr int kDefLS = 0;
constexpr int kDefUnroll = 4;

// bytes [4q + r/8, 4q + r/8 + 16) of the 32-byte concatenation (a, b): the
// 16 B vector starting m = 4q + r/8 bytes into a (q < 4, r in {0, 8, 16, 24})
__device__ __forceinline__ uint4 realign16(const uint4 &a, const uint4 &b, uint32_t q, uint32_t r) {
  const uint32_t w0 = q == 0 ? a.x : q == 1 ? a.y : q == 2 ? a.z : a.w;
  const uint32_t w1 = q == 0 ? a.y : q == 1 ? a.z : q == 2 ? a.w : b.x;
  const uint32_t w2 = q == 0 ? a.z : q == 1 ? a.w : q == 2 ? b.x : b.y;
  const uint32_t w3 = q == 0 ? a.w : q == 1 ? b.x : q == 2 ? b.y : b.z;
  const uint32_t w4 = q == 0 ? b.x : q == 1 ? b.y : q == 2 ? b.z : b.w;
  return make_uint4(__funnelshift_r(w0, w1, r), __funnelshift_r(w1, w2, r), __funnelshift_r(w2, w3, r),
                    __funnelshift_r(w3, w4, r));
}

// dst[0..n) = src[0..n) (element granular, arbitrary relative alignment), or
// zeros if src == nullptr.  Stores are 16 B aligned vectors; loads are 16 B
// vectors, realigned in registers when src and dst are not congruent.
template <int ESZ, int UNROLL, int LS = kDefLS>
__device__ __forceinline__ void cta_copy(char *dst, const char *src, uint64_t n, uint32_t tid,
                                         uint32_t nt) {
  typedef LdSt<LS> M;
  typedef typename ElemT<ESZ>::T E;
  constexpr uint32_t VE = 16 / ESZ;
  const uintptr_t d = (uintptr_t)dst;
  uint64_t head = ((16 - (d & 15)) & 15) / ESZ;
  if (head > n) head = n;
  const uint64_t body = (n - head) / VE;
  const uint64_t tail0 = head + body * VE;
  E *de = (E *)dst;
  const E *se = (const E *)src;
  for (uint64_t e = tid; e < head; e += nt) de[e] = src ? se[e] : E(0);
  for (uint64_t e = tail0 + tid; e < n; e += nt) de[e] = src ? se[e] : E(0);
  uint4 *dv = (uint4 *)(dst + head * ESZ);
  if (src == nullptr) {
    const uint4 z = make_uint4(0, 0, 0, 0);
    for (uint64_t v = tid; v < body; v += nt) M::st(dv + v, z);
    return;
  }
  const char *sb = src + head * ESZ;
  if ((((uintptr_t)sb) & 15) == 0) {
    // batches of UNROLL independent 16 B loads per thread, all issued before
    // the stores; loads past the end are clamped (re-read the last vector) so
    // they stay unconditional and the compiler cannot interleave them
    const uint4 *sv = (const uint4 *)sb;
    for (uint64_t v0 = tid; v0 < body; v0 += UNROLL * (uint64_t)nt) {
      uint4 r[UNROLL];
#pragma unroll
      for (int u = 0; u < UNROLL; ++u) r[u] = M::ld(sv + min(v0 + u * (uint64_t)nt, body - 1));
#pragma unroll
      for (int u = 0; u < UNROLL; ++u)
        if (v0 + u * (uint64_t)nt < body) M::st(dv + v0 + u * nt, r[u]);
    }
  } else {
    // source not congruent with the destination: aligned 16 B loads of the
    // source; output vector v is assembled from aligned vectors v and v + 1
    // shifted by the byte misalignment.  Each warp loads a window of 32
    // consecutive aligned vectors and writes the 31 outputs it fully holds
    // (lane l takes lane l + 1's vector by shuffle), so no lane loads twice
    // and registers stay at U vectors.  Loop bounds are warp-uniform
    // (shuffles); loads are clamped to vector `body` of the aligned source --
    // an aligned 16 B vector holding at least one source byte, so it never
    // leaves a mapped page.
    const uint32_t m = (uint32_t)((uintptr_t)sb & 15), q = m >> 2, r = (m & 3) * 8;
    const uint4 *sa = (const uint4 *)(sb - m);
    // (at most 4 vectors in flight: the kernels' register budget is set by
    // their congruent paths)
    constexpr int UR = UNROLL > 4 ? 4 : UNROLL;
    const uint32_t lane = tid & 31, nw = nt >> 5;
    for (uint64_t w0 = tid >> 5; 31 * w0 < body; w0 += UR * (uint64_t)nw) {
      uint4 a[UR];
#pragma unroll
      for (int k = 0; k < UR; ++k) a[k] = M::ld(sa + min(31 * (w0 + k * (uint64_t)nw) + lane, body));
#pragma unroll
      for (int k = 0; k < UR; ++k) {
        uint4 h;
        h.x = __shfl_down_sync(0xffffffffu, a[k].x, 1);
        h.y = __shfl_down_sync(0xffffffffu, a[k].y, 1);
        h.z = __shfl_down_sync(0xffffffffu, a[k].z, 1);
        h.w = __shfl_down_sync(0xffffffffu, a[k].w, 1);
        const uint64_t v = 31 * (w0 + k * (uint64_t)nw) + lane;
        if (lane < 31 && v < body) M::st(dv + v, realign16(a[k], h, q, r));
      }
    }
  }
}

// typed wrapping / IEEE add used by the r/w passes
template <typename T> struct AddOp {
  __device__ __forceinline__ static T apply(T x, T a) { return (T)(x + a); }
};
template <> struct AddOp<int8_t> {
  __device__ __forceinline__ static int8_t apply(int8_t x, int8_t a) {
    return (int8_t)(uint8_t)((uint8_t)x + (uint8_t)a);
  }
};
template <> struct AddOp<int16_t> {
  __device__ __forceinline__ static int16_t apply(int16_t x, int16_t a) {
    return (int16_t)(uint16_t)((uint16_t)x + (uint16_t)a);
  }
};
template <> struct AddOp<int32_t> {
  __device__ __forceinline__ static int32_t apply(int32_t x, int32_t a) {
    return (int32_t)((uint32_t)x + (uint32_t)a);
  }
};
template <> struct AddOp<long long> {
  __device__ __forceinline__ static long long apply(long long x, long long a) {
    return (long long)((unsigned long long)x + (unsigned long long)a);
  }
};
template <> struct AddOp<float> {
  __device__ __forceinline__ static float apply(float x, float a) { return __fadd_rn(x, a); }
};
template <> struct AddOp<double> {
  __device__ __forceinline__ static double apply(double x, double a) { return __dadd_rn(x, a); }
};
template <> struct AddOp<__half> {
  // numpy float16 arithmetic: widen to float32, add, round back (exact RN)
  __device__ __forceinline__ static __half apply(__half x, __half a) {
    return __float2half_rn(__half2float(x) + __half2float(a));
  }
};

// in-place p[0..n) = p + a (applied `reps` times in registers; reps = 1 for a
// separate sweep per pass)
template <typename T, int UNROLL, int LS = kDefLS>
__device__ __forceinline__ void cta_add(char *p, uint64_t n, T a, uint32_t reps, uint32_t tid,
                                        uint32_t nt) {
  typedef LdSt<LS == 1 ? 2 : LS> M;   // no read-only path for in-place updates
  constexpr uint32_t VE = 16 / sizeof(T);
  const uintptr_t d = (uintptr_t)p;
  uint64_t head = ((16 - (d & 15)) & 15) / sizeof(T);
  if (head > n) head = n;
  const uint64_t body = (n - head) / VE;
  const uint64_t tail0 = head + body * VE;
  T *pe = (T *)p;
  for (uint64_t e = tid; e < head; e += nt) {
    T x = pe[e];
    for (uint32_t r = 0; r < reps; ++r) x = AddOp<T>::apply(x, a);
    pe[e] = x;
  }
  for (uint64_t e = tail0 + tid; e < n; e += nt) {
    T x = pe[e];
    for (uint32_t r = 0; r < reps; ++r) x = AddOp<T>::apply(x, a);
    pe[e] = x;
  }
  uint4 *pv = (uint4 *)(p + head * sizeof(T));
  for (uint64_t v0 = tid; v0 < body; v0 += UNROLL * (uint64_t)nt) {
    union { uint4 q; T e[VE]; } u[UNROLL];
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) u[k].q = M::ld(pv + min(v0 + k * (uint64_t)nt, body - 1));
#pragma unroll
    for (int k = 0; k < UNROLL; ++k) {
      if (v0 + k * (uint64_t)nt < body) {
        for (uint32_t r = 0; r < reps; ++r)
#pragma unroll
          for (uint32_t j = 0; j < VE; ++j) u[k].e[j] = AddOp<T>::apply(u[k].e[j], a);
        M::st(pv + v0 + k * nt, u[k].q);
      }
    }
  }
}

// ---- tile walker ------------------------------------------------------------
// The work space is an index range [0, total) partitioned among shards by a
// directory dir[S+1] (CSR offsets for inserts, the committed prefix for
// duplicate / flatten / r/w).  A CTA takes one tile and walks it
// in pieces over which shard, source bucket and destination bucket are all
// constant; every thread computes the (uniform) piece bounds itself.
enum { W_INSERT = 0, W_DUP = 1, W_FLATTEN = 2, W_RW = 3 };

__device__ __forceinline__ uint32_t upper_shard(const uint64_t *dir, uint32_t S, uint64_t g) {
  // largest s with dir[s] <= g (bisect_right - 1, sharded_array.py:136)
  uint32_t lo = 0, hi = S;  // dir[0] = 0 <= g
  while (hi - lo > 1) {
    uint32_t mid = (lo + hi) >> 1;
    if (dir[mid] <= g) lo = mid; else hi = mid;
  }
  return lo;
}


// Bucket (s, b) sits at a fixed slot of class b's slab (gg_device_view), so
// kernels compute bucket addresses instead of loading them: scb[] holds the
// class bases staged in shared memory, lg0 = log2(fb * element bytes).
__device__ __forceinline__ char *slot_addr(char *const *scb, uint32_t s, uint32_t b, uint32_t lg0) {
  return scb[b] + ((uint64_t)s << max(lg0 + b, 4u));
}

// directory accessor: loads dir[i], or i * ulen for a uniform directory
struct DirV {
  const uint64_t *p;
  uint64_t u;
  __device__ __forceinline__ uint64_t operator[](uint32_t i) const { return u ? (uint64_t)i * u : p[i]; }
};

// shard of work index g: largest s with dir[s] <= g (bisect_right - 1,
// sharded_array.py:136) by a 32-ary warp search -- 2 dependent loads for
// S <= 1024, 3 up to 32768.  Called by a full warp; result in every lane.
__device__ __forceinline__ uint32_t warp_find_shard(const uint64_t *dir, uint32_t S, uint64_t g) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = S;                 // answer in [lo, hi)
  while (hi - lo > 1) {
    const uint32_t step = (hi - lo + 31) >> 5;
    const uint32_t p = lo + lane * step;
    const bool ok = p < hi && dir[p] <= g;
    const unsigned m = __ballot_sync(0xffffffffu, ok);   // lane 0 (p = lo) always ok
    lo = lo + (31u - __clz(m)) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

// One tile [g, gend) lying inside shard s with 16 B-congruent source and
// destination: each thread moves U vectors, resolving every vector's bucket
// on its own (clz locate + slot arithmetic) and issuing all U loads before
// any store -- one memory round trip per tile however many buckets it
// touches.  Returns false (tile not handled) when the tile crosses a shard
// or the alignment does not hold.
template <int ESZ, int W, typename T, int U, int LS>
__device__ __forceinline__ bool vector_tile(const Tables &t, char *const *scb, const DirV dir,
                                            uint32_t s, uint64_t dbase, uint64_t g, uint64_t gend,
                                            const char *flat_src, char *flat_dst, T addend,
                                            uint32_t reps) {
  constexpr uint32_t VE = 16 / ESZ;
  const uint64_t lo = dir[s];
  if (gend > dir[s + 1] || ((g - lo) % VE) || ((gend - g) % VE) || (t.log2fb < 31 && ((1u << t.log2fb) % VE)))
    return false;
  if constexpr (W == W_INSERT || W == W_DUP) {
    if (dbase % VE) return false;
  }
  if constexpr (W == W_INSERT) {
    if (((uintptr_t)(flat_src + g * ESZ)) & 15) return false;
  }
  if constexpr (W == W_FLATTEN) {
    if (((uintptr_t)(flat_dst + g * ESZ)) & 15) return false;
  }
  typedef LdSt<(W == W_RW && LS == 1) ? 2 : LS> M;
  constexpr uint32_t LGE = ESZ == 1 ? 0 : ESZ == 2 ? 1 : ESZ == 4 ? 2 : 3;
  const uint32_t lg0 = t.log2fb + LGE;
  const uint64_t nvec = (gend - g) / VE;
  const uint64_t k0 = g - lo;              // work-space offset inside the shard
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  for (uint64_t v0 = tid; v0 < nvec; v0 += U * (uint64_t)nt) {
    uint4 r[U];
    char *sp[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = min(v0 + u * (uint64_t)nt, nvec - 1);
      if constexpr (W == W_INSERT) {
        sp[u] = (char *)flat_src + (g + v * VE) * ESZ;
      } else {
        uint32_t b; uint64_t o;
        locate(k0 + v * VE, t.log2fb, b, o);
        sp[u] = slot_addr(scb, s, b, lg0) + o * ESZ;
      }
      r[u] = M::ld((const uint4 *)sp[u]);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = v0 + u * (uint64_t)nt;
      if (v >= nvec) continue;
      char *dp;
      if constexpr (W == W_FLATTEN) {
        dp = flat_dst + (g + v * VE) * ESZ;
      } else if constexpr (W == W_RW) {
        dp = sp[u];
        union { uint4 q; T e[VE]; } x;
        x.q = r[u];
        for (uint32_t rr = 0; rr < reps; ++rr)
#pragma unroll
          for (uint32_t j = 0; j < VE; ++j) x.e[j] = AddOp<T>::apply(x.e[j], addend);
        r[u] = x.q;
      } else {
        uint32_t b; uint64_t o;
        locate(dbase + k0 + v * VE, t.log2fb, b, o);
        dp = slot_addr(scb, s, b, lg0) + o * ESZ;
      }
      M::st((uint4 *)dp, r[u]);
    }
  }
  return true;
}

// Planned append (PLANNED): the host has already backed every destination
// slot and knows each shard's count, so the copy needs no reservation phase:
// destinations are slot arithmetic from the unchanged size[s]; k_planned_meta
// applies the metadata right after.  (A last-CTA epilogue in the walk itself
// costs more: the completion atomic lengthens every CTA's life.)
struct Fuse {
  int rmode;
  int commit;
  uint64_t g0 = 0;                 // first work index (ranges)
  // metadata CTA inside the planned walk (double-buffered size / prefix):
  // the walk's copy CTAs read the current buffers, the last CTA writes the
  // next ones (and publishes the buckets of a deferred uniform grow_k)
  uint64_t *size_next = nullptr;
  uint64_t *prefix_next = nullptr;
  uint32_t grow_k = 0;
  // uniform directory (every shard's work length = ulen, known on the host):
  // shard lookup is a division, no directory loads; planned walks also take
  // the common destination start ustart instead of loading size[s]
  uint64_t ulen = 0;
  uint64_t ustart = 0;
  // (host only) longest shard work length of a non-uniform directory, 0 =
  // unknown: enables the shard-grid walk (k_walk_shard)
  uint64_t maxlen = 0;
};


// metadata of a planned append, run by one CTA after every tile is copied.
// Latency shaped: all loads (directory pair, size, pmask) issued up front,
// counters updated with fire-and-forget reductions, the commit scan runs on
// the new sizes held in registers (no reload).
__device__ void planned_metadata(const Tables &t, char *const *scb, const Fuse &fz) {
  __shared__ uint64_t ws[32];
  const uint32_t lg0 = t.log2fb + (31u - __clz(t.esz));
  const uint64_t *dir = fz.rmode == 0 ? t.offsets : t.prefix;
  // pass 1: every count is read before the commit below rewrites the prefix
  // (the duplicate's directory); with more shards than threads a later chunk
  // would otherwise read prefix entries an earlier chunk already replaced
  if (t.S > blockDim.x) {
    for (uint32_t s = threadIdx.x; s < t.S; s += blockDim.x) t.count[s] = dir[s + 1] - dir[s];
    __syncthreads();
  }
  uint64_t carry = 0;
  for (uint32_t base = 0; base < t.S; base += blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    const bool live = s < t.S;
    uint64_t c = 0, start = 0;
    unsigned long long pm = 0;
    if (live) {
      c = t.S > blockDim.x ? t.count[s] : dir[s + 1] - dir[s];
      start = t.size[s];
      pm = t.pmask[s];
    }
    const uint64_t nsz = start + c;
    unsigned long long want = 0;
    if (c) {
      // the batch's reservation: ONE atomicAdd on the LFVector size
      // (insert_index.py:118-122), fire-and-forget -- the start was read above
      // and this launch is the shard's only writer
      atomicAdd((unsigned long long *)&t.size[s], (unsigned long long)c);
      atomicAdd((unsigned long long *)&t.ops[s], 1ull);
      t.start[s] = start;
      uint32_t b0, b1; uint64_t o;
      locate(start, t.log2fb, b0, o);
      locate(nsz - 1, t.log2fb, b1, o);
      want = (b1 >= 63 ? ~0ull : ((2ull << b1) - 1ull)) & ~((1ull << b0) - 1ull) & ~pm;
    }
    if (live) t.count[s] = c;
    publish_buckets_cta<1024>(t, scb, base, pm, live ? want : 0ull, lg0);
    if (fz.commit) {
      uint64_t tot;
      const uint64_t ex = block_exclusive_scan(live ? nsz : 0, &tot, ws);
      if (live) t.prefix[s + 1] = carry + ex + nsz;
      carry += tot;
    }
  }
  if (fz.commit && threadIdx.x == 0) t.prefix[0] = 0;
}

// Metadata of a planned append run by the walk's extra CTA, concurrently with
// the copy CTAs: everything the copy reads (size, directory) is read from the
// current buffers and written to the next ones; nothing else it writes is
// read by the copy (addresses are slot arithmetic).  Also publishes the
// buckets of a deferred uniform grow (grow_k).
__device__ void planned_metadata_db(const Tables &t, char **scb, const Fuse &fz) {
  __shared__ uint64_t ws[32];
  constexpr int K = 4;                    // shards per thread whose loads are hoisted
  const uint32_t lg0 = t.log2fb + (31u - __clz(t.esz));
  const DirV dir{fz.rmode == 0 ? t.offsets : t.prefix, fz.ulen};
  const unsigned long long gmask = fz.grow_k >= 64 ? ~0ull : ((1ull << fz.grow_k) - 1ull);
  // latency: every per-shard load of the first K slices is issued before the
  // class bases are staged and before any dependent work (a uniform append
  // knows its start, no size load)
  uint64_t hc[K], hst[K], hpre[K];
  unsigned long long hpm[K];
#pragma unroll
  for (int i = 0; i < K; ++i) {
    const uint32_t s = threadIdx.x + i * blockDim.x;
    hc[i] = hst[i] = hpre[i] = 0;
    hpm[i] = 0;
    if (s < t.S) {
      hc[i] = dir[s + 1] - dir[s];
      hst[i] = fz.ulen ? fz.ustart : t.size[s];
      hpm[i] = t.pmask[s];
      if (!fz.commit) hpre[i] = t.prefix[s + 1];
    }
  }
  stage_cbase(t, scb);
  __syncthreads();
  uint64_t carry = 0;
  uint32_t it = 0;
  for (uint32_t base = 0; base < t.S; base += blockDim.x, ++it) {
    const uint32_t s = base + threadIdx.x;
    const bool live = s < t.S;
    uint64_t c = 0, start = 0, pre = 0;
    unsigned long long pm = 0;
    if (it < K) {
#pragma unroll
      for (int i = 0; i < K; ++i)
        if (i == (int)it) { c = hc[i]; start = hst[i]; pm = hpm[i]; pre = hpre[i]; }
    } else if (live) {
      c = dir[s + 1] - dir[s];
      start = fz.ulen ? fz.ustart : t.size[s];
      pm = t.pmask[s];
      if (!fz.commit) pre = t.prefix[s + 1];
    }
    const uint64_t nsz = start + c;
    unsigned long long want = live ? (gmask & ~pm) : 0ull;
    if (c) {
      atomicAdd((unsigned long long *)&t.ops[s], 1ull);
      t.start[s] = start;
      uint32_t b0, b1; uint64_t o;
      locate(start, t.log2fb, b0, o);
      locate(nsz - 1, t.log2fb, b1, o);
      want |= (b1 >= 63 ? ~0ull : ((2ull << b1) - 1ull)) & ~((1ull << b0) - 1ull) & ~pm;
    }
    if (live) {
      t.count[s] = c;
      fz.size_next[s] = nsz;            // the batch's reservation: one update per LFVector
    }
    publish_buckets_cta<256>(t, scb, base, pm, want, lg0);
    if (fz.commit) {
      uint64_t tot;
      const uint64_t ex = block_exclusive_scan(live ? nsz : 0, &tot, ws);
      if (live) fz.prefix_next[s + 1] = carry + ex + nsz;
      carry += tot;
    } else if (live) {
      fz.prefix_next[s + 1] = pre;
    }
  }
  if (threadIdx.x == 0) fz.prefix_next[0] = 0;
}

// copy the current size / prefix buffers into the other pair (restores the
// buffer parity at the end of a captured sequence)
__global__ void k_copy_db(uint64_t *size_dst, const uint64_t *size_src, uint64_t *pre_dst,
                          const uint64_t *pre_src, uint32_t S) {
  pdl_begin();
  for (uint32_t i = blockIdx.x * blockDim.x + threadIdx.x; i <= S; i += gridDim.x * blockDim.x) {
    if (i < S) size_dst[i] = size_src[i];
    pre_dst[i] = pre_src[i];
  }
}

// Tiles whose pieces are short (many LFVectors with a few elements each:
// small per-shard batches, ragged directories) are walked element by
// element: every thread resolves its own elements' shard (a bisect inside
// the tile's shard range, or a division for a uniform directory) and bucket,
// instead of the whole CTA stepping through the pieces one after another.
template <int ESZ, int W, typename T, bool PLANNED>
__device__ __forceinline__ void element_tile(const Tables &t, char *const *scb, const DirV &dir,
                                             uint32_t s_lo, uint32_t s_hi, uint64_t g, uint64_t gend,
                                             const char *flat_src, char *flat_dst, T addend,
                                             uint32_t reps, const Fuse &fz, uint32_t lg0) {
  typedef typename ElemT<ESZ>::T E;
  for (uint64_t x = g + threadIdx.x; x < gend; x += blockDim.x) {
    uint32_t s;
    if (dir.u) {
      s = (uint32_t)(x / dir.u);
    } else {                                   // largest s in [s_lo, s_hi] with dir[s] <= x
      uint32_t lo = s_lo, hi = s_hi + 1;
      while (hi - lo > 1) {
        const uint32_t mid = (lo + hi) >> 1;
        if (dir.p[mid] <= x) lo = mid; else hi = mid;
      }
      s = lo;
    }
    const uint64_t k = x - dir[s];
    const uint32_t ctl = (W == W_INSERT || W == W_DUP) && !PLANNED && t.ctl ? t.ctl[s] : kCtlWrite;
    const char *sp;
    if constexpr (W == W_INSERT) {
      sp = flat_src + x * ESZ;
    } else {
      uint32_t b; uint64_t o;
      locate(k, t.log2fb, b, o);
      sp = slot_addr(scb, s, b, lg0) + o * ESZ;
    }
    if constexpr (W == W_RW) {
      T v = *(const T *)sp;
      for (uint32_t r = 0; r < reps; ++r) v = AddOp<T>::apply(v, addend);
      *(T *)sp = v;
    } else {
      char *dp;
      bool dst_ok = true;
      if constexpr (W == W_FLATTEN) {
        dp = flat_dst + x * ESZ;
      } else {
        uint32_t b; uint64_t o;
        locate((PLANNED ? (fz.ulen ? fz.ustart : t.size[s]) : t.start[s]) + k, t.log2fb, b, o);
        if (!PLANNED) dst_ok = t.flag[(size_t)s * t.MB + b] == kFlagPublished;
        dp = slot_addr(scb, s, b, lg0) + o * ESZ;
      }
      if (dst_ok && (ctl & (kCtlWrite | kCtlZero)))
        *(E *)dp = (ctl & kCtlWrite) ? *(const E *)sp : E(0);
    }
  }
}

// The tile walker: ONE tile per CTA (a non-persistent grid streams ~15%
// faster than a persistent grid-stride loop on B200, tools/probe), tile =
// U vectors per thread.  The work space [0, total) is partitioned among
// shards by dir[S+1] (CSR offsets for inserts, the committed prefix for
// duplicate / flatten / r/w); a tile inside one shard with congruent
// alignment takes vector_tile, anything else the piece walker (pieces over
// which shard, source bucket and destination bucket are constant).
template <int ESZ, int W, typename T, int U = 4, int LS = kDefLS, bool PLANNED = false>
__global__ void __launch_bounds__(256) k_walk(Tables t, const char *flat_src, char *flat_dst,
                                              uint64_t total, T addend, uint32_t reps,
                                              uint32_t tile, Fuse fz) {
  __shared__ char *scb[kMaxBuckets];
  __shared__ uint32_t s_sh, s_last_sh;
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  pdl_begin();
  if constexpr (PLANNED) {
    // block 0 is the metadata CTA (dispatched first, so it overlaps the copy
    // instead of trailing it); the copy tiles are blocks 1..
    if (fz.size_next && blockIdx.x == 0) {
      planned_metadata_db(t, scb, fz);   // stages the class bases itself
      return;
    }
  }
  const DirV dir{(W == W_INSERT) ? t.offsets : t.prefix, fz.ulen};
  const uint64_t tile_idx = (PLANNED && fz.size_next) ? blockIdx.x - 1 : blockIdx.x;
  uint64_t g = fz.g0 + tile_idx * tile;
  const uint64_t gend = min(total, g + tile);
  if (fz.ulen) {
    if (tid == 0) s_sh = (uint32_t)(g / fz.ulen);
  } else if (tid < 32) {
    const uint32_t s0 = warp_find_shard(dir.p, t.S, g);
    if (tid == 0) s_sh = s0;
  }
  stage_cbase(t, scb);
  __syncthreads();
  constexpr uint32_t LGE = ESZ == 1 ? 0 : ESZ == 2 ? 1 : ESZ == 4 ? 2 : 3;
  const uint32_t lg0 = t.log2fb + LGE;
  uint32_t s = s_sh;
  bool fast = true;
  uint64_t dbase = 0;                      // destination local index of shard s's work index 0
  if constexpr (W == W_INSERT || W == W_DUP) {
    if (!PLANNED && t.ctl && t.ctl[s] != (kCtlWrite | t.MB)) fast = false;   // planned failure
    dbase = PLANNED ? (fz.ulen ? fz.ustart : t.size[s]) : t.start[s];
  }
  if (!(fast && vector_tile<ESZ, W, T, U, LS>(t, scb, dir, s, dbase, g, gend, flat_src, flat_dst,
                                              addend, reps))) {
    // short pieces (average < 128 elements): element by element
    uint32_t s_last;
    if (fz.ulen) {
      s_last = (uint32_t)((gend - 1) / fz.ulen);
    } else {
      if (tid < 32) {
        const uint32_t sl = warp_find_shard(dir.p, t.S, gend - 1);
        if (tid == 0) s_last_sh = sl;
      }
      __syncthreads();
      s_last = s_last_sh;
    }
    if (gend - g < 128ull * (s_last - s + 1)) {
      element_tile<ESZ, W, T, PLANNED>(t, scb, dir, s, s_last, g, gend, flat_src, flat_dst, addend, reps,
                                       fz, lg0);
      return;
    }
    while (g < gend) {
      uint64_t shard_end = dir[s + 1];
      while (shard_end <= g) { ++s; shard_end = dir[s + 1]; }
      const uint64_t k = g - dir[s];
      uint64_t len = min(gend, shard_end) - g;
      const uint32_t ctl = (W == W_INSERT || W == W_DUP) && !PLANNED && t.ctl ? t.ctl[s] : kCtlWrite;
      const char *sp = nullptr;
      char *dp = nullptr;
      bool dst_ok = true;
      // source side
      if constexpr (W == W_INSERT) {
        sp = flat_src + g * ESZ;
      } else {
        uint32_t b; uint64_t o;
        locate(k, t.log2fb, b, o);
        len = min(len, (uint64_t)((1ull << (t.log2fb + b)) - o));
        sp = slot_addr(scb, s, b, lg0) + o * ESZ;
      }
      // destination side
      if constexpr (W == W_FLATTEN) {
        dp = flat_dst + g * ESZ;
      } else if constexpr (W == W_RW) {
        dp = (char *)sp;
      } else {
        uint32_t b; uint64_t o;
        locate((PLANNED ? (fz.ulen ? fz.ustart : t.size[s]) : t.start[s]) + k, t.log2fb, b, o);
        len = min(len, (uint64_t)((1ull << (t.log2fb + b)) - o));
        if (!PLANNED) dst_ok = t.flag[(size_t)s * t.MB + b] == kFlagPublished;
        dp = slot_addr(scb, s, b, lg0) + o * ESZ;
      }
      if constexpr (W == W_RW) {
        cta_add<T, U, LS>(dp, len, addend, reps, tid, nt);
      } else if (dst_ok && (ctl & (kCtlWrite | kCtlZero))) {
        cta_copy<ESZ, U, LS>(dp, (ctl & kCtlWrite) ? sp : nullptr, len, tid, nt);
      }
      g += len;
    }
  }
}

// The shard-grid walker for non-uniform directories (ragged CSR inserts,
// duplicates / flattens / r/w of ragged arrays): blockIdx.y = shard,
// blockIdx.x = tile of that shard's work, so a tile never searches the
// directory and never crosses a shard (CTAs past a shard's end exit at
// once).  Tiles are aligned to the DESTINATION: tile 0 first stores the h
// head elements up to the first 16 B boundary of the destination, every
// tile then moves U x 256 full 16 B destination vectors.  When the source is
// congruent with the destination the loads are plain 16 B vectors; when not
// (a shard's CSR batch or committed range starting at another offset mod 16
// B than its destination) each warp loads a window of 32 consecutive aligned
// source vectors (every lane resolving its own bucket) and writes the 31
// output vectors it fully holds, each assembled by a funnel shift from its
// own load and the next lane's.  Source/destination positions: INSERT flat
// src[dir[s] + k] -> bucket size[s] + k (planned); DUP bucket k -> bucket
// size[s] + k (planned); FLATTEN bucket k -> flat dst[dir[s] + k]; RW bucket k
// in place.
template <int ESZ, int W, typename T, int U>
__device__ __forceinline__ void walk_shard_body(const Tables &t, const char *flat_src, char *flat_dst, T addend,
                                           uint32_t reps) {
  typedef typename ElemT<ESZ>::T E;
  constexpr uint32_t VE = 16 / ESZ, TL = U * 256 * VE;
  constexpr uint32_t LGE = ESZ == 1 ? 0 : ESZ == 2 ? 1 : ESZ == 4 ? 2 : 3;
  typedef LdSt<W == W_RW ? 2 : kDefLS> M;
  __shared__ char *scb[kMaxBuckets];
  pdl_begin();
  const uint32_t s = blockIdx.y, i = blockIdx.x, tid = threadIdx.x, lane = tid & 31;
  const uint64_t *dirp = W == W_INSERT ? t.offsets : t.prefix;
  const uint64_t lo = dirp[s], hi = dirp[s + 1];
  uint64_t dbase = 0;
  if constexpr (W == W_INSERT || W == W_DUP) dbase = t.size[s];   // planned: the append starts at size[s]
  const uint64_t len = hi - lo;
  // head elements before the destination's first 16 B boundary (buckets are
  // 16 B aligned and hold multiples of 16 B: fb * ESZ >= 16 is required)
  uint32_t h;
  if constexpr (W == W_FLATTEN) h = (uint32_t)(((16 - ((uintptr_t)(flat_dst + lo * ESZ) & 15)) & 15) / ESZ);
  else h = (uint32_t)((VE - dbase % VE) % VE);
  const uint64_t kb = h + (uint64_t)i * TL;                         // first body element of the tile
  if (kb >= len && !(i == 0 && len)) return;
  stage_cbase(t, scb);
  __syncthreads();
  const uint32_t lg0 = t.log2fb + LGE;
  // element addresses
  auto src_at = [&](uint64_t k) -> char * {
    if constexpr (W == W_INSERT) {
      return (char *)flat_src + (lo + k) * ESZ;
    } else {
      uint32_t b; uint64_t o;
      locate(k, t.log2fb, b, o);
      return slot_addr(scb, s, b, lg0) + o * ESZ;
    }
  };
  auto dst_at = [&](uint64_t k) -> char * {
    if constexpr (W == W_FLATTEN) {
      return flat_dst + (lo + k) * ESZ;
    } else if constexpr (W == W_RW) {
      return src_at(k);
    } else {
      uint32_t b; uint64_t o;
      locate(dbase + k, t.log2fb, b, o);
      return slot_addr(scb, s, b, lg0) + o * ESZ;
    }
  };
  auto elem = [&](uint64_t k) {
    if constexpr (W == W_RW) {
      T *p = (T *)src_at(k);
      T x = *p;
      for (uint32_t r = 0; r < reps; ++r) x = AddOp<T>::apply(x, addend);
      *p = x;
    } else {
      *(E *)dst_at(k) = *(const E *)src_at(k);
    }
  };
  // head (tile 0) and tail (last tile): element by element
  if (i == 0)
    for (uint64_t k = tid; k < min((uint64_t)h, len); k += 256) elem(k);
  if (kb >= len) return;
  const uint64_t ke = min(len, kb + TL);
  const uint32_t nv = (uint32_t)((ke - kb) / VE);
  for (uint64_t k = kb + (uint64_t)nv * VE + tid; k < ke; k += 256) elem(k);
  if (!nv) return;
  // source position (element index in the source's own space) of body element k
  const uint32_t sig = W == W_INSERT ? (uint32_t)(((uintptr_t)(flat_src + (lo + kb) * ESZ) & 15) / ESZ)
                                     : (uint32_t)(kb % VE);
  if (sig == 0) {
    for (uint32_t v0 = tid; v0 < nv; v0 += U * 256) {
      uint4 r[U];
      char *sp[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        sp[u] = src_at(kb + (uint64_t)min(v0 + u * 256u, nv - 1) * VE);
        r[u] = M::ld((const uint4 *)sp[u]);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t v = v0 + u * 256u;
        if (v >= nv) continue;
        if constexpr (W == W_RW) {
          union { uint4 q; T e[VE]; } x;
          x.q = r[u];
          for (uint32_t rr = 0; rr < reps; ++rr)
#pragma unroll
            for (uint32_t j = 0; j < VE; ++j) x.e[j] = AddOp<T>::apply(x.e[j], addend);
          M::st((uint4 *)sp[u], x.q);
        } else {
          M::st((uint4 *)dst_at(kb + (uint64_t)v * VE), r[u]);
        }
      }
    }
    return;
  }
  if constexpr (W != W_RW) {
    // non-congruent source: windows of 32 aligned source vectors -> 31 outputs
    const uint64_t k0 = kb - sig;                    // body-relative: aligned source vector j holds k0 + j * VE ..
    const uint32_t m = sig * ESZ, q = m >> 2, rsh = (m & 3) * 8;
    const uint32_t nw = (uint32_t)(blockDim.x >> 5), wid = tid >> 5;
    constexpr int UR = U > 4 ? 4 : U;       // (8 in flight: 76-80 registers, 3 CTAs per SM, slower)
    for (uint32_t w0 = wid; 31 * w0 < nv; w0 += UR * nw) {
      uint4 a[UR];
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        const uint32_t j = min(31 * (w0 + u * nw) + lane, nv);        // aligned source vector (clamped)
        if constexpr (W == W_INSERT) {
          a[u] = M::ld((const uint4 *)(flat_src + (lo + k0) * ESZ) + j);
        } else {
          a[u] = M::ld((const uint4 *)src_at(k0 + (uint64_t)j * VE));
        }
      }
#pragma unroll
      for (int u = 0; u < UR; ++u) {
        uint4 hn;
        hn.x = __shfl_down_sync(0xffffffffu, a[u].x, 1);
        hn.y = __shfl_down_sync(0xffffffffu, a[u].y, 1);
        hn.z = __shfl_down_sync(0xffffffffu, a[u].z, 1);
        hn.w = __shfl_down_sync(0xffffffffu, a[u].w, 1);
        const uint32_t v = 31 * (w0 + u * nw) + lane;
        if (lane < 31 && v < nv) M::st((uint4 *)dst_at(kb + (uint64_t)v * VE), realign16(a[u], hn, q, rsh));
      }
    }
  }
}

template <int ESZ, int W, typename T, int U>
__global__ void __launch_bounds__(256) k_walk_shard(Tables t, const char *flat_src, char *flat_dst, T addend,
                                                    uint32_t reps) {
  walk_shard_body<ESZ, W, T, U>(t, flat_src, flat_dst, addend, reps);
}
// the duplicate (bucket -> bucket, both located per vector) capped at 40
// registers: 6 CTAs per SM instead of 4 (ragged duplicate 0.82 -> 0.89 of HBM)
template <int ESZ, int W, typename T, int U>
__global__ void __launch_bounds__(256, 6) k_walk_shard_dup(Tables t, const char *flat_src, char *flat_dst, T addend,
                                                           uint32_t reps) {
  walk_shard_body<ESZ, W, T, U>(t, flat_src, flat_dst, addend, reps);
}

// Metadata of a planned append (launched right behind its copy walk, PDL):
// one size update per LFVector (the reference's single fetch_add per batch),
// bucket publication (flag, ptr, pmask, cap) and, if asked, the commit scan.
__global__ void __launch_bounds__(1024) k_planned_meta(Tables t, Fuse fz) {
  __shared__ char *scb[kMaxBuckets];
  pdl_begin();
  stage_cbase(t, scb);
  __syncthreads();
  planned_metadata(t, scb, fz);
}

// A deferred planned-append metadata pass fused with the grow that follows it
// (the doubling schedule's grow(2n) after every duplicate): one launch, the
// metadata first, then buckets [0, uk) of every shard published.
__global__ void __launch_bounds__(1024) k_meta_grow(Tables t, Fuse fz, uint32_t uk) {
  __shared__ char *scb[kMaxBuckets];
  pdl_begin();
  stage_cbase(t, scb);
  __syncthreads();
  planned_metadata(t, scb, fz);
  __syncthreads();
  const uint32_t lg0 = t.log2fb + (31u - __clz(t.esz));
  const unsigned long long all = uk >= 64 ? ~0ull : ((1ull << uk) - 1ull);
  for (uint32_t base = 0; base < t.S; base += blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    const bool live = s < t.S;
    const unsigned long long pm = live ? t.pmask[s] : 0ull;
    publish_buckets_cta<1024>(t, scb, base, pm, live ? (all & ~pm) : 0ull, lg0);
  }
}

// rw_g (bench_cli.py:339-366, the paper's rw_g): every 16 B group of
// consecutive GLOBAL indices is resolved through the directory on its own --
// a warp-uniform bisect on the smem prefix for the chunk, a per-lane fix-up
// and a clz locate -- and each thread keeps kDefUnroll such vectors in flight.
// Groups that straddle a shard or are not 16 B-aligned inside their bucket
// are updated element by element.
template <typename T, int U = kDefUnroll>
__global__ void __launch_bounds__(kThreads) k_rw_global(Tables t, uint64_t total, T addend) {
  pdl_begin();
  __shared__ char *scb[kMaxBuckets];
  stage_cbase(t, scb);
  __syncthreads();
  const uint64_t *pre = t.prefix;
  constexpr uint32_t LGE = sizeof(T) == 1 ? 0 : sizeof(T) == 2 ? 1 : sizeof(T) == 4 ? 2 : 3;
  const uint32_t lg0 = t.log2fb + LGE;
  constexpr uint32_t VE = 16 / sizeof(T);
  
  typedef LdSt<kDefLS == 1 ? 2 : kDefLS> M;
  const uint64_t nvec = (total + VE - 1) / VE;
  const uint32_t lane = threadIdx.x & 31;
  const uint64_t nwarps = ((uint64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t wid = ((uint64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  for (uint64_t c0 = wid * 32 * U; c0 < nvec; c0 += nwarps * 32 * U) {
    uint32_t s = warp_find_shard(pre, t.S, c0 * VE);  // warp-uniform 32-ary search
    {
      // warp-uniform fast path: the warp's 32*U vectors resolve (global index
      // -> shard -> bucket) to one aligned run inside one bucket of shard s --
      // one locate for the span instead of one per vector
      const uint64_t g0 = c0 * VE, span = 32ull * U * VE;
      const uint64_t lo = pre[s], hi = pre[s + 1];
      uint32_t b0; uint64_t o0;
      locate(g0 - lo, t.log2fb, b0, o0);
      if (g0 + span <= hi && (o0 % VE) == 0 && o0 + span <= (1ull << (t.log2fb + b0))) {
        T *base = (T *)slot_addr(scb, s, b0, lg0) + o0;
        uint4 r[U];
#pragma unroll
        for (int u = 0; u < U; ++u) r[u] = M::ld((const uint4 *)(base + (size_t)(lane + 32u * u) * VE));
#pragma unroll
        for (int u = 0; u < U; ++u) {
          union { uint4 q; T e[VE]; } x;
          x.q = r[u];
#pragma unroll
          for (uint32_t j = 0; j < VE; ++j) x.e[j] = AddOp<T>::apply(x.e[j], addend);
          M::st((uint4 *)(base + (size_t)(lane + 32u * u) * VE), x.q);
        }
        continue;
      }
    }
    uint4 r[U];
    T *p[U];
    bool vec[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = c0 + lane + 32u * u;
      const uint64_t g = v * VE;
      vec[u] = false;
      p[u] = nullptr;
      if (v < nvec) {
        while (pre[s + 1] <= g) ++s;
        uint32_t b; uint64_t o;
        locate(g - pre[s], t.log2fb, b, o);
        p[u] = (T *)slot_addr(scb, s, b, lg0) + o;
        vec[u] = g + VE <= pre[s + 1] && (o % VE) == 0 && o + VE <= (1ull << (t.log2fb + b));
        if (vec[u]) r[u] = M::ld((const uint4 *)p[u]);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t v = c0 + lane + 32u * u;
      if (v >= nvec) continue;
      if (vec[u]) {
        union { uint4 q; T e[VE]; } x;
        x.q = r[u];
#pragma unroll
        for (uint32_t j = 0; j < VE; ++j) x.e[j] = AddOp<T>::apply(x.e[j], addend);
        M::st((uint4 *)p[u], x.q);
      } else {
        const uint64_t g = v * VE;
        uint32_t sj = upper_shard(pre, t.S, g);
        for (uint32_t j = 0; j < VE && g + j < total; ++j) {
          const uint64_t gj = g + j;
          while (pre[sj + 1] <= gj) ++sj;
          uint32_t b; uint64_t o;
          locate(gj - pre[sj], t.log2fb, b, o);
          T *q = (T *)slot_addr(scb, sj, b, lg0) + o;
          *q = AddOp<T>::apply(*q, addend);
        }
      }
    }
  }
}

// get_many / set_many (sharded_array.py:152-158 batched): the directory
// prefix[S+1] staged in shared memory (SMEM, S < 4096) so the bisect of each
// index costs shared-memory loads, bucket addresses by slot arithmetic, and
// U independent indices per thread so their random element accesses are in
// flight together (the kernel is bound by random 32 B sectors, not by the
// directory chain).
constexpr int kGatherU = 4;                      // indices per thread (independent chains)

// the random element read of the gather, by cache policy (ldm, uniform):
// 0 = default (L1-allocating: ncu showed 4 L2 sectors = a 128 B line
// requested per random 4 B element), 1 = .cg (L2 only), 2 =
// .L1::no_allocate, 3 = .nc.L1::no_allocate, 4 = .cs
#define GG_LDR(Q, T, R)                                                                            \
  if (ldm == 1) asm volatile("ld.global.cg." T " %0, [%1];" : "=" R(v) : "l"(p));                   \
  else if (ldm == 2) asm volatile("ld.global.L1::no_allocate." T " %0, [%1];" : "=" R(v) : "l"(p)); \
  else if (ldm == 3) asm volatile("ld.global.nc.L1::no_allocate." T " %0, [%1];" : "=" R(v) : "l"(p)); \
  else if (ldm == 4) asm volatile("ld.global.cs." T " %0, [%1];" : "=" R(v) : "l"(p));              \
  else v = (Q)*p;
template <int ESZ>
__device__ __forceinline__ typename ElemT<ESZ>::T ld_rand(const typename ElemT<ESZ>::T *p, int ldm) {
  typedef typename ElemT<ESZ>::T E;
  if constexpr (ESZ == 8) {
    unsigned long long v;
    GG_LDR(unsigned long long, "u64", "l")
    return (E)v;
  } else {
    uint32_t v;
    if constexpr (ESZ == 4) { GG_LDR(uint32_t, "u32", "r") }
    else if constexpr (ESZ == 2) { GG_LDR(uint16_t, "u16", "r") }
    else { GG_LDR(uint8_t, "u8", "r") }
    return (E)v;
  }
}
#undef GG_LDR

template <int ESZ, bool SMEM, int U = kGatherU>
__global__ void __launch_bounds__(256) k_gather(Tables t, const int64_t *idx, uint64_t n, char *out,
                                                const char *vals, int scatter, int ldm, uint64_t lim,
                                                unsigned int *bad) {
  typedef typename ElemT<ESZ>::T E;
  extern __shared__ uint64_t sdir[];
  __shared__ char *scb[kMaxBuckets];
  pdl_begin();
  // checked scatter: k_check_idx (the predecessor) flagged a bad index -> no writes at all
  if (scatter && bad && *(volatile unsigned int *)bad) return;
  stage_cbase(t, scb);
  if constexpr (SMEM)
    for (uint32_t i = threadIdx.x; i <= t.S; i += blockDim.x) sdir[i] = t.prefix[i];
  __syncthreads();
  const uint64_t *dir = SMEM ? sdir : t.prefix;
  const uint32_t lg0 = t.log2fb + (ESZ == 1 ? 0 : ESZ == 2 ? 1 : ESZ == 4 ? 2 : 3);
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x * U;
  for (uint64_t j0 = (uint64_t)blockIdx.x * blockDim.x * U + threadIdx.x; j0 < n; j0 += stride) {
    E *p[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint64_t j = j0 + (uint64_t)u * blockDim.x;
      uint64_t g = j < n ? (uint64_t)__ldcs(idx + j) : 0;
      if (!scatter && bad && g >= lim) {                      // checked gather: flag it, read element 0
        *bad = 1u;                                // (lim > 0; the call fails with GG_EINDEX)
        g = 0;
      }
      const uint32_t s = upper_shard(dir, t.S, g);
      uint32_t b; uint64_t o;
      locate(g - dir[s], t.log2fb, b, o);
      p[u] = (E *)slot_addr(scb, s, b, lg0) + o;
    }
    if (scatter) {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t j = j0 + (uint64_t)u * blockDim.x;
        if (j < n) *p[u] = ((const E *)vals)[j];
      }
    } else {
      E v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = j0 + (uint64_t)u * blockDim.x < n ? ld_rand<ESZ>(p[u], ldm) : E(0);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint64_t j = j0 + (uint64_t)u * blockDim.x;
        if (j < n) ((E *)out)[j] = v[u];
      }
    }
  }
}

// bounds pass of the checked scatter: flag any index outside [0, lim)
// (negative int64 indices are huge as uint64); the scatter behind it skips
// every write when the flag is set
__global__ void __launch_bounds__(256) k_check_idx(const int64_t *idx, uint64_t n, uint64_t lim,
                                                   unsigned int *bad) {
  pdl_begin();
  bool oob = false;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
#pragma unroll 4
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride)
    oob |= (uint64_t)__ldcs(idx + j) >= lim;
  if (__any_sync(0xffffffffu, oob) && (threadIdx.x & 31) == 0) *bad = 1u;
}

// zero whole buckets listed as (shard, bucket) pairs (dirty shards only)
__global__ void k_zero_buckets(Tables t, const uint32_t *pairs, uint32_t npairs) {
  for (uint32_t k = blockIdx.x; k < npairs; k += gridDim.x) {
    uint32_t s = pairs[2 * k], b = pairs[2 * k + 1];
    char *p = t.ptr[(size_t)s * t.MB + b];
    uint64_t n = (1ull << (t.log2fb + b)) * t.esz;
    if (t.flag[(size_t)s * t.MB + b] != kFlagPublished) continue;
    cta_copy<1, 4>(p, nullptr, n, threadIdx.x, blockDim.x);
  }
}

// ---- static-array baselines ---------------------------------------------------
// Flat-array insert_batch with the reference's semantics (baselines.py:59-72,
// 143-157, 224-236): ONE reservation of the whole batch, then an
// argument-order copy to [start, start + n).  The reservation is the host's
// (single host thread per array: `start` = the mirrored counter); CTA 0
// publishes it on the device counter.  The copy is the walker's tile shape:
// one tile of 256 threads x U 16 B vectors per CTA, all U loads issued
// before the stores (cta_copy handles any relative alignment).
// ---- paper Alg. 1 at throughput: the tiled lanes insert --------------------
// The lanes of shard s ([offsets[s], offsets[s+1])) are cut into tiles of T
// consecutive lanes that never cross a shard; tpre[s] = first tile of shard
// s (tpre[S] = number of tiles).  Three launches, no host round trip (the
// host backed the slots for the upper bound lanes x values_per_lane):
//   k_lanes_sum:     a warp per tile sums its lanes' counts (coalesced) and
//                    records the tile (shard, first lane, lanes, sum);
//   k_lanes_reserve: a CTA per shard scans its tile sums (tile order = lane
//                    order), reserves the whole batch with ONE atomicAdd on
//                    the LFVector size (insert_index.py:118-143), publishes
//                    the buckets the range covers (paper Alg. 2) and turns
//                    the sums into absolute destination indices;
//   k_lanes_scatter: a CTA per tile loads its [T x K] block of values with
//                    coalesced 16 B loads and its counts, block-scans the
//                    counts, compacts the valid values into shared memory
//                    (lane order) and stores them as aligned 16 B vectors
//                    through the bucket slots.
struct LaneTile {
  uint64_t base;      // sum of the tile's counts -> absolute destination index
  uint64_t lane_lo;   // first lane of the tile
  uint32_t shard, nl; // shard, lanes in the tile
  uint32_t pad[2];
};

// largest s with tpre[s] <= x (tiles of empty shards skipped), 32-ary warp
// search; called by a full warp, result in every lane
__device__ __forceinline__ uint32_t warp_find_u32(const uint32_t *tpre, uint32_t S, uint32_t x) {
  const uint32_t lane = threadIdx.x & 31;
  uint32_t lo = 0, hi = S;
  while (hi - lo > 1) {
    const uint32_t step = (hi - lo + 31) >> 5;
    const uint32_t p = lo + lane * step;
    const bool ok = p < hi && tpre[p] <= x;
    const unsigned m = __ballot_sync(0xffffffffu, ok);
    lo = lo + (31u - __clz(m)) * step;
    hi = min(hi, lo + step);
  }
  return lo;
}

__global__ void __launch_bounds__(256) k_lanes_sum(Tables t, const uint32_t *counts, const uint32_t *tpre,
                                                   LaneTile *tiles, uint32_t ntiles, uint32_t T, uint32_t K) {
  pdl_begin();
  const uint32_t lane = threadIdx.x & 31;
  const uint32_t tile = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (tile >= ntiles) return;
  const uint32_t s = warp_find_u32(tpre, t.S, tile);
  const uint64_t lo = t.offsets[s] + (uint64_t)(tile - tpre[s]) * T;
  const uint32_t nl = (uint32_t)min((uint64_t)T, t.offsets[s + 1] - lo);
  uint32_t acc = 0;
#pragma unroll 8
  for (uint32_t j = lane; j < nl; j += 32) acc += min(__ldcs(counts + lo + j), K);
  acc = __reduce_add_sync(0xffffffffu, acc);
  if (lane == 0) {
    LaneTile lt;
    lt.base = acc; lt.lane_lo = lo; lt.shard = s; lt.nl = nl; lt.pad[0] = lt.pad[1] = 0;
    tiles[tile] = lt;
  }
}

__global__ void __launch_bounds__(256) k_lanes_reserve(Tables t, const uint32_t *tpre, LaneTile *tiles) {
  __shared__ uint64_t ws[32];
  __shared__ uint64_t start_sh;
  pdl_begin();
  const uint32_t s = blockIdx.x, tid = threadIdx.x;
  const uint32_t first = tpre[s], nts = tpre[s + 1] - first;
  if (!nts) return;
  uint64_t carry = 0;
  for (uint32_t j0 = 0; j0 < nts; j0 += blockDim.x) {
    const uint32_t j = j0 + tid;
    const uint64_t v = j < nts ? tiles[first + j].base : 0;
    uint64_t ct;
    const uint64_t ex = block_exclusive_scan(v, &ct, ws);
    if (j < nts) tiles[first + j].base = carry + ex;
    carry += ct;
  }
  if (tid == 0) {
    uint64_t start = t.size[s];
    if (carry) {
      // the batch's reservation: ONE atomicAdd on the LFVector size
      start = atomicAdd((unsigned long long *)&t.size[s], (unsigned long long)carry);
      t.ops[s] += 1;
      uint32_t b0, b1; uint64_t o;
      locate(start, t.log2fb, b0, o);
      locate(start + carry - 1, t.log2fb, b1, o);
      const unsigned long long pm = t.pmask[s];
      const unsigned long long want = (b1 >= 63 ? ~0ull : ((2ull << b1) - 1ull)) & ~((1ull << b0) - 1ull) & ~pm;
      uint64_t add = 0;
      const uint32_t lg0 = t.log2fb + (31u - __clz(t.esz));
      for (unsigned long long mm = want; mm; mm &= mm - 1) {
        const uint32_t b = __ffsll((long long)mm) - 1;
        t.ptr[(size_t)s * t.MB + b] = t.cbase[b] + ((uint64_t)s << max(lg0 + b, 4u));
        t.flag[(size_t)s * t.MB + b] = kFlagPublished;
        add += 1ull << (t.log2fb + b);
      }
      if (want) {
        t.pmask[s] = pm | want;
        t.cap[s] += add;
        atomicAdd(&t.misc[MISC_ALLOCS], (unsigned long long)__popcll(want));
      }
    }
    t.start[s] = start;
    t.count[s] = carry;
    start_sh = start;
  }
  __syncthreads();
  const uint64_t start = start_sh;
  for (uint32_t j = tid; j < nts; j += blockDim.x) tiles[first + j].base += start;
}

// One tile of the lanes insert.  Every thread holds 64 B of values in
// registers: R rows of GL consecutive lanes (GL = 16 / KB lanes share one
// 16 B vector when a lane's values are narrower than 16 B, else GL = 1 and
// a lane is KB / 16 vectors), so counts and values move as 16 B (or 8 B)
// loads; consecutive threads hold consecutive groups (coalesced).  Warp
// scans of the per-row group totals (several rows packed into one 32-bit
// scan, 8- or 16-bit fields) give every group's offset in its warp's run;
// the whole run is staged in the warp's shared buffer congruent with its
// destination and leaves as aligned 16 B vector stores.  Lanes outside the
// valid range [vlo, vhi) count 0 (tiles start at a GL-aligned lane so the
// groups are aligned; only the edge groups take per-lane loads).  One
// __syncthreads per tile (the warps' totals, double-buffered by `par`).
template <int ESZ, int KB, bool VEC = true>
struct LaneShape {
  static constexpr uint32_t K = KB / ESZ, GL = (VEC && KB < 16) ? 16 / KB : 1, R = 64 / (KB * GL),
                            T = 256 * GL * R, VE = 16 / ESZ, WPR = GL * KB / 4;   // words per row
};

template <int ESZ, int KB, bool VEC = true>
struct LaneSmem {
  typedef typename ElemT<ESZ>::T E;
  typedef LaneShape<ESZ, KB, VEC> L;
  __align__(16) E stage[8][32 * L::R * L::GL * L::K + 2 * L::VE];
  uint32_t wsum[2][8];
  char *scb[kMaxBuckets];
  unsigned long long base;
};

// lane j's KB bytes of values into w[0 .. KB/4) (KB a power of two in [4, 64])
template <int KB>
__device__ __forceinline__ void lane_load(uint32_t *w, const char *p) {
  if constexpr (KB >= 16) {
#pragma unroll
    for (int i = 0; i < KB / 16; ++i) {
      const uint4 v = ldg_stream((const uint4 *)p + i);
      w[4 * i] = v.x; w[4 * i + 1] = v.y; w[4 * i + 2] = v.z; w[4 * i + 3] = v.w;
    }
  } else if constexpr (KB == 8) {
    const uint2 v = __ldcs((const uint2 *)p);
    w[0] = v.x; w[1] = v.y;
  } else {
    w[0] = __ldcs((const uint32_t *)p);
  }
}

template <int ESZ, int KB, bool VEC = true>
__device__ __forceinline__ void lanes_load(const char *vals, const uint32_t *counts, uint64_t wlo, uint64_t vlo,
                                           uint64_t vhi,
                                           uint32_t (&c)[LaneShape<ESZ, KB, VEC>::R][LaneShape<ESZ, KB, VEC>::GL],
                                           uint32_t (&w)[16]) {
  typedef LaneShape<ESZ, KB, VEC> L;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  {
    // interior thread (every row's group inside [vlo, vhi), GL-aligned since
    // wlo is): all rows' loads issue before any is consumed -- a per-row
    // bounds branch around load + use would serialise them
    const uint64_t ga = wlo + ((uint64_t)(wid * L::R) * 32 + lane) * L::GL;
    const uint64_t gz = wlo + ((uint64_t)(wid * L::R + L::R - 1) * 32 + lane) * L::GL;
    if (ga >= vlo && gz + L::GL <= vhi && (L::GL == 1 || ga % L::GL == 0)) {
      uint32_t cr[L::R][L::GL];
#pragma unroll
      for (uint32_t r = 0; r < L::R; ++r) {
        const uint64_t g0 = ga + (uint64_t)r * 32 * L::GL;
        if constexpr (L::GL == 4) {
          const uint4 x = __ldcs((const uint4 *)(counts + g0));
          cr[r][0] = x.x; cr[r][1] = x.y; cr[r][2] = x.z; cr[r][3] = x.w;
        } else if constexpr (L::GL == 2) {
          const uint2 x = __ldcs((const uint2 *)(counts + g0));
          cr[r][0] = x.x; cr[r][1] = x.y;
        } else {
          cr[r][0] = __ldcs(counts + g0);
        }
        lane_load<L::GL * KB>(w + r * L::WPR, vals + g0 * KB);
      }
#pragma unroll
      for (uint32_t r = 0; r < L::R; ++r)
#pragma unroll
        for (uint32_t g = 0; g < L::GL; ++g) c[r][g] = min(cr[r][g], L::K);
      return;
    }
  }
#pragma unroll
  for (uint32_t r = 0; r < L::R; ++r) {
    const uint64_t g0 = wlo + ((uint64_t)(wid * L::R + r) * 32 + lane) * L::GL;
    uint32_t *wr = w + r * L::WPR;
    if (g0 >= vlo && g0 + L::GL <= vhi && (L::GL == 1 || g0 % L::GL == 0)) {
      if constexpr (L::GL == 4) {
        const uint4 x = __ldcs((const uint4 *)(counts + g0));
        c[r][0] = min(x.x, L::K); c[r][1] = min(x.y, L::K); c[r][2] = min(x.z, L::K); c[r][3] = min(x.w, L::K);
      } else if constexpr (L::GL == 2) {
        const uint2 x = __ldcs((const uint2 *)(counts + g0));
        c[r][0] = min(x.x, L::K); c[r][1] = min(x.y, L::K);
      } else {
        c[r][0] = min(__ldcs(counts + g0), L::K);
      }
      lane_load<L::GL * KB>(wr, vals + g0 * KB);
    } else {
#pragma unroll
      for (uint32_t g = 0; g < L::GL; ++g) {
        c[r][g] = 0;
        if (g0 + g >= vlo && g0 + g < vhi) {
          c[r][g] = min(__ldcs(counts + g0 + g), L::K);
          lane_load<KB>(wr + g * (KB / 4), vals + (g0 + g) * KB);
        }
      }
    }
  }
}

// scans + staging + stores of a loaded tile; returns the tile total
struct NoSyncHook { __device__ void operator()() const {} };

template <int ESZ, int KB, bool VEC = true, typename OnSync = NoSyncHook>
__device__ __forceinline__ uint32_t lanes_store(const Tables &t, LaneSmem<ESZ, KB, VEC> &sm, uint32_t s,
                                                const uint32_t (&c)[LaneShape<ESZ, KB, VEC>::R][LaneShape<ESZ, KB, VEC>::GL],
                                                const uint32_t (&w)[16], uint64_t base, int par,
                                                OnSync on_sync = OnSync()) {
  typedef typename ElemT<ESZ>::T E;
  typedef LaneShape<ESZ, KB, VEC> L;
  constexpr uint32_t R = L::R, GL = L::GL, K = L::K, VE = L::VE;
  constexpr uint32_t FW = (32 * GL * K < 256) ? 8 : 16, PF = 32 / FW, FM = (1u << FW) - 1;
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  uint32_t ex[R];
  uint32_t carry = 0;
#pragma unroll
  for (uint32_t r0 = 0; r0 < R; r0 += PF) {
    uint32_t x = 0;
#pragma unroll
    for (uint32_t f = 0; f < PF; ++f)
      if (r0 + f < R) {
        uint32_t cr = 0;
#pragma unroll
        for (uint32_t g = 0; g < GL; ++g) cr += c[r0 + f][g];
        x |= cr << (f * FW);
      }
    const uint32_t v = x;
#pragma unroll
    for (int d = 1; d < 32; d <<= 1) {
      const uint32_t y = __shfl_up_sync(0xffffffffu, x, d);
      if (lane >= (uint32_t)d) x += y;
    }
    const uint32_t tot = __shfl_sync(0xffffffffu, x, 31);
    const uint32_t xe = x - v;
#pragma unroll
    for (uint32_t f = 0; f < PF; ++f) {
      if (r0 + f < R) {
        ex[r0 + f] = carry + ((xe >> (f * FW)) & FM);
        carry += (tot >> (f * FW)) & FM;
      }
    }
  }
  if (lane == 0) sm.wsum[par][wid] = carry;
  __syncthreads();
  on_sync();                                    // (every thread holds its tile in registers)
  uint32_t woff = 0, total = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) {
    const uint32_t x = sm.wsum[par][q];
    if (q < (int)wid) woff += x;
    total += x;
  }
  const uint32_t run = carry;
  if (run) {
    const uint64_t rb = base + woff;              // destination index of the warp's run
    E *st = sm.stage[wid];
    const uint32_t lg0 = t.log2fb + (ESZ == 1 ? 0 : ESZ == 2 ? 1 : ESZ == 4 ? 2 : 3);
    const bool vec = (1u << lg0) >= 16;           // 16 B vectors never straddle a bucket
    const uint32_t shift = vec ? (uint32_t)(rb % VE) : 0u;
#pragma unroll
    for (uint32_t r = 0; r < R; ++r) {
      const E *ev = (const E *)(w + r * L::WPR);
      uint32_t o = shift + ex[r];
#pragma unroll
      for (uint32_t g = 0; g < GL; ++g) {
#pragma unroll
        for (uint32_t k = 0; k < K; ++k)
          if (k < c[r][g]) st[o + k] = ev[g * K + k];
        o += c[r][g];
      }
    }
    __syncwarp();
    if (vec) {
      const uint32_t nv = (shift + run + VE - 1) / VE;
      // the warp's run (warp-uniform) usually lies in ONE bucket: its slot
      // address is computed once and each vector is an offset from it (4 / 8 B
      // elements: K16 int32 0.68 -> 0.71, K8 0.79 -> 0.80 of HBM; for 1 / 2 B
      // elements the extra live registers cost more than the locates)
      uint32_t bf = 0, bl = 1; uint64_t of = 0, ol;
      if constexpr (ESZ >= 4) {
        locate(rb - shift, t.log2fb, bf, of);
        locate(rb + run - 1, t.log2fb, bl, ol);
      }
      E *const rbase = (E *)(slot_addr(sm.scb, s, bf, lg0) + of * ESZ);
      for (uint32_t v = lane; v < nv; v += 32) {
        E *dp;
        if (ESZ >= 4 && bf == bl) {
          dp = rbase + v * VE;
        } else {
          uint32_t b; uint64_t o;
          locate(rb - shift + (uint64_t)v * VE, t.log2fb, b, o);
          dp = (E *)(slot_addr(sm.scb, s, b, lg0) + o * ESZ);
        }
        const uint32_t k0 = v * VE;
        if (k0 >= shift && k0 + VE <= shift + run) {
          stg((uint4 *)dp, ((const uint4 *)st)[v]);
        } else {
#pragma unroll
          for (uint32_t j = 0; j < VE; ++j)
            if (k0 + j >= shift && k0 + j < shift + run) dp[j] = st[k0 + j];
        }
      }
    } else {
      for (uint32_t k = lane; k < run; k += 32) {
        uint32_t b; uint64_t o;
        locate(rb + k, t.log2fb, b, o);
        ((E *)(slot_addr(sm.scb, s, b, lg0)))[o] = st[k];
      }
    }
    __syncwarp();                                 // the stage buffer is reused by the next tile
  }
  return total;
}

// the batch's reservation (ONE atomicAdd on the LFVector size,
// insert_index.py:118-143) and the publication of the buckets [start, end)
// covers (paper Alg. 2; the host backed the slots for the upper bound)
__device__ __forceinline__ void lanes_reserve_publish(const Tables &t, uint32_t s, uint64_t start,
                                                      uint64_t total) {
  if (total) {
    atomicAdd((unsigned long long *)&t.size[s], (unsigned long long)total);
    t.ops[s] += 1;
    uint32_t b0, b1; uint64_t o;
    locate(start, t.log2fb, b0, o);
    locate(start + total - 1, t.log2fb, b1, o);
    const unsigned long long pm = t.pmask[s];
    const unsigned long long want = (b1 >= 63 ? ~0ull : ((2ull << b1) - 1ull)) & ~((1ull << b0) - 1ull) & ~pm;
    uint64_t add = 0;
    const uint32_t lg0 = t.log2fb + (31u - __clz(t.esz));
    for (unsigned long long mm = want; mm; mm &= mm - 1) {
      const uint32_t b = __ffsll((long long)mm) - 1;
      t.ptr[(size_t)s * t.MB + b] = t.cbase[b] + ((uint64_t)s << max(lg0 + b, 4u));
      t.flag[(size_t)s * t.MB + b] = kFlagPublished;
      add += 1ull << (t.log2fb + b);
    }
    if (want) {
      t.pmask[s] = pm | want;
      t.cap[s] += add;
      atomicAdd(&t.misc[MISC_ALLOCS], (unsigned long long)__popcll(want));
    }
  }
  t.start[s] = start;
  t.count[s] = total;
}

// k_lanes_scatter: the 3-pass path's last pass, one tile per CTA at the
// destination k_lanes_reserve computed (GG_LANES_CHAIN=0, A/B)
template <int ESZ, int KB>
__global__ void __launch_bounds__(256) k_lanes_scatter(Tables t, const char *vals, const uint32_t *counts,
                                                       const LaneTile *tiles) {
  __shared__ LaneSmem<ESZ, KB> sm;
  pdl_begin();
  const LaneTile lt = tiles[blockIdx.x];
  uint32_t c[LaneShape<ESZ, KB>::R][LaneShape<ESZ, KB>::GL], w[16];
  lanes_load<ESZ, KB>(vals, counts, lt.lane_lo, lt.lane_lo, lt.lane_lo + lt.nl, c, w);
  stage_cbase(t, sm.scb);
  lanes_store<ESZ, KB>(t, sm, lt.shard, c, w, lt.base, 0);
}

// ---- paper Alg. 1 in ONE pass over HBM: the chunked lanes insert ----------
// The lanes of shard s are cut into chunks of C lanes (a multiple of the
// tile) that never cross a shard; cpre[s] = first chunk of shard s.  A CTA
// per chunk:
//   1. sums the chunk's counts (16 B loads, many in flight; the chunk's
//      counts -- 64 KiB -- stay in L2 for step 3, so HBM sees them once);
//   2. chains the chunk sums of its shard with a decoupled look-back: the
//      first chunk reads the LFVector size (the batch's start) and publishes
//      start + its sum as an INCLUSIVE prefix, every other chunk publishes
//      its sum as an AGGREGATE at once and warp 0 looks back over its
//      shard's predecessors (32 status words per step) to an inclusive
//      prefix, then publishes its own; chunks are CTA indices, dispatched in
//      order, so every chunk waited on is already running;
//   3. walks its tiles in order (register-resident values, warp runs staged
//      in shared memory, 16 B vector stores) from that destination;
//   4. the last chunk of the shard holds start + total: it makes the
//      batch's reservation -- ONE atomicAdd on the LFVector size -- and
//      publishes the buckets (tiles write through slot arithmetic, which
//      does not depend on the publication).
// Status word: flag in bits 62-63 (1 = aggregate, 2 = inclusive), value below.
// lanes per chunk: 64 KiB of counts (L2-resident between steps 1 and 3); 4 B lanes run
// 6 CTAs per SM (more tiles in flight: 0.57 -> 0.64 of HBM at K = 1 int32)
constexpr uint32_t kLanesChunk = 16384;

// TMA bulk prefetch of [p, p + bytes) into L2 (a hint: no completion, no
// destination); p 16 B aligned, bytes a multiple of 16 (rounded down here)
__device__ __forceinline__ void prefetch_l2(const void *p, uint32_t bytes) {
  bytes &= ~15u;
  if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(p), "r"(bytes) : "memory");
}
constexpr unsigned long long kChainA = 1ull << 62, kChainP = 2ull << 62, kChainV = (1ull << 62) - 1;

__device__ __forceinline__ unsigned long long ld_chain(const unsigned long long *p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_chain(unsigned long long *p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

// sum of min(counts[lo + j], K) over j < n, by the whole CTA (result in every thread)
__device__ __forceinline__ uint32_t chunk_count_sum(const uint32_t *counts, uint64_t lo, uint32_t n, uint32_t K,
                                                    uint32_t *red) {
  const uint32_t tid = threadIdx.x;
  uint32_t acc = 0;
  const uint32_t head = (uint32_t)min((uint64_t)n, (uint64_t)((4 - (lo & 3)) & 3));
  if (tid < head) acc += min(__ldcs(counts + lo + tid), K);
  const uint32_t nv = (n - head) >> 2;
  const uint4 *cv = (const uint4 *)(counts + lo + head);
#pragma unroll 4
  for (uint32_t v = tid; v < nv; v += 256) {
    const uint4 x = __ldcg(cv + v);               // kept in L2 for the tile walk
    acc += min(x.x, K) + min(x.y, K) + min(x.z, K) + min(x.w, K);
  }
  for (uint32_t j = head + 4 * nv + tid; j < n; j += 256) acc += min(__ldcs(counts + lo + j), K);
  acc = __reduce_add_sync(0xffffffffu, acc);
  if ((tid & 31) == 0) red[tid >> 5] = acc;
  __syncthreads();
  uint32_t tot = 0;
#pragma unroll
  for (int q = 0; q < 8; ++q) tot += red[q];
  return tot;
}

template <int ESZ, int KB, bool VEC = true>
__global__ void __launch_bounds__(256, KB == 4 ? 6 : 1) k_lanes_chunk(Tables t, const char *vals, const uint32_t *counts,
                                                     const uint32_t *cpre, unsigned long long *chain,
                                                     uint32_t C, uint32_t pf) {
  typedef LaneShape<ESZ, KB, VEC> L;
  constexpr uint32_t K = L::K, T = L::T;
  __shared__ LaneSmem<ESZ, KB, VEC> sm;
  __shared__ uint32_t red[8];
  pdl_begin();
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t chunk = blockIdx.x;
  const uint32_t s = warp_find_u32(cpre, t.S, chunk);
  const uint32_t first = cpre[s], last = cpre[s + 1] - 1;
  const uint64_t lo = t.offsets[s] + (uint64_t)(chunk - first) * C;
  const uint32_t nl = (uint32_t)min((uint64_t)C, t.offsets[s + 1] - lo);
  stage_cbase(t, sm.scb);
  // pf tiles ahead of the walk, the value block is prefetched into L2 by TMA
  // (the first pf tiles while the counts are summed and chained)
  const uint64_t wlo = lo - lo % L::GL;
  auto pf_tile = [&](uint64_t p0) {
    if (p0 < lo + nl) prefetch_l2(vals + p0 * KB, (uint32_t)(min((uint64_t)T, lo + nl - p0) * KB));
  };
  if (tid < pf) pf_tile(wlo + (uint64_t)tid * T);
  const uint32_t agg = chunk_count_sum(counts, lo, nl, K, red);
  if (wid == 0) {
    unsigned long long excl = 0;
    if (chunk == first) {
      if (lane == 0) {
        excl = t.size[s];                            // the batch's start (before any reservation)
        st_chain(chain + chunk, kChainP | (excl + agg));
      }
      excl = __shfl_sync(0xffffffffu, excl, 0);
    } else {
      if (lane == 0) st_chain(chain + chunk, kChainA | agg);
      int64_t j = (int64_t)chunk - 1;
      for (;;) {
        const int64_t idx = j - lane;
        unsigned long long v;
        do {                                         // wait until the window is published
          v = idx >= (int64_t)first ? ld_chain(chain + idx) : kChainP;
        } while (__any_sync(0xffffffffu, (v >> 62) == 0));
        const unsigned pm = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const uint32_t stop = pm ? (uint32_t)(__ffs(pm) - 1) : 31u;
        unsigned long long x = lane <= stop ? (v & kChainV) : 0ull;
#pragma unroll
        for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        excl += x;
        if (pm) break;
        j -= 32;
      }
      if (lane == 0) st_chain(chain + chunk, kChainP | (excl + agg));
    }
    if (lane == 0) {
      sm.base = excl;
      if (chunk == last) {                           // the size the first chunk read: no other writer yet
        const unsigned long long start = t.size[s];
        lanes_reserve_publish(t, s, start, excl + agg - start);
      }
    }
  }
  __syncthreads();
  uint64_t base = sm.base;
  int par = 0;
  // tiles from a GL-aligned lane: whole groups take the vector loads
  for (uint64_t t0 = wlo; t0 < lo + nl; t0 += T) {
    uint32_t c[L::R][L::GL], w[16];
    if (pf && tid == 0) pf_tile(t0 + (uint64_t)pf * T);
    lanes_load<ESZ, KB, VEC>(vals, counts, t0, lo, lo + nl, c, w);
    base += lanes_store<ESZ, KB, VEC>(t, sm, s, c, w, base, par);
    par ^= 1;
  }
}

// ---- the same one-pass insert with the value blocks streamed by TMA ------
// k_lanes_bulk: as k_lanes_chunk, but each tile's [T x K] value block (16 KiB
// = 256 threads x 64 B) arrives in a shared-memory ring of NS stages through
// cp.async.bulk (the TMA's 1-D bulk copy, completion counted on an mbarrier):
// thread 0 issues the chunk's first NS tiles before the counts are summed and
// chained, and refills a stage as soon as the CTA has moved its tile into
// registers, so the value loads of up to NS tiles are in flight while the
// CTA scans / stages / stores -- without holding registers for them.  Counts
// still come through the LSU (L2-resident after the count sum).  Tiles whose
// copy would be misaligned or run past the value array take the register
// path of k_lanes_chunk.  Used where it measured faster (lanes of 8, 32 or
// 64 B, lanes_tiled).
__device__ __forceinline__ uint32_t smem_addr(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ void mbar_wait(uint32_t bar, uint32_t parity) {
  asm volatile("{\n .reg .pred p;\n W: mbarrier.try_wait.parity.shared.b64 p, [%0], %1;\n @!p bra W;\n}"
               ::"r"(bar), "r"(parity) : "memory");
}

// lanes_load with the values read from a tile staged in shared memory
// (ring = the tile's first lane wlo; counts as in lanes_load)
template <int ESZ, int KB>
__device__ __forceinline__ void lanes_load_ring(const char *ring, const uint32_t *counts, uint64_t wlo, uint64_t vlo,
                                                uint64_t vhi,
                                                uint32_t (&c)[LaneShape<ESZ, KB, true>::R][LaneShape<ESZ, KB, true>::GL],
                                                uint32_t (&w)[16]) {
  typedef LaneShape<ESZ, KB, true> L;
  const uint32_t lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  constexpr uint32_t GB = L::GL * KB;                 // bytes per group (16 or KB)
#pragma unroll
  for (uint32_t r = 0; r < L::R; ++r) {
    const uint32_t gi = (wid * L::R + r) * 32 + lane;   // group index in the tile
    const uint4 *sp = reinterpret_cast<const uint4 *>(ring + (size_t)gi * GB);
#pragma unroll
    for (uint32_t q = 0; q < GB / 16; ++q) {
      const uint4 v = sp[q];
      w[r * L::WPR + 4 * q] = v.x; w[r * L::WPR + 4 * q + 1] = v.y;
      w[r * L::WPR + 4 * q + 2] = v.z; w[r * L::WPR + 4 * q + 3] = v.w;
    }
  }
  const uint64_t ga = wlo + ((uint64_t)(wid * L::R) * 32 + lane) * L::GL;
  const uint64_t gz = wlo + ((uint64_t)(wid * L::R + L::R - 1) * 32 + lane) * L::GL;
  if (ga >= vlo && gz + L::GL <= vhi) {
    uint32_t cr[L::R][L::GL];
#pragma unroll
    for (uint32_t r = 0; r < L::R; ++r) {
      const uint64_t g0 = ga + (uint64_t)r * 32 * L::GL;
      if constexpr (L::GL == 4) {
        const uint4 x = __ldcs((const uint4 *)(counts + g0));
        cr[r][0] = x.x; cr[r][1] = x.y; cr[r][2] = x.z; cr[r][3] = x.w;
      } else if constexpr (L::GL == 2) {
        const uint2 x = __ldcs((const uint2 *)(counts + g0));
        cr[r][0] = x.x; cr[r][1] = x.y;
      } else {
        cr[r][0] = __ldcs(counts + g0);
      }
    }
#pragma unroll
    for (uint32_t r = 0; r < L::R; ++r)
#pragma unroll
      for (uint32_t g = 0; g < L::GL; ++g) c[r][g] = min(cr[r][g], L::K);
  } else {
#pragma unroll
    for (uint32_t r = 0; r < L::R; ++r) {
      const uint64_t g0 = wlo + ((uint64_t)(wid * L::R + r) * 32 + lane) * L::GL;
#pragma unroll
      for (uint32_t g = 0; g < L::GL; ++g)
        c[r][g] = (g0 + g >= vlo && g0 + g < vhi) ? min(__ldcs(counts + g0 + g), L::K) : 0u;
    }
  }
}

template <int ESZ, int KB, int NS>
__global__ void __launch_bounds__(256) k_lanes_bulk(Tables t, const char *vals, const uint32_t *counts,
                                                    const uint32_t *cpre, unsigned long long *chain, uint32_t C) {
  typedef LaneShape<ESZ, KB, true> L;
  constexpr uint32_t K = L::K, T = L::T, TB = T * KB;
  static_assert(TB == 16384, "a tile's value block is 256 threads x 64 B");
  extern __shared__ __align__(128) char ring[];        // NS x TB
  __shared__ LaneSmem<ESZ, KB, true> sm;
  __shared__ uint32_t red[8];
  __shared__ __align__(8) unsigned long long bar[NS];
  pdl_begin();
  const uint32_t tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const uint32_t chunk = blockIdx.x;
  const uint32_t s = warp_find_u32(cpre, t.S, chunk);
  const uint32_t first = cpre[s], last = cpre[s + 1] - 1;
  const uint64_t lo = t.offsets[s] + (uint64_t)(chunk - first) * C;
  const uint32_t nl = (uint32_t)min((uint64_t)C, t.offsets[s + 1] - lo);
  const uint64_t hi = lo + nl, total = t.offsets[t.S];
  const uint64_t wlo = lo - lo % L::GL;                 // tiles from a GL-aligned lane
  const uint32_t ntiles = (uint32_t)((hi - wlo + T - 1) / T);
  // bytes of tile i's bulk copy (0 = the tile takes the register path); the
  // value array is 16 B aligned (lanes_tiled) and tiles start on 16 B
  auto tile_bytes = [&](uint32_t i) -> uint32_t {
    const uint64_t ts = wlo + (uint64_t)i * T, te = min(ts + T, hi);
    if (te == total && ((te * KB) & 15)) return 0;     // the copy would run past the value array
    return (uint32_t)(((te - ts) * KB + 15) & ~uint64_t(15));
  };
  auto issue = [&](uint32_t i) {
    const uint32_t nb = tile_bytes(i);
    if (!nb) return;
    const uint32_t k = i % NS, b = smem_addr(&bar[k]);
    asm volatile("mbarrier.arrive.expect_tx.shared.b64 _, [%0], %1;" ::"r"(b), "r"(nb) : "memory");
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_addr(ring + (size_t)k * TB)), "l"(vals + (wlo + (uint64_t)i * T) * KB), "r"(nb), "r"(b)
                 : "memory");
  };
  if (tid == 0) {
#pragma unroll
    for (int k = 0; k < NS; ++k) asm volatile("mbarrier.init.shared.b64 [%0], 1;" ::"r"(smem_addr(&bar[k])));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    for (uint32_t i = 0; i < (uint32_t)NS && i < ntiles; ++i) issue(i);
  }
  stage_cbase(t, sm.scb);
  const uint32_t agg = chunk_count_sum(counts, lo, nl, K, red);   // (its barrier publishes the mbarrier init)
  if (wid == 0) {
    unsigned long long excl = 0;
    if (chunk == first) {
      if (lane == 0) {
        excl = t.size[s];
        st_chain(chain + chunk, kChainP | (excl + agg));
      }
      excl = __shfl_sync(0xffffffffu, excl, 0);
    } else {
      if (lane == 0) st_chain(chain + chunk, kChainA | agg);
      int64_t j = (int64_t)chunk - 1;
      for (;;) {
        const int64_t idx = j - lane;
        unsigned long long v;
        do {
          v = idx >= (int64_t)first ? ld_chain(chain + idx) : kChainP;
        } while (__any_sync(0xffffffffu, (v >> 62) == 0));
        const unsigned pm = __ballot_sync(0xffffffffu, (v >> 62) == 2);
        const uint32_t stop = pm ? (uint32_t)(__ffs(pm) - 1) : 31u;
        unsigned long long x = lane <= stop ? (v & kChainV) : 0ull;
#pragma unroll
        for (int d = 16; d; d >>= 1) x += __shfl_xor_sync(0xffffffffu, x, d);
        excl += x;
        if (pm) break;
        j -= 32;
      }
      if (lane == 0) st_chain(chain + chunk, kChainP | (excl + agg));
    }
    if (lane == 0) {
      sm.base = excl;
      if (chunk == last) {
        const unsigned long long start = t.size[s];
        lanes_reserve_publish(t, s, start, excl + agg - start);
      }
    }
  }
  __syncthreads();
  uint64_t base = sm.base;
  uint32_t phase = 0;                                  // bit k: parity of stage k's next completion
  for (uint32_t i = 0; i < ntiles; ++i) {
    const uint64_t t0 = wlo + (uint64_t)i * T;
    uint32_t c[L::R][L::GL], w[16];
    if (tile_bytes(i)) {
      const uint32_t k = i % NS;
      mbar_wait(smem_addr(&bar[k]), (phase >> k) & 1u);
      phase ^= 1u << k;
      lanes_load_ring<ESZ, KB>(ring + (size_t)k * TB, counts, t0, lo, hi, c, w);
    } else {
      lanes_load<ESZ, KB, true>(vals, counts, t0, lo, hi, c, w);
    }
    // refill the stage right after lanes_store's barrier (every thread has
    // moved its tile into registers by then)
    base += lanes_store<ESZ, KB, true>(t, sm, s, c, w, base, (int)(i & 1), [&] {
      if (tid == 0 && i + NS < ntiles) {
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");   // generic reads before the async refill
        issue(i + NS);
      }
    });
  }
}

template <int ESZ, int U>
__global__ void __launch_bounds__(256) k_flat_append(char *buf, uint64_t start, unsigned long long *counter,
                                                     const char *vals, uint64_t n, uint64_t tile) {
  pdl_begin();
  if (blockIdx.x == 0 && threadIdx.x == 0 && counter) atomicAdd(counter, (unsigned long long)n);
  const uint64_t lo = (uint64_t)blockIdx.x * tile;
  if (lo >= n) return;
  const uint64_t cnt = min(tile, n - lo);
  cta_copy<ESZ, U>(buf + (start + lo) * ESZ, vals + lo * ESZ, cnt, threadIdx.x, blockDim.x);
}

// Paper 3-B-3 (block-level reservation), vectorised: each CTA reserves its
// tile of 256 x U 16 B vectors with ONE atomicAdd on the shared counter and
// copies it with 16 B stores (order between tiles is the atomics' order).
// Elements past the capacity are dropped (counted in *counter).
template <int ESZ, int U>
__global__ void __launch_bounds__(256) k_flat_insert_block(char *buf, uint64_t cap,
                                                           unsigned long long *counter,
                                                           const char *vals, uint64_t n, uint64_t tile) {
  __shared__ unsigned long long base_s;
  pdl_begin();
  const uint64_t lo = (uint64_t)blockIdx.x * tile;
  if (lo >= n) return;
  const uint64_t cnt = min(tile, n - lo);
  if (threadIdx.x == 0) base_s = atomicAdd(counter, (unsigned long long)cnt);
  __syncthreads();
  const uint64_t base = base_s;
  if (base >= cap) return;
  cta_copy<ESZ, U>(buf + base * ESZ, vals + lo * ESZ, min(cnt, cap - base), threadIdx.x, blockDim.x);
}

template <int ESZ>
__global__ void k_flat_insert(char *buf, uint64_t cap, unsigned long long *counter,
                              const char *vals, uint64_t n, int algo, uint64_t opaque_zero) {
  typedef typename ElemT<ESZ>::T E;
  const E *v = (const E *)vals;
  E *out = (E *)buf;
  __shared__ unsigned long long base_s;
  const uint64_t stride = (uint64_t)gridDim.x * blockDim.x;
  for (uint64_t j0 = (uint64_t)blockIdx.x * blockDim.x; j0 < n; j0 += stride) {
    uint64_t j = j0 + threadIdx.x;
    bool have = j < n;
    unsigned long long idx = 0;
    if (algo == GG_ALGO_ATOMIC) {
      // paper 3-B-1: one atomic per element.  The compiler warp-aggregates an
      // atomicAdd on a provably uniform address by itself (ncu: 32x fewer L2
      // atomic requests), which would turn this baseline into the warp one;
      // the per-thread `j * opaque_zero` offset (0 at run time) keeps the
      // address non-uniform to the compiler.
      if (have) idx = atomicAdd(counter + j * opaque_zero, 1ull);
    } else if (algo == GG_ALGO_WARP) {
      // paper 3-B-2 (warp shuffle scan of 0/1 counts, one atomic per warp)
      unsigned mask = __ballot_sync(0xffffffffu, have);
      unsigned lane = threadIdx.x & 31;
      unsigned long long wb = 0;
      if (lane == 0 && mask) wb = atomicAdd(counter, (unsigned long long)__popc(mask));
      wb = __shfl_sync(0xffffffffu, wb, 0);
      idx = wb + __popc(mask & ((1u << lane) - 1u));
    } else {  // GG_ALGO_BLOCK: block scan, one atomic per CTA
      uint64_t cnt = min((uint64_t)blockDim.x, n - j0);
      if (threadIdx.x == 0) base_s = atomicAdd(counter, (unsigned long long)cnt);
      __syncthreads();
      idx = base_s + threadIdx.x;
      __syncthreads();
    }
    if (have && idx < cap) out[idx] = v[j];
  }
}

template <typename T, int UNROLL = kDefUnroll, int LS = kDefLS>
__global__ void __launch_bounds__(512) k_flat_add(char *buf, uint64_t n, T a, uint32_t reps) {
  pdl_begin();
  // one kFlatChunk chunk of the contiguous array per CTA (non-persistent grid)
  constexpr uint64_t CH = kFlatChunk / sizeof(T);
  const uint64_t nch = (n + CH - 1) / CH;
  for (uint64_t c = blockIdx.x; c < nch; c += gridDim.x) {
    uint64_t lo = c * CH, len = min(n - lo, CH);
    cta_add<T, UNROLL, LS>(buf + lo * sizeof(T), len, a, reps, threadIdx.x, blockDim.x);
  }
}

}  // namespace gg

#endif  // GG_DEVICE_CUH
