// ggarray.cu -- B200 (sm_100a) GGArray: device tables, VMM bucket arena,
// bump allocator, and the hot kernels (reserve+allocate, insert, duplicate,
// commit, r/w, flatten, gather/scatter) behind the C ABI in include/ggarray.h.
//
// Layout in HBM (one handle per GPU):
//   * metadata (plain cudaMalloc, never in the slabs): size[S], cap[S],
//     ops[S], start[S], count[S], prefix[S+1], offsets[S+1], ctl[S],
//     flag[S*MB] (u32 once-flags: 0 free, 1 allocating, 2 published),
//     ptr[S*MB] (bucket base pointers), pmask/amask[S], cbase[MB], misc[].
//   * bucket slabs: class b owns a VA region of S slots of bucket_bytes(b)
//     (classes whose region is below one 2 MiB granule share one packed
//     region), so bucket (s, b) always lives at cbase[b] + s*bytes(b).  The
//     host backs slots with physical memory in chunks (cuMemCreate/cuMemMap,
//     refcounted by live buckets) before a launch can publish them, and a
//     shrink unmaps chunks none of whose buckets is live any more -- the
//     footprint follows the live capacity (<= 2x the needed bytes) both ways.
// The host keeps exact mirrors of sizes / flags / capacities (every quantity
// is a deterministic function of the op sequence), which lets it back
// memory, raise the reference's errors and run the allocator hook without
// any device round trip per insert.
#include <cuda.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <utility>
#include <type_traits>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <atomic>
#include <chrono>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/ggarray.h"
#include "../../include/ggarray_device.cuh"

#define GG_VERSION 1

namespace gg {

typedef gg_device_view Tables;

thread_local std::string g_err;
std::atomic<unsigned long long> g_launches{0};   // kernels launched by this library

int fail(int code, const std::string &msg) {
  g_err = msg;
  return code;
}

// Driver VMM entry points resolved through cudaGetDriverEntryPoint, so the
// library has no link-time libcuda dependency (it loads on GPU-less hosts).
struct Drv {
  decltype(&cuMemGetAllocationGranularity) granularity = nullptr;
  decltype(&cuMemAddressReserve) reserve = nullptr;
  decltype(&cuMemAddressFree) addr_free = nullptr;
  decltype(&cuMemCreate) create = nullptr;
  decltype(&cuMemRelease) release = nullptr;
  decltype(&cuMemMap) map = nullptr;
  decltype(&cuMemUnmap) unmap = nullptr;
  decltype(&cuMemSetAccess) set_access = nullptr;
  decltype(&cuGetErrorString) err_string = nullptr;
  bool ok = false;
};

Drv &drv() {
  static Drv d;
  static std::once_flag once;
  std::call_once(once, [] {
    auto get = [](const char *name, void **fn) {
      cudaDriverEntryPointQueryResult q;
      return cudaGetDriverEntryPoint(name, fn, cudaEnableDefault, &q) == cudaSuccess &&
             q == cudaDriverEntryPointSuccess && *fn != nullptr;
    };
    d.ok = get("cuMemGetAllocationGranularity", (void **)&d.granularity) &&
           get("cuMemAddressReserve", (void **)&d.reserve) &&
           get("cuMemAddressFree", (void **)&d.addr_free) &&
           get("cuMemCreate", (void **)&d.create) && get("cuMemRelease", (void **)&d.release) &&
           get("cuMemMap", (void **)&d.map) && get("cuMemUnmap", (void **)&d.unmap) &&
           get("cuMemSetAccess", (void **)&d.set_access) &&
           get("cuGetErrorString", (void **)&d.err_string);
  });
  return d;
}

#define CUDA_TRY(expr)                                                                 \
  do {                                                                                 \
    cudaError_t e_ = (expr);                                                           \
    if (e_ != cudaSuccess)                                                             \
      return fail(GG_ECUDA, std::string(#expr) + ": " + cudaGetErrorString(e_));       \
  } while (0)

#define CU_TRY(expr)                                                                   \
  do {                                                                                 \
    CUresult r_ = (expr);                                                              \
    if (r_ != CUDA_SUCCESS) {                                                          \
      const char *s_ = nullptr;                                                        \
      if (drv().err_string) drv().err_string(r_, &s_);                                 \
      return fail(r_ == CUDA_ERROR_OUT_OF_MEMORY ? GG_ENOMEM : GG_ECUDA,               \
                  std::string(#expr) + ": " + (s_ ? s_ : "?"));                        \
    }                                                                                  \
  } while (0)

constexpr int kMaxBuckets = 64;
constexpr uint64_t kDefaultVaBudget = uint64_t(16) << 40;   // slab VA per array (16 TiB)
constexpr int kThreads = 256;          // CTA size of the streaming kernels
constexpr uint64_t kFlatChunk = 16 * 1024;  // bytes per CTA of the contiguous +c kernel

// ctl word per shard (only uploaded when an op plans a failure)
constexpr uint32_t kCtlLimitMask = 0xffu;   // allocate buckets < limit
constexpr uint32_t kCtlWrite = 1u << 8;     // write the values
constexpr uint32_t kCtlZero = 1u << 9;      // write zeros instead (failed shard)

inline uint32_t elem_bytes_of(uint32_t dt) {
  switch (dt) {
    case GG_I8: case GG_U8: return 1;
    case GG_I16: case GG_U16: case GG_F16: return 2;
    case GG_I32: case GG_U32: case GG_F32: return 4;
    case GG_I64: case GG_U64: case GG_F64: return 8;
    default: return 0;
  }
}

inline uint64_t round16(uint64_t x) { return (x + 15) & ~uint64_t(15); }

inline int ilog2(uint64_t x) { return 63 - __builtin_clzll(x); }

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

// Publish buckets `want` of shard s (host-planned, slots already backed) from
// the one thread that owns s in this launch: slot pointer + once-flag per
// bucket, the shard's pmask (pm = its value at kernel start) and capacity,
// and one allocation-count update per warp.  Plain stores: the kernel
// boundary orders them before any reader.  Call with the full warp.
__device__ __forceinline__ void publish_buckets(const Tables &t, char *const *scb, uint32_t s,
                                                unsigned long long pm, unsigned long long want,
                                                uint32_t lg0) {
  uint64_t add = 0;
  for (unsigned long long m = want; m; m &= m - 1) {
    const uint32_t b = __ffsll((long long)m) - 1;
    t.ptr[(size_t)s * t.MB + b] = scb[b] + ((uint64_t)s << max(lg0 + b, 4u));
    t.flag[(size_t)s * t.MB + b] = kFlagPublished;
    add += 1ull << (t.log2fb + b);
  }
  if (want) {
    t.pmask[s] = pm | want;
    atomicAdd((unsigned long long *)&t.cap[s], (unsigned long long)add);
  }
  const uint32_t tot = __reduce_add_sync(0xffffffffu, (uint32_t)__popcll(want));
  if ((threadIdx.x & 31) == 0 && tot) atomicAdd(&t.misc[MISC_ALLOCS], (unsigned long long)tot);
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
  publish_buckets(t, scb, live ? s : 0u, pm, live ? want : 0ull, t.log2fb + (31u - __clz(t.esz)));
}

__global__ void k_new_bucket(Tables t, uint32_t s, uint32_t b, int *won) {
  *won = alloc_bucket(t, s, b);
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
__global__ void __launch_bounds__(1024) k_lanes_count(Tables t, const uint32_t *counts) {
  __shared__ uint64_t ws[32];
  const uint32_t s = blockIdx.x;
  const uint64_t lo = t.offsets[s], hi = t.offsets[s + 1];
  uint64_t acc = 0;
  for (uint64_t j = lo + threadIdx.x; j < hi; j += blockDim.x) acc += counts[j];
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
    const uint32_t cnt = j < hi ? counts[j] : 0;
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
__global__ void __launch_bounds__(1024) k_shrink(Tables t, const uint64_t *new_sizes) {
  __shared__ uint64_t ws[32];
  pdl_begin();
  uint64_t carry = 0;
  for (uint32_t base = 0; base < t.S; base += blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    const bool live = s < t.S;
    uint64_t ns = 0, cap = 0;
    unsigned long long m = 0;
    if (live) { ns = new_sizes[s]; m = t.pmask[s]; cap = t.cap[s]; }
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

// dst[0..n) = src[0..n) (element granular, arbitrary relative alignment), or
// zeros if src == nullptr.  Stores are 16 B aligned vectors; loads are 16 B
// vectors when src shares dst's alignment, else element loads.
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
    const E *s2 = (const E *)sb;
    for (uint64_t v0 = tid; v0 < body; v0 += UNROLL * (uint64_t)nt) {
      union { uint4 q; E e[VE]; } u[UNROLL];
#pragma unroll
      for (int k = 0; k < UNROLL; ++k) {
        const uint64_t v = min(v0 + k * (uint64_t)nt, body - 1);
#pragma unroll
        for (uint32_t j = 0; j < VE; ++j) u[k].e[j] = M::ld(s2 + v * VE + j);
      }
#pragma unroll
      for (int k = 0; k < UNROLL; ++k)
        if (v0 + k * (uint64_t)nt < body) M::st(dv + v0 + k * nt, u[k].q);
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
__device__ __forceinline__ bool vector_tile(const Tables &t, char *const *scb, const uint64_t *dir,
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
struct Fuse { int rmode; int commit; uint64_t g0 = 0; };   // g0: first work index (ranges)

// metadata of a planned append, run by one CTA after every tile is copied.
// Latency shaped: all loads (directory pair, size, pmask) issued up front,
// counters updated with fire-and-forget reductions, the commit scan runs on
// the new sizes held in registers (no reload).
__device__ void planned_metadata(const Tables &t, char *const *scb, const Fuse &fz) {
  __shared__ uint64_t ws[32];
  const uint32_t lg0 = t.log2fb + (31u - __clz(t.esz));
  const uint64_t *dir = fz.rmode == 0 ? t.offsets : t.prefix;
  uint64_t carry = 0;
  for (uint32_t base = 0; base < t.S; base += blockDim.x) {
    const uint32_t s = base + threadIdx.x;
    const bool live = s < t.S;
    uint64_t lo = 0, hi = 0, start = 0;
    unsigned long long pm = 0;
    if (live) { lo = dir[s]; hi = dir[s + 1]; start = t.size[s]; pm = t.pmask[s]; }
    const uint64_t c = hi - lo, nsz = start + c;
    unsigned long long want = 0;
    if (c) {
      t.size[s] = nsz;
      atomicAdd((unsigned long long *)&t.ops[s], 1ull);
      t.start[s] = start;
      uint32_t b0, b1; uint64_t o;
      locate(start, t.log2fb, b0, o);
      locate(nsz - 1, t.log2fb, b1, o);
      want = (b1 >= 63 ? ~0ull : ((2ull << b1) - 1ull)) & ~((1ull << b0) - 1ull) & ~pm;
    }
    if (live) t.count[s] = c;
    publish_buckets(t, scb, live ? s : 0u, pm, want, lg0);
    if (fz.commit) {
      uint64_t tot;
      const uint64_t ex = block_exclusive_scan(live ? nsz : 0, &tot, ws);
      if (live) t.prefix[s + 1] = carry + ex + nsz;
      carry += tot;
    }
  }
  if (fz.commit && threadIdx.x == 0) t.prefix[0] = 0;
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
  __shared__ uint32_t s_sh;
  const uint32_t tid = threadIdx.x, nt = blockDim.x;
  pdl_begin();
  const uint64_t *dir = (W == W_INSERT) ? t.offsets : t.prefix;
  uint64_t g = fz.g0 + (uint64_t)blockIdx.x * tile;
  const uint64_t gend = min(total, g + tile);
  if (tid < 32) {
    const uint32_t s0 = warp_find_shard(dir, t.S, g);
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
    dbase = PLANNED ? t.size[s] : t.start[s];
  }
  if (!(fast && vector_tile<ESZ, W, T, U, LS>(t, scb, dir, s, dbase, g, gend, flat_src, flat_dst,
                                              addend, reps))) {
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
        locate((PLANNED ? t.size[s] : t.start[s]) + k, t.log2fb, b, o);
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
    publish_buckets(t, scb, live ? s : 0u, pm, live ? (all & ~pm) : 0ull, lg0);
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

template <int ESZ>
__global__ void k_gather(Tables t, const int64_t *idx, uint64_t n, char *out, const char *vals,
                         int scatter) {
  typedef typename ElemT<ESZ>::T E;
  for (uint64_t j = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n;
       j += (uint64_t)gridDim.x * blockDim.x) {
    uint64_t g = (uint64_t)idx[j];
    uint32_t s = upper_shard(t.prefix, t.S, g);
    uint32_t b; uint64_t o;
    locate(g - t.prefix[s], t.log2fb, b, o);
    E *p = (E *)(t.ptr[(size_t)s * t.MB + b]) + o;
    if (scatter) *p = ((const E *)vals)[j];
    else ((E *)out)[j] = *p;
  }
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

// ------------------------------------------------------------------ host side

struct Arena {
  int dev = 0;
  CUdeviceptr base = 0;
  size_t va = 0, gran = 0, mapped = 0;
  struct Map { size_t off, size; CUmemGenericAllocationHandle h; };
  std::vector<Map> maps;

  int init(int device, uint64_t va_bytes) {
    dev = device;
    if (!drv().ok) return fail(GG_ECUDA, "CUDA driver VMM entry points unavailable");
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = device;
    CU_TRY(drv().granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    va = (va_bytes + gran - 1) / gran * gran;
    CU_TRY(drv().reserve(&base, va, gran, 0, 0));
    return GG_OK;
  }
  // map physical granules so that [0, bytes) is backed, in pieces of at most
  // kMapChunk so a later trim() can release unused headroom
  static constexpr size_t kMapChunk = size_t(64) << 20;
  int ensure(uint64_t bytes) {
    while (mapped < bytes) {
      size_t want = (bytes + gran - 1) / gran * gran;
      if (want > va) return fail(GG_ENOMEM, "arena VA reservation exhausted");
      size_t add = std::min(want - mapped, std::max(kMapChunk, gran));
      int rc = map_piece(add);
      if (rc) return rc;
    }
    return GG_OK;
  }
  int map_piece(size_t add) {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev;
    CUmemGenericAllocationHandle h;
    CU_TRY(drv().create(&h, add, &prop, 0));
    CUresult r = drv().map(base + mapped, add, 0, h, 0);
    if (r != CUDA_SUCCESS) {
      drv().release(h);
      return fail(GG_ECUDA, "cuMemMap failed");
    }
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    r = drv().set_access(base + mapped, add, &acc, 1);
    if (r != CUDA_SUCCESS) {
      drv().unmap(base + mapped, add);
      drv().release(h);
      return fail(GG_ECUDA, "cuMemSetAccess failed");
    }
    maps.push_back({mapped, add, h});
    mapped += add;
    return GG_OK;
  }
  // release whole mappings lying at or above `keep` bytes
  void trim(uint64_t keep) {
    cudaDeviceSynchronize();
    while (!maps.empty() && maps.back().off >= keep) {
      Map m = maps.back();
      maps.pop_back();
      drv().unmap(base + m.off, m.size);
      drv().release(m.h);
      mapped = m.off;
    }
  }
  void destroy() {
    trim(0);
    if (base) drv().addr_free(base, va);
    base = 0;
  }
};

// Slab store of one GGArray: a VA region per bucket class, slot s of class b
// = bucket (s, b).  Physical memory is mapped per chunk (a gran-multiple
// piece of a region) and refcounted by the live buckets overlapping it, so
// releasing buckets returns memory as soon as a chunk empties.  Classes whose
// region is smaller than one granule share one packed region ("small"), so a
// tiny array costs one granule, not one per class.
struct Slab {
  struct Chunk { uint32_t refs = 0; bool mapped = false; CUmemGenericAllocationHandle h = 0; };
  struct Region { CUdeviceptr base = 0; size_t va = 0, chunk = 0; std::vector<Chunk> chunks; };
  static constexpr size_t kChunk = size_t(64) << 20;   // mapping unit of large regions
  int dev = 0;
  size_t gran = 0;
  uint32_t S = 0, MB = 0;
  uint64_t va_budget = 0, va_used = 0, mapped = 0, cached = 0;  // cached: mapped, 0 refs
  uint64_t n_map = 0, n_unmap = 0, ns_map = 0, ns_unmap = 0, n_regions = 0;  // cost counters
  static uint64_t now_ns() {
    return (uint64_t)std::chrono::duration_cast<std::chrono::nanoseconds>(
        std::chrono::steady_clock::now().time_since_epoch()).count();
  }
  std::vector<uint64_t> bytes;        // bucket bytes per class (powers of two >= 16)
  std::vector<uint64_t> small_off;    // offset in the small region, ~0 = own region
  Region small;
  std::vector<Region> big;

  int init(int device, uint32_t shards, uint32_t mb, const std::vector<uint64_t> &bb, uint64_t budget) {
    dev = device; S = shards; MB = mb; bytes = bb; va_budget = budget;
    if (!drv().ok) return fail(GG_ECUDA, "CUDA driver VMM entry points unavailable");
    CUmemAllocationProp prop = props();
    CU_TRY(drv().granularity(&gran, &prop, CU_MEM_ALLOC_GRANULARITY_MINIMUM));
    small_off.assign(MB, ~uint64_t(0));
    big.assign(MB, Region());
    uint64_t off = 0;
    for (uint32_t b = 0; b < MB; ++b) {
      const long double r = (long double)S * bytes[b];
      if (r >= gran) break;
      small_off[b] = off;
      off += S * bytes[b];
    }
    if (off) {
      small.va = round_up(off, gran);
      small.chunk = gran;
      small.chunks.assign(small.va / gran, Chunk());
      int rc = reserve_va(small);
    if (rc) return rc;
    }
    return GG_OK;
  }
  static size_t round_up(uint64_t x, uint64_t m) { return (x + m - 1) / m * m; }
  CUmemAllocationProp props() const {
    CUmemAllocationProp prop = {};
    prop.type = CU_MEM_ALLOCATION_TYPE_PINNED;
    prop.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    prop.location.id = dev;
    return prop;
  }
  int reserve_va(Region &r) {
    if (va_used + r.va > va_budget) return fail(GG_ENOMEM, "slab VA budget exhausted");
    CUresult e = drv().reserve(&r.base, r.va, r.chunk, 0, 0);
    if (e != CUDA_SUCCESS) { r.base = 0; return fail(GG_ENOMEM, "cuMemAddressReserve failed (VA exhausted)"); }
    va_used += r.va;
    n_regions += 1;
    return GG_OK;
  }
  // mapping unit of class b's region: a power of two >= one granule and >=
  // one bucket, about 1/16 of the region (so a partly live top class -- an
  // uneven split -- strands at most one chunk), at most kChunk otherwise
  uint64_t chunk_for(uint32_t b) const {
    if (bytes[b] >= kChunk) return bytes[b];
    const uint64_t R = S * bytes[b];
    uint64_t c = gran;
    while (c < kChunk && c * 32 <= R) c <<= 1;
    return std::max<uint64_t>(c, bytes[b]);
  }
  Region &region(uint32_t b) { return small_off[b] != ~uint64_t(0) ? small : big[b]; }
  // reserve class b's region on first use; *created = true if it is new
  int ensure_region(uint32_t b, bool *created) {
    *created = false;
    if (small_off[b] != ~uint64_t(0)) return GG_OK;
    Region &r = big[b];
    if (r.base) return GG_OK;
    const long double want = (long double)S * bytes[b];
    if (want > (long double)va_budget) return fail(GG_ENOMEM, "bucket class region exceeds the VA budget");
    const uint64_t R = S * bytes[b];
    r.chunk = chunk_for(b);
    r.va = round_up(R, r.chunk);
    r.chunks.assign(r.va / r.chunk, Chunk());
    int rc = reserve_va(r);
    if (rc) { r = Region(); return rc; }
    *created = true;
    return GG_OK;
  }
  uint64_t class_base(uint32_t b) const {
    if (small_off[b] != ~uint64_t(0)) return (uint64_t)small.base + small_off[b];
    return (uint64_t)big[b].base;
  }
  void span(uint32_t s, uint32_t b, Region *&r, size_t &c0, size_t &c1) {
    r = &region(b);
    const uint64_t off = (small_off[b] != ~uint64_t(0) ? small_off[b] : 0) + (uint64_t)s * bytes[b];
    c0 = off / r->chunk;
    c1 = (off + bytes[b] - 1) / r->chunk;
  }
  int map_chunk(Region &r, size_t c) {
    Chunk &k = r.chunks[c];
    if (k.mapped) { if (!k.refs) cached -= r.chunk; return GG_OK; }
    const uint64_t t0 = now_ns();
    CUmemAllocationProp prop = props();
    CU_TRY(drv().create(&k.h, r.chunk, &prop, 0));
    const CUdeviceptr at = r.base + c * r.chunk;
    if (drv().map(at, r.chunk, 0, k.h, 0) != CUDA_SUCCESS) {
      drv().release(k.h);
      return fail(GG_ENOMEM, "cuMemMap failed");
    }
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    if (drv().set_access(at, r.chunk, &acc, 1) != CUDA_SUCCESS) {
      drv().unmap(at, r.chunk);
      drv().release(k.h);
      return fail(GG_ENOMEM, "cuMemSetAccess failed");
    }
    k.mapped = true;
    mapped += r.chunk;
    n_map += 1;
    ns_map += now_ns() - t0;
    return GG_OK;
  }
  void unmap_chunk(Region &r, size_t c) {
    Chunk &k = r.chunks[c];
    const uint64_t t0 = now_ns();
    drv().unmap(r.base + c * r.chunk, r.chunk);
    drv().release(k.h);
    k.mapped = false;
    k.h = 0;
    mapped -= r.chunk;
    cached -= r.chunk;
    n_unmap += 1;
    ns_unmap += now_ns() - t0;
  }
  // back bucket (s, b) with physical memory (region must exist)
  int back(uint32_t s, uint32_t b) {
    Region *r; size_t c0, c1;
    span(s, b, r, c0, c1);
    for (size_t c = c0; c <= c1; ++c) {
      int rc = map_chunk(*r, c);
      if (rc) {                                  // undo this bucket's earlier chunks
        for (size_t d = c0; d < c; ++d) drop(*r, d);
        return rc;
      }
      r->chunks[c].refs += 1;
    }
    return GG_OK;
  }
  void drop(Region &r, size_t c) {
    Chunk &k = r.chunks[c];
    if (--k.refs == 0) cached += r.chunk;      // stays mapped until trim()
  }
  // bucket (s, b) is no longer live
  void unback(uint32_t s, uint32_t b) {
    Region *r; size_t c0, c1;
    span(s, b, r, c0, c1);
    for (size_t c = c0; c <= c1; ++c) drop(*r, c);
  }
  // chunks [c0, c1] overlapped by slots [s0, s1) of class b, with the number
  // of those slots touching each chunk (batched refcounting of uniform ops)
  template <typename F>
  void for_range(uint32_t b, uint32_t s0, uint32_t s1, F f) {
    Region &r = region(b);
    const uint64_t base = small_off[b] != ~uint64_t(0) ? small_off[b] : 0, bb = bytes[b];
    const uint64_t lo = base + (uint64_t)s0 * bb, hi = base + (uint64_t)s1 * bb;   // [lo, hi)
    for (size_t c = lo / r.chunk; c <= (hi - 1) / r.chunk; ++c) {
      const uint64_t clo = std::max<uint64_t>(lo, c * r.chunk), chi = std::min<uint64_t>(hi, (c + 1) * r.chunk);
      // slots with [base + s*bb, base + (s+1)*bb) intersecting [clo, chi)
      const uint64_t first = (clo - base) / bb, last = (chi - 1 - base) / bb;
      f(r, c, (uint32_t)(last - first + 1));
    }
  }
  // back slots [s0, s1) of class b (region must exist); all-or-nothing
  int back_range(uint32_t b, uint32_t s0, uint32_t s1) {
    if (s1 <= s0) return GG_OK;
    int rc = GG_OK;
    std::vector<std::pair<Region *, size_t>> done;
    for_range(b, s0, s1, [&](Region &r, size_t c, uint32_t n) {
      if (rc) return;
      if ((rc = map_chunk(r, c))) return;
      r.chunks[c].refs += n;
      done.push_back({&r, c});
    });
    if (rc) {                                   // roll back this call's refs
      size_t i = 0;
      for_range(b, s0, s1, [&](Region &r, size_t c, uint32_t n) {
        if (i < done.size() && done[i].first == &r && done[i].second == c) {
          r.chunks[c].refs -= n;
          if (!r.chunks[c].refs) cached += r.chunk;
          ++i;
        }
      });
    }
    return rc;
  }
  void unback_range(uint32_t b, uint32_t s0, uint32_t s1) {
    if (s1 <= s0) return;
    for_range(b, s0, s1, [&](Region &r, size_t c, uint32_t n) {
      r.chunks[c].refs -= n;
      if (!r.chunks[c].refs) cached += r.chunk;
    });
  }
  // bytes backing (s, b) would newly map
  uint64_t new_bytes(uint32_t s, uint32_t b) {
    if (small_off[b] == ~uint64_t(0) && !big[b].base) return chunk_for(b);
    Region *r; size_t c0, c1;
    span(s, b, r, c0, c1);
    uint64_t n = 0;
    for (size_t c = c0; c <= c1; ++c) if (!r->chunks[c].mapped) n += r->chunk;
    return n;
  }
  // unmap chunks without live buckets, largest class first, until at most
  // `keep` bytes stay mapped (caller synchronised the device)
  void trim_to(uint64_t keep) {
    for (int b = (int)MB - 1; b >= 0 && mapped > keep && cached; --b) {
      if (small_off[b] != ~uint64_t(0)) continue;
      Region &r = big[b];
      for (size_t c = r.chunks.size(); c-- > 0 && mapped > keep;)
        if (r.chunks[c].mapped && r.chunks[c].refs == 0) unmap_chunk(r, c);
    }
    for (size_t c = small.chunks.size(); c-- > 0 && mapped > keep;)
      if (small.chunks[c].mapped && small.chunks[c].refs == 0) unmap_chunk(small, c);
  }
  // unmap every chunk without live buckets (caller synchronised the device)
  void trim() {
    auto go = [&](Region &r) {
      for (size_t c = 0; c < r.chunks.size(); ++c)
        if (r.chunks[c].mapped && r.chunks[c].refs == 0) unmap_chunk(r, c);
    };
    go(small);
    for (auto &r : big) go(r);
  }
  void destroy() {
    auto go = [&](Region &r) {
      for (size_t c = 0; c < r.chunks.size(); ++c)
        if (r.chunks[c].mapped) {
          drv().unmap(r.base + c * r.chunk, r.chunk);
          drv().release(r.chunks[c].h);
        }
      if (r.base) drv().addr_free(r.base, r.va);
      r = Region();
    };
    go(small);
    for (auto &r : big) go(r);
    mapped = cached = va_used = 0;
  }
};

// Every library kernel is launched with programmatic stream serialization
// (PDL): it may start while its predecessor drains and waits in
// pdl_begin(), so back-to-back kernels (grow -> append -> grow ...) overlap
// launch latency and prologue with the previous kernel's tail.
bool g_pdl = true;
template <typename... KArgs, typename... Args>
cudaError_t launch_k(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                     Args &&...args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  at[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = at;
  cfg.numAttrs = g_pdl ? 1 : 0;
  g_launches.fetch_add(1, std::memory_order_relaxed);
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

int g_sms[64] = {0};

// runtime tuning of the 4-byte streaming kernels (sweep); -1 / 0 = default
struct Tuning { int unroll = -1; };   // streaming-kernel U forced by gg_set_tuning (-1 = built in)
Tuning g_tune;

int sm_count(int dev) {
  if (dev < 0 || dev >= 64) return 148;
  if (!g_sms[dev]) {
    int v = 0;
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0)
      v = 148;
    g_sms[dev] = v;
  }
  return g_sms[dev];
}

// Pinned upload ring: small per-op host arrays (offsets, ctl words) travel
// through pinned slots; a slot is reused only after its copy completed.  One
// ring per device, shared by every array of the process (created on first
// use), so constructing an array costs no pinned allocation; uploads larger
// than a slot go through a per-array pinned buffer.
struct Ring {
  static constexpr int kSlots = 64;
  static constexpr size_t kSlot = 64 << 10;
  char *block = nullptr;
  cudaEvent_t ev[kSlots] = {nullptr};
  bool used[kSlots] = {false};
  int next = 0;
  std::mutex mu;
  int init() {
    CUDA_TRY(cudaMallocHost(&block, kSlot * kSlots));
    for (int i = 0; i < kSlots; ++i) CUDA_TRY(cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming));
    return GG_OK;
  }
};

Ring *ring_for(int dev) {
  static std::mutex m;
  static Ring *rings[64] = {nullptr};
  if (dev < 0 || dev >= 64) return nullptr;
  std::lock_guard<std::mutex> g(m);
  if (!rings[dev]) {
    Ring *r = new Ring();
    if (r->init() != GG_OK) { delete r; return nullptr; }
    rings[dev] = r;          // process lifetime (driver teardown frees it)
  }
  return rings[dev];
}

struct Uploader {
  int dev = 0;
  char *big = nullptr;           // per-array pinned buffer for uploads above a ring slot
  size_t big_cap = 0;
  cudaEvent_t big_ev = nullptr;
  bool big_used = false;
  int init(int device) {
    dev = device;
    return GG_OK;
  }
  // copy `n` arrays (dst device ptr, src host ptr, bytes) in one slot
  // graph capture: uploads are carved from a pinned pool allocated when
  // capture mode is switched on (allocation is illegal during capture); the
  // pools stay alive, owned by the captured graphs, until release_captured
  static constexpr size_t kCapturePool = 4u << 20;
  bool capturing = false;
  std::vector<char *> captured;
  size_t pool_off = 0;
  int begin_capture() {
    char *h = nullptr;
    CUDA_TRY(cudaHostAlloc(&h, kCapturePool, cudaHostAllocDefault));
    captured.push_back(h);
    pool_off = 0;
    capturing = true;
    return GG_OK;
  }
  static int copy_in(char *h, cudaStream_t st, int n, void *const *dst, const void *const *src,
                     const size_t *bytes) {
    size_t off = 0;
    for (int i = 0; i < n; ++i) {
      memcpy(h + off, src[i], bytes[i]);
      CUDA_TRY(cudaMemcpyAsync(dst[i], h + off, bytes[i], cudaMemcpyHostToDevice, st));
      off += (bytes[i] + 15) & ~size_t(15);
    }
    return GG_OK;
  }
  int upload(cudaStream_t st, int n, void *const *dst, const void *const *src, const size_t *bytes) {
    if (capturing) {
      char *h = captured.back();
      for (int i = 0; i < n; ++i) {
        if (pool_off + bytes[i] > kCapturePool) return fail(GG_EVALUE, "capture upload pool exhausted");
        memcpy(h + pool_off, src[i], bytes[i]);
        CUDA_TRY(cudaMemcpyAsync(dst[i], h + pool_off, bytes[i], cudaMemcpyHostToDevice, st));
        pool_off += (bytes[i] + 15) & ~size_t(15);
      }
      return GG_OK;
    }
    size_t total = 0;
    for (int i = 0; i < n; ++i) total += (bytes[i] + 15) & ~size_t(15);
    if (total <= Ring::kSlot) {
      Ring *r = ring_for(dev);
      if (!r) return fail(GG_ECUDA, "pinned upload ring unavailable");
      std::lock_guard<std::mutex> g(r->mu);
      const int k = r->next;
      r->next = (r->next + 1) % Ring::kSlots;
      if (r->used[k]) CUDA_TRY(cudaEventSynchronize(r->ev[k]));
      int rc = copy_in(r->block + Ring::kSlot * k, st, n, dst, src, bytes);
      if (rc) return rc;
      CUDA_TRY(cudaEventRecord(r->ev[k], st));
      r->used[k] = true;
      return GG_OK;
    }
    if (big_used) CUDA_TRY(cudaEventSynchronize(big_ev));
    if (total > big_cap) {
      if (big) cudaFreeHost(big);
      big = nullptr;
      big_cap = 0;
      CUDA_TRY(cudaMallocHost(&big, total));
      big_cap = total;
      if (!big_ev) CUDA_TRY(cudaEventCreateWithFlags(&big_ev, cudaEventDisableTiming));
    }
    int rc = copy_in(big, st, n, dst, src, bytes);
    if (rc) return rc;
    CUDA_TRY(cudaEventRecord(big_ev, st));
    big_used = true;
    return GG_OK;
  }
  void release_captured() {
    for (char *h : captured) cudaFreeHost(h);
    captured.clear();
  }
  void destroy() {
    if (big_ev) cudaEventSynchronize(big_ev), cudaEventDestroy(big_ev);
    if (big) cudaFreeHost(big);
    release_captured();
  }

};

}  // namespace gg

using namespace gg;

struct gg_array {
  int dev;
  uint32_t S, fb, log2fb, dtype, esz, MB;
  // exact host mirrors
  std::vector<uint64_t> size, cap, ops, prefix, flags;  // flags: bitmask per shard
  std::vector<uint8_t> dirty;                            // shard saw a failed reservation
  uint64_t live = 0;                                     // bytes of live buckets
  std::vector<uint32_t> headroom;                        // (s, b) backed for a device view
  bool cbase_dirty = false;                              // a class region appeared
  // metadata pass of the last planned append, not launched yet (eager issue
  // only): fused into the next grow, launched by any other device-touching call
  bool pend = false;
  Fuse pend_fz{0, 0};
  cudaStream_t pend_st = nullptr;
  bool defer_in_capture = false;                         // capture mode 2: caller flushes in-capture
  uint64_t alloc_calls = 0;
  uint64_t limit = 0;                                    // live-bytes cap (0 = none)
  gg_alloc_hook hook = nullptr;
  void *hook_ctx = nullptr;
  Slab slab;
  Uploader up;
  Tables t;          // device pointers (kernel argument)
  void *dmem = nullptr;
  int *d_won = nullptr;
  char *d_scratch = nullptr;   // 64 B element scratch for get/set
  char *h_scratch = nullptr;   // pinned
  std::mutex mu;
};

namespace {

inline uint64_t bucket_elems(const gg_array *a, uint32_t b) { return uint64_t(a->fb) << b; }
// saturates at 2^63 for classes no device could hold (max_buckets up to 64)
inline uint64_t bucket_bytes(const gg_array *a, uint32_t b) {
  const uint32_t lg = a->log2fb + b + (uint32_t)ilog2(a->esz);
  return lg >= 63 ? (uint64_t(1) << 63) : round16(bucket_elems(a, b) * a->esz);
}
inline void host_locate(const gg_array *a, uint64_t i, uint32_t &b, uint64_t &off) {
  uint64_t q = (i >> a->log2fb) + 1;
  b = (uint32_t)ilog2(q);
  off = i - (((uint64_t(1) << b) - 1) << a->log2fb);
}
inline uint32_t min_buckets_for(const gg_array *a, uint64_t n) {
  if (n == 0) return 0;
  uint64_t t = (n + a->fb - 1) / a->fb;
  return (uint32_t)ilog2(t) + 1;
}
inline cudaStream_t S_(void *s) { return (cudaStream_t)s; }
// make the handle's device current only when it is not (cheap, capture-safe)
inline void use_dev(int dev) {
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != dev) cudaSetDevice(dev);
}


Tables tables_for_launch(gg_array *a, bool with_ctl) {
  Tables t = a->t;
  if (!with_ctl) t.ctl = nullptr;
  t.amask = nullptr;          // library launches only publish host-backed buckets
  return t;
}

// Plan of one allocating operation, computed on the host before launch.
// Backing (physical mapping) happens while planning, so a real out-of-memory
// fails exactly the shard whose bucket could not be had, like a failing
// allocator in the reference (bucket_vector.py:194-201).
struct Plan {
  std::vector<uint64_t> size, cap, flags;
  uint64_t live, alloc_calls;
  std::vector<uint32_t> ctl;        // per shard
  std::vector<int32_t> status;      // per shard
  std::vector<uint32_t> zero_pairs; // (s, b) buckets to zero after allocation
  bool any_fail = false, any_ctl = false;
};

void plan_init(const gg_array *a, Plan &p) {
  p.size = a->size; p.cap = a->cap; p.flags = a->flags;
  p.live = a->live; p.alloc_calls = a->alloc_calls;
  p.ctl.assign(a->S, kCtlWrite | a->MB);
  p.status.assign(a->S, GG_OK);
}

// reserve class b's region if needed and back slot (s, b)
int back_bucket(gg_array *a, uint32_t s, uint32_t b) {
  bool created = false;
  int rc = a->slab.ensure_region(b, &created);
  if (rc) return rc;
  if (created) a->cbase_dirty = true;
  return a->slab.back(s, b);
}

// Try to allocate bucket b of shard s in the plan; false on (hook/memory) failure.
bool plan_alloc(gg_array *a, Plan &p, uint32_t s, uint32_t b) {
  if (a->hook && a->hook(a->hook_ctx, s, b, bucket_elems(a, b)) != 0) return false;
  const uint64_t nb = bucket_bytes(a, b);
  if (a->limit && p.live + nb > a->limit) return false;
  if (back_bucket(a, s, b) != GG_OK) return false;
  p.live += nb;
  p.flags[s] |= uint64_t(1) << b;
  p.cap[s] += bucket_elems(a, b);
  p.alloc_calls += 1;
  if (a->dirty[s]) { p.zero_pairs.push_back(s); p.zero_pairs.push_back(b); }
  return true;
}

// Plan an append of counts[s] at starts (explicit) or at size[s] (reserve).
void plan_append(gg_array *a, Plan &p, const uint64_t *counts, const uint64_t *starts) {
  for (uint32_t s = 0; s < a->S; ++s) {
    uint64_t c = counts[s];
    if (c == 0) continue;
    uint64_t start = starts ? starts[s] : p.size[s];
    if (!starts) p.size[s] += c;
    uint32_t b0, b1; uint64_t o;
    host_locate(a, start, b0, o);
    host_locate(a, start + c - 1, b1, o);
    if (b1 >= a->MB) {                       // bucket_vector.py:208-211
      p.status[s] = GG_ECAPACITY;
      p.ctl[s] = 0;                          // reserve only: no allocation, no write
      p.any_fail = p.any_ctl = true;
      continue;
    }
    for (uint32_t b = b0; b <= b1; ++b) {
      if (p.flags[s] >> b & 1) continue;
      if (!plan_alloc(a, p, s, b)) {         // bucket_vector.py:194-201
        p.status[s] = GG_ENOMEM;
        p.ctl[s] = b | kCtlZero;             // keep buckets < b; zero the reserved range
        p.any_fail = p.any_ctl = true;
        break;
      }
    }
  }
}

// class bases travel to the device when a new class region was reserved
int push_cbase(gg_array *a, cudaStream_t st) {
  if (!a->cbase_dirty) return GG_OK;
  std::vector<uint64_t> cb(a->MB);
  for (uint32_t b = 0; b < a->MB; ++b) cb[b] = a->slab.class_base(b);
  void *dst[1] = {a->t.cbase};
  const void *src[1] = {cb.data()};
  size_t bytes[1] = {a->MB * sizeof(uint64_t)};
  int rc = a->up.upload(st, 1, dst, src, bytes);
  if (rc) return rc;
  a->cbase_dirty = false;
  return GG_OK;
}

int commit_plan(gg_array *a, Plan &p, cudaStream_t st) {
  a->size = p.size; a->cap = p.cap; a->flags = p.flags;
  a->live = p.live; a->alloc_calls = p.alloc_calls;
  for (uint32_t s = 0; s < a->S; ++s)
    if (p.status[s] != GG_OK) a->dirty[s] = 1;
  return push_cbase(a, st);
}

// Streaming launches: one tile per CTA of kThreads threads x U 16 B vectors.
// Large work spaces use the U the sweep measured best per walk (tools/
// sweep.py, B200: copies into / in place on the slabs U = 8 -- 32 KiB tiles,
// flatten U = 4); smaller ones shrink U so small rounds still spread over
// every SM.  gg_set_tuning can force U.
uint32_t walk_unroll(const gg_array *a, uint64_t total, int w) {
  if (g_tune.unroll > 0) return (uint32_t)g_tune.unroll;
  const uint64_t bytes = total * a->esz;
  if (bytes < (uint64_t(32) << 20)) return 2u;
  if (bytes < (uint64_t(256) << 20)) return 4u;
  return w == W_FLATTEN ? 4u : 8u;
}

template <int ESZ, int W, typename T, bool P, int U>
cudaError_t walk_u(const gg_array *a, const Tables &t, const char *src, char *dst, uint64_t total,
                   T add, uint32_t reps, Fuse fz, cudaStream_t st) {
  const uint32_t tile = (uint32_t)U * kThreads * (16 / ESZ);
  const uint64_t grid = (total - fz.g0 + tile - 1) / tile;
  return launch_k(k_walk<ESZ, W, T, U, kDefLS, P>, (unsigned)grid, kThreads, 0, st, t, src, dst,
                  total, add, reps, tile, fz);
}

template <int ESZ, int W, typename T, bool P = false>
int walk(const gg_array *a, const Tables &t, const char *src, char *dst, uint64_t total, T add,
         uint32_t reps, Fuse fz, cudaStream_t st) {
  if (total == 0) return GG_OK;
  cudaError_t e;
  switch (walk_unroll(a, total, W)) {
    case 1: e = walk_u<ESZ, W, T, P, 1>(a, t, src, dst, total, add, reps, fz, st); break;
    case 2: e = walk_u<ESZ, W, T, P, 2>(a, t, src, dst, total, add, reps, fz, st); break;
    case 8: e = walk_u<ESZ, W, T, P, 8>(a, t, src, dst, total, add, reps, fz, st); break;
    default: e = walk_u<ESZ, W, T, P, 4>(a, t, src, dst, total, add, reps, fz, st); break;
  }
  if (e != cudaSuccess) return fail(GG_ECUDA, std::string("walk launch: ") + cudaGetErrorString(e));
  return GG_OK;
}

// copy-type walks (insert / duplicate / flatten) for every element size
template <int W, bool P = false>
int walk_copy(const gg_array *a, const Tables &t, const char *src, char *dst, uint64_t total,
              Fuse fz, cudaStream_t st) {
  switch (a->esz) {
    case 1: return walk<1, W, uint8_t, P>(a, t, src, dst, total, (uint8_t)0, 0u, fz, st);
    case 2: return walk<2, W, uint16_t, P>(a, t, src, dst, total, (uint16_t)0, 0u, fz, st);
    case 4: return walk<4, W, uint32_t, P>(a, t, src, dst, total, 0u, 0u, fz, st);
    default: return walk<8, W, uint64_t, P>(a, t, src, dst, total, (uint64_t)0, 0u, fz, st);
  }
}

template <int W>
int launch_walk(gg_array *a, const Tables &t, const char *src, char *dst, uint64_t total,
                cudaStream_t st) {
  return walk_copy<W, false>(a, t, src, dst, total, Fuse{0, 0}, st);
}

bool g_defer = true;            // defer + fuse planned metadata (GG_DEFER=0 disables)

uint32_t meta_threads(const gg_array *a) { return std::min<uint32_t>(1024, (a->S + 31) / 32 * 32); }

// launch a deferred metadata pass, if any (on the stream of its walk)
int flush_pending(gg_array *a) {
  if (!a->pend) return GG_OK;
  a->pend = false;
  Tables t = tables_for_launch(a, false);
  CUDA_TRY(launch_k(k_planned_meta, 1, meta_threads(a), 0, a->pend_st, t, a->pend_fz));
  return GG_OK;
}

// after a planned walk: its metadata pass now, or deferred (eager issue) so
// that a following grow can run both in one launch
int finish_planned(gg_array *a, Fuse fz, cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  const bool capturing = a->up.capturing ||
                         (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone);
  if (g_defer && (!capturing || a->defer_in_capture)) {
    a->pend = true;
    a->pend_fz = fz;
    a->pend_st = st;
    return GG_OK;
  }
  Tables t = tables_for_launch(a, false);
  CUDA_TRY(launch_k(k_planned_meta, 1, meta_threads(a), 0, st, t, fz));
  return GG_OK;
}

void host_commit(gg_array *a) {
  uint64_t acc = 0;
  a->prefix[0] = 0;
  for (uint32_t s = 0; s < a->S; ++s) { acc += a->size[s]; a->prefix[s + 1] = acc; }
}

// run an allocating append: upload ctl/zero list if needed, then either one
// fused launch (reserve + allocate + copy [+ commit]) or the unfused
// reserve / zero / copy sequence (failure paths that must zero buckets).
int run_append(gg_array *a, Plan &p, int reserve_mode, int wk, const char *src,
               uint64_t total, cudaStream_t st, uint32_t flags, bool *committed) {
  *committed = false;
  int rc = commit_plan(a, p, st);
  if (rc) return rc;
  Tables t = tables_for_launch(a, p.any_ctl);
  if (p.any_ctl) {
    void *dst[1] = {a->t.ctl};
    const void *srcs[1] = {p.ctl.data()};
    size_t bytes[1] = {a->S * sizeof(uint32_t)};
    if ((rc = a->up.upload(st, 1, dst, srcs, bytes))) return rc;
  }
  // No failure planned: ONE launch copies into host-backed slots and applies
  // the reservation metadata (+ commit) in its last CTA.  Failure paths
  // (ctl words, zeroing, explicit starts) take the separate reserve / zero /
  // copy kernels.
  if (!p.any_ctl && p.zero_pairs.empty() && reserve_mode != 2 && !(flags & GG_F_UNFUSED)) {
    const bool commit = (flags & GG_F_COMMIT) != 0;
    if (total) {
      Fuse fz{reserve_mode, commit ? 1 : 0};
      rc = wk == W_INSERT ? walk_copy<W_INSERT, true>(a, t, src, nullptr, total, fz, st)
                            : walk_copy<W_DUP, true>(a, t, nullptr, nullptr, total, fz, st);
      if (rc) return rc;
      if ((rc = finish_planned(a, fz, st))) return rc;
    } else if (commit) {
      CUDA_TRY(launch_k(k_commit, 1, 1024, 0, st, a->t));
    }
    if (commit) { host_commit(a); *committed = true; }
    return GG_OK;
  }
  CUDA_TRY(launch_k(k_reserve, (a->S + 255) / 256, 256, 0, st, t, reserve_mode));
  CUDA_TRY(cudaGetLastError());
  if (!p.zero_pairs.empty()) {
    uint32_t *d_pairs = nullptr;
    CUDA_TRY(cudaMallocAsync((void **)&d_pairs, p.zero_pairs.size() * 4, st));
    CUDA_TRY(cudaMemcpyAsync(d_pairs, p.zero_pairs.data(), p.zero_pairs.size() * 4,
                             cudaMemcpyHostToDevice, st));
    uint32_t np = (uint32_t)(p.zero_pairs.size() / 2);
    { k_zero_buckets<<<std::min<uint32_t>(np, 1024), kThreads, 0, st>>>(t, d_pairs, np); g_launches.fetch_add(1, std::memory_order_relaxed); }
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaFreeAsync(d_pairs, st));
    CUDA_TRY(cudaStreamSynchronize(st));  // zero_pairs host memory is pageable
  }
  rc = wk == W_INSERT ? launch_walk<W_INSERT>(a, t, src, nullptr, total, st)
                      : launch_walk<W_DUP>(a, t, nullptr, nullptr, total, st);
  if (rc) return rc;
  if ((flags & GG_F_COMMIT) && !p.any_fail) {
    host_commit(a);
    CUDA_TRY(launch_k(k_commit, 1, 1024, 0, st, a->t));
    CUDA_TRY(cudaGetLastError());
    *committed = true;
  }
  return GG_OK;
}

int finish_status(gg_array *a, const Plan &p, int32_t *h_status) {
  if (h_status)
    for (uint32_t s = 0; s < a->S; ++s) h_status[s] = p.status[s];
  if (!p.any_fail) return GG_OK;
  return fail(GG_EPARTIAL, "insert failed on some shards; commit withheld");
}

template <typename T>
int launch_rw(gg_array *a, const Tables &t, T addend, uint32_t passes, int mode, uint64_t total,
              cudaStream_t st) {
  if (mode == GG_RW_GLOBAL) {
    const uint64_t nvec = (total * sizeof(T) + 15) / 16;
    // sweep (tools/sweep.py): rw_g peaks at U = 4 (U = 8 spills the per-vector
    // pointers / masks into a lower occupancy)
    const uint32_t U = std::min<uint32_t>(walk_unroll(a, total, W_RW), 4u);
    const uint64_t grid = (nvec + kThreads * U - 1) / (kThreads * U);
    for (uint32_t p = 0; p < passes; ++p) {
      cudaError_t e;
      switch (U) {
        case 2: e = launch_k(k_rw_global<T, 2>, (unsigned)grid, kThreads, 0, st, t, total, addend); break;
        case 8: e = launch_k(k_rw_global<T, 8>, (unsigned)grid, kThreads, 0, st, t, total, addend); break;
        case 1: e = launch_k(k_rw_global<T, 1>, (unsigned)grid, kThreads, 0, st, t, total, addend); break;
        default: e = launch_k(k_rw_global<T, 4>, (unsigned)grid, kThreads, 0, st, t, total, addend); break;
      }
      CUDA_TRY(e);
    }
    return GG_OK;
  }
  const Fuse none{0, 0};
  if (mode == GG_RW_FUSED)
    return walk<sizeof(T), W_RW, T>(a, t, nullptr, nullptr, total, addend, passes, none, st);
  for (uint32_t p = 0; p < passes; ++p) {
    int rc = walk<sizeof(T), W_RW, T>(a, t, nullptr, nullptr, total, addend, 1u, none, st);
    if (rc) return rc;
  }
  return GG_OK;
}

template <typename T>
int launch_flat_add(char *buf, uint64_t n, T a, uint32_t passes, int fused, int dev,
                    cudaStream_t st) {
  (void)dev;
  if (n == 0) return GG_OK;
  const uint64_t ch = kFlatChunk / sizeof(T);
  const uint64_t grid = (n + ch - 1) / ch;      // one chunk per CTA
  if (fused) CUDA_TRY(launch_k(k_flat_add<T>, (unsigned)grid, kThreads, 0, st, buf, n, a, passes));
  else
    for (uint32_t p = 0; p < passes; ++p)
      CUDA_TRY(launch_k(k_flat_add<T>, (unsigned)grid, kThreads, 0, st, buf, n, a, 1u));
  return GG_OK;
}

#define DISPATCH_DTYPE(dt, T, ...)                                          \
  switch (dt) {                                                             \
    case GG_I8: { typedef int8_t T; __VA_ARGS__; break; }                   \
    case GG_U8: { typedef uint8_t T; __VA_ARGS__; break; }                  \
    case GG_I16: { typedef int16_t T; __VA_ARGS__; break; }                 \
    case GG_U16: { typedef uint16_t T; __VA_ARGS__; break; }                \
    case GG_I32: { typedef int32_t T; __VA_ARGS__; break; }                 \
    case GG_U32: { typedef uint32_t T; __VA_ARGS__; break; }                \
    case GG_I64: { typedef long long T; __VA_ARGS__; break; }               \
    case GG_U64: { typedef unsigned long long T; __VA_ARGS__; break; }      \
    case GG_F16: { typedef __half T; __VA_ARGS__; break; }                  \
    case GG_F32: { typedef float T; __VA_ARGS__; break; }                   \
    case GG_F64: { typedef double T; __VA_ARGS__; break; }                  \
    default: return fail(GG_EVALUE, "bad dtype");                           \
  }

// the committed range of every shard must lie in published buckets
// (bucket_vector.py:279-295 raises RuntimeError otherwise)
int check_committed_published(const gg_array *a) {
  for (uint32_t s = 0; s < a->S; ++s) {
    uint64_t n = a->prefix[s + 1] - a->prefix[s];
    uint32_t k = min_buckets_for(a, n);
    if (k == 0) continue;
    uint64_t need = (k >= 64) ? ~uint64_t(0) : ((uint64_t(1) << k) - 1);
    if ((a->flags[s] & need) != need)
      return fail(GG_EUNPUBLISHED, "bucket unpublished while walking shard " + std::to_string(s));
  }
  return GG_OK;
}

}  // namespace

namespace gg {
// Example user kernel of the device API (paper Alg. 1): block b appends the
// elements i of its slice with pred[i] != 0 to shard b % S, warp- or
// block-aggregated.
template <int ESZ, int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_push_if(gg_device_view t, const char *vals,
                                                   const uint8_t *pred, uint64_t n, int block_mode) {
  typedef typename ElemT<ESZ>::T E;
  __shared__ unsigned long long scratch[34];
  const uint32_t s = blockIdx.x % t.S;
  for (uint64_t base = (uint64_t)blockIdx.x * BLOCK; base < n; base += (uint64_t)gridDim.x * BLOCK) {
    const uint64_t i = base + threadIdx.x;
    const bool p = i < n && pred[i];
    const E v = p ? reinterpret_cast<const E *>(vals)[i] : E(0);
    if (block_mode) block_push_back<BLOCK, E>(t, s, p ? 1u : 0u, &v, scratch);
    else warp_push_back<E>(t, s, p, v);
  }
}

}  // namespace gg

// =================================================================== C ABI
extern "C" {

const char *gg_last_error(void) { return g_err.c_str(); }
int gg_version(void) { return GG_VERSION; }
uint64_t gg_kernel_launches(void) { return g_launches.load(); }

int gg_device_sms(int device, int32_t *h_sms) {
  *h_sms = sm_count(device);
  return GG_OK;
}

int gg_create(int device, uint32_t shards, uint32_t fb, uint32_t dtype, uint32_t max_buckets,
              uint64_t arena_va_bytes, gg_array **out) {
  *out = nullptr;
  if (shards < 1) return fail(GG_EVALUE, "shards must be >= 1");
  if (fb < 1 || (fb & (fb - 1))) return fail(GG_EVALUE, "first_bucket_size must be a power of two");
  if (max_buckets < 1 || max_buckets > kMaxBuckets) return fail(GG_EVALUE, "max_buckets must be in [1, 64]");
  uint32_t esz = elem_bytes_of(dtype);
  if (!esz) return fail(GG_EVALUE, "unsupported dtype");
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaFree(0));
  gg_array *a = new gg_array();
  a->dev = device; a->S = shards; a->fb = fb; a->log2fb = ilog2(fb); a->dtype = dtype;
  a->esz = esz; a->MB = max_buckets;
  a->size.assign(shards, 0); a->cap.assign(shards, 0); a->ops.assign(shards, 0);
  a->prefix.assign(shards + 1, 0); a->flags.assign(shards, 0); a->dirty.assign(shards, 0);
  if (arena_va_bytes == 0) arena_va_bytes = kDefaultVaBudget;
  std::vector<uint64_t> bb(max_buckets);
  for (uint32_t b = 0; b < max_buckets; ++b) bb[b] = bucket_bytes(a, b);
  int rc = a->slab.init(device, shards, max_buckets, bb, arena_va_bytes);
  if (rc) { a->slab.destroy(); delete a; return rc; }
  // metadata block
  const size_t S = shards, T = S * max_buckets;
  size_t bytes = 0;
  auto take = [&](size_t n) { size_t o = bytes; bytes += (n + 255) & ~size_t(255); return o; };
  size_t o_size = take(S * 8), o_cap = take(S * 8), o_ops = take(S * 8), o_start = take(S * 8),
         o_count = take(S * 8), o_prefix = take((S + 1) * 8), o_off = take((S + 1) * 8),
         o_ctl = take(S * 4), o_flag = take(T * 4), o_status = take(S * 4), o_ptr = take(T * 8),
         o_misc = take(MISC_N * 8), o_won = take(16), o_scr = take(64), o_am = take(S * 8),
         o_cb = take(max_buckets * 8), o_pm = take(S * 8);
  cudaError_t e = cudaMalloc(&a->dmem, bytes);
  if (e != cudaSuccess) { a->slab.destroy(); delete a; return fail(GG_ECUDA, cudaGetErrorString(e)); }
  cudaMemset(a->dmem, 0, bytes);
  char *base = (char *)a->dmem;
  Tables &t = a->t;
  t.size = (uint64_t *)(base + o_size); t.cap = (uint64_t *)(base + o_cap);
  t.ops = (uint64_t *)(base + o_ops); t.start = (uint64_t *)(base + o_start);
  t.count = (uint64_t *)(base + o_count); t.prefix = (uint64_t *)(base + o_prefix);
  t.offsets = (uint64_t *)(base + o_off); t.ctl = (uint32_t *)(base + o_ctl);
  t.flag = (uint32_t *)(base + o_flag); t.status = (uint32_t *)(base + o_status);
  t.ptr = (char **)(base + o_ptr); t.misc = (unsigned long long *)(base + o_misc);
  t.amask = (unsigned long long *)(base + o_am); t.cbase = (char **)(base + o_cb);
  t.pmask = (unsigned long long *)(base + o_pm);
  t.S = shards; t.log2fb = a->log2fb; t.MB = max_buckets; t.esz = esz;
  a->d_won = (int *)(base + o_won);
  a->d_scratch = base + o_scr;
  if ((rc = a->up.init(device))) { gg_destroy(a); return rc; }
  if (a->slab.small.base) {           // the packed small-class region exists from the start
    std::vector<uint64_t> cb(max_buckets);
    for (uint32_t b = 0; b < max_buckets; ++b) cb[b] = a->slab.class_base(b);
    CUDA_TRY(cudaMemcpy(t.cbase, cb.data(), max_buckets * 8, cudaMemcpyHostToDevice));
  }
  CUDA_TRY(cudaDeviceSynchronize());
  *out = a;
  return GG_OK;
}

int gg_destroy(gg_array *a) {
  if (!a) return GG_OK;
  use_dev(a->dev);
  cudaDeviceSynchronize();
  a->up.destroy();
  if (a->h_scratch) cudaFreeHost(a->h_scratch);
  if (a->dmem) cudaFree(a->dmem);
  a->slab.destroy();
  delete a;
  return GG_OK;
}

int gg_set_alloc_hook(gg_array *a, gg_alloc_hook hook, void *ctx) {
  a->hook = hook; a->hook_ctx = ctx;
  return GG_OK;
}

int gg_set_arena_limit(gg_array *a, uint64_t bytes) {
  a->limit = bytes;
  return GG_OK;
}

int gg_insert_ex(gg_array *a, const void *d_values, const uint64_t *h_offsets,
                 const uint64_t *h_starts, uint32_t flags, int32_t *h_status, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  if (h_offsets[0] != 0) return fail(GG_EVALUE, "offsets[0] must be 0");
  std::vector<uint64_t> counts(a->S);
  for (uint32_t s = 0; s < a->S; ++s) {
    if (h_offsets[s + 1] < h_offsets[s]) return fail(GG_EVALUE, "offsets must be non-decreasing");
    counts[s] = h_offsets[s + 1] - h_offsets[s];
  }
  const uint64_t total = h_offsets[a->S];
  Plan p;
  plan_init(a, p);
  plan_append(a, p, counts.data(), h_starts);
  // upload directory (+ explicit starts / counts)
  int rc;
  if (h_starts) {
    std::vector<uint64_t> st0(a->S, 0);
    for (uint32_t s = 0; s < a->S; ++s) st0[s] = counts[s] ? h_starts[s] : 0;
    void *dst[3] = {a->t.offsets, a->t.start, a->t.count};
    const void *src[3] = {h_offsets, st0.data(), counts.data()};
    size_t bytes[3] = {(a->S + 1) * 8, a->S * 8, a->S * 8};
    if ((rc = a->up.upload(st, 3, dst, src, bytes))) return rc;
  } else {
    void *dst[1] = {a->t.offsets};
    const void *src[1] = {h_offsets};
    size_t bytes[1] = {(a->S + 1) * 8};
    if ((rc = a->up.upload(st, 1, dst, src, bytes))) return rc;
  }
  bool committed;
  if ((rc = run_append(a, p, h_starts ? 2 : 0, W_INSERT, (const char *)d_values, total, st, flags,
                       &committed)))
    return rc;
  if (!h_starts)
    for (uint32_t s = 0; s < a->S; ++s) if (counts[s]) a->ops[s] += 1;
  return finish_status(a, p, h_status);
}

int gg_insert_duplicate_ex(gg_array *a, uint32_t flags, int32_t *h_status, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  {
    // uniform fast path: every shard has the same committed length, size and
    // buckets, no hook / cap / failed shard -> plan shard 0 once
    const uint64_t c = a->prefix[1] - a->prefix[0];
    bool uni = !a->hook && !a->limit && !(flags & GG_F_UNFUSED);
    for (uint32_t s = 0; s < a->S && uni; ++s)
      uni = a->prefix[s + 1] - a->prefix[s] == c && a->size[s] == a->size[0] &&
            a->flags[s] == a->flags[0] && !a->dirty[s];
    if (uni && c) {
      const uint32_t kc = min_buckets_for(a, c);
      const uint64_t need = kc >= 64 ? ~uint64_t(0) : ((uint64_t(1) << kc) - 1);
      if ((a->flags[0] & need) != need)
        return fail(GG_EUNPUBLISHED, "bucket unpublished while walking shard 0");
      const uint64_t start = a->size[0];
      uint32_t b0, b1; uint64_t o;
      host_locate(a, start, b0, o);
      host_locate(a, start + c - 1, b1, o);
      if (b1 < a->MB) {
        uint64_t want = 0;
        for (uint32_t b = b0; b <= b1; ++b) if (!(a->flags[0] >> b & 1)) want |= uint64_t(1) << b;
        int rc = GG_OK;
        uint64_t got = 0;
        for (uint32_t b = b0; b <= b1 && !rc; ++b) {
          if (!(want >> b & 1)) continue;
          bool created = false;
          if (!(rc = a->slab.ensure_region(b, &created)) && !(rc = a->slab.back_range(b, 0, a->S))) {
            if (created) a->cbase_dirty = true;
            got |= uint64_t(1) << b;
          }
        }
        if (!rc) {
          uint64_t elems = 0, bytes = 0;
          for (uint32_t b = b0; b <= b1; ++b)
            if (want >> b & 1) { elems += bucket_elems(a, b); bytes += bucket_bytes(a, b); }
          for (uint32_t s = 0; s < a->S; ++s) {
            a->size[s] += c; a->ops[s] += 1; a->flags[s] |= want; a->cap[s] += elems;
          }
          a->live += bytes * a->S;
          a->alloc_calls += (uint64_t)__builtin_popcountll(want) * a->S;
          if ((rc = push_cbase(a, st))) return rc;
          const bool commit = (flags & GG_F_COMMIT) != 0;
          Tables t = tables_for_launch(a, false);
          if ((rc = walk_copy<W_DUP, true>(a, t, nullptr, nullptr, a->prefix[a->S],
                                           Fuse{1, commit ? 1 : 0}, st)))
            return rc;
          if ((rc = finish_planned(a, Fuse{1, commit ? 1 : 0}, st))) return rc;
          if (commit) host_commit(a);
          if (h_status) memset(h_status, 0, a->S * sizeof(int32_t));
          return GG_OK;
        }
        for (uint32_t b = b0; b <= b1; ++b)     // out of memory: undo, take the exact path
          if (got >> b & 1) a->slab.unback_range(b, 0, a->S);
      }
    }
  }
  int rc = check_committed_published(a);
  if (rc) return rc;
  std::vector<uint64_t> counts(a->S);
  for (uint32_t s = 0; s < a->S; ++s) counts[s] = a->prefix[s + 1] - a->prefix[s];
  Plan p;
  plan_init(a, p);
  plan_append(a, p, counts.data(), nullptr);
  bool committed;
  const uint64_t total = a->prefix[a->S];
  if ((rc = run_append(a, p, 1, W_DUP, nullptr, total, st, flags, &committed))) return rc;
  for (uint32_t s = 0; s < a->S; ++s) if (counts[s]) a->ops[s] += 1;
  return finish_status(a, p, h_status);
}

int gg_insert(gg_array *a, const void *d_values, const uint64_t *h_offsets,
              const uint64_t *h_starts, int32_t *h_status, void *stream) {
  return gg_insert_ex(a, d_values, h_offsets, h_starts, 0, h_status, stream);
}

int gg_insert_duplicate(gg_array *a, int32_t *h_status, void *stream) {
  return gg_insert_duplicate_ex(a, 0, h_status, stream);
}

int gg_commit(gg_array *a, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  uint64_t acc = 0;
  a->prefix[0] = 0;
  for (uint32_t s = 0; s < a->S; ++s) { acc += a->size[s]; a->prefix[s + 1] = acc; }
  CUDA_TRY(launch_k(k_commit, 1, 1024, 0, S_(stream), a->t));
  CUDA_TRY(cudaGetLastError());
  return GG_OK;
}

int gg_reserve(gg_array *a, const uint64_t *h_min_capacity, int64_t *h_failed_shard, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  cudaStream_t st = S_(stream);
  if (h_failed_shard) *h_failed_shard = -1;
  if (a->pend && a->pend_st != st) { int frc_ = flush_pending(a); if (frc_) return frc_; }
  {
    // uniform fast path (every shard the same target and bucket set, no hook,
    // no cap, no failed shard): class-batched backing, no per-shard planning
    bool uni = !a->hook && !a->limit;
    for (uint32_t s = 0; s < a->S && uni; ++s)
      uni = h_min_capacity[s] == h_min_capacity[0] && a->flags[s] == a->flags[0] && !a->dirty[s];
    const uint32_t k = uni ? min_buckets_for(a, h_min_capacity[0]) : 0;
    if (uni && k <= a->MB) {
      const uint64_t want = (k >= 64 ? ~uint64_t(0) : ((uint64_t(1) << k) - 1)) & ~a->flags[0];
      if (!want) return GG_OK;             // (a deferred metadata pass stays deferred)
      int rc = GG_OK;
      uint64_t got = 0;
      for (uint32_t b = 0; b < k && !rc; ++b) {
        if (!(want >> b & 1)) continue;
        bool created = false;
        if (!(rc = a->slab.ensure_region(b, &created)) && !(rc = a->slab.back_range(b, 0, a->S))) {
          if (created) a->cbase_dirty = true;
          got |= uint64_t(1) << b;
        }
      }
      if (!rc) {
        uint64_t elems = 0, bytes = 0;
        for (uint32_t b = 0; b < k; ++b)
          if (want >> b & 1) { elems += bucket_elems(a, b); bytes += bucket_bytes(a, b); }
        for (uint32_t s = 0; s < a->S; ++s) { a->flags[s] |= want; a->cap[s] += elems; }
        a->live += bytes * a->S;
        a->alloc_calls += (uint64_t)__builtin_popcountll(want) * a->S;
        if ((rc = push_cbase(a, st))) return rc;
        Tables t = tables_for_launch(a, true);
        if (a->pend) {                         // metadata of the last append + this grow: one launch
          a->pend = false;
          CUDA_TRY(launch_k(k_meta_grow, 1, meta_threads(a), 0, st, t, a->pend_fz, k));
        } else {
          CUDA_TRY(launch_k(k_grow, (a->S + 255) / 256, 256, 0, st, t, k));
        }
        return GG_OK;
      }
      for (uint32_t b = 0; b < k; ++b)            // out of memory: undo, take the exact path
        if (got >> b & 1) a->slab.unback_range(b, 0, a->S);
    }
  }
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  Plan p;
  plan_init(a, p);
  std::vector<uint32_t> lim(a->S, 0);
  int err = GG_OK;
  bool any = false;
  for (uint32_t s = 0; s < a->S && err == GG_OK; ++s) {
    uint32_t k = min_buckets_for(a, h_min_capacity[s]);
    if (k > a->MB) {                                    // bucket_vector.py:252-255
      err = fail(GG_ECAPACITY, "capacity needs more buckets than the table holds");
      if (h_failed_shard) *h_failed_shard = s;
      break;
    }
    for (uint32_t b = 0; b < k; ++b) {
      if (p.flags[s] >> b & 1) continue;
      if (!plan_alloc(a, p, s, b)) {
        err = fail(GG_ENOMEM, "bucket allocation failed");
        if (h_failed_shard) *h_failed_shard = s;
        break;
      }
      lim[s] = b + 1;
      any = true;
    }
  }
  if (any) {
    int rc = commit_plan(a, p, st);
    if (rc) return rc;
    // uniform target without failures: every shard allocates [0, k) -- no upload
    bool uniform = err == GG_OK;
    for (uint32_t s = 1; s < a->S && uniform; ++s) uniform = h_min_capacity[s] == h_min_capacity[0];
    uint32_t uk = uniform ? min_buckets_for(a, h_min_capacity[0]) : ~0u;
    if (!uniform) {
      void *dst[1] = {a->t.ctl};
      const void *src[1] = {lim.data()};
      size_t bytes[1] = {a->S * 4};
      if ((rc = a->up.upload(st, 1, dst, src, bytes))) return rc;
    }
    Tables t = tables_for_launch(a, true);
    CUDA_TRY(launch_k(k_grow, (a->S + 255) / 256, 256, 0, st, t, uk));
    CUDA_TRY(cudaGetLastError());
    if (!p.zero_pairs.empty()) {
      // grow on a dirty shard: zero the new buckets (reference buckets are np.zeros)
      uint32_t *d_pairs = nullptr;
      CUDA_TRY(cudaMallocAsync((void **)&d_pairs, p.zero_pairs.size() * 4, st));
      CUDA_TRY(cudaMemcpyAsync(d_pairs, p.zero_pairs.data(), p.zero_pairs.size() * 4,
                               cudaMemcpyHostToDevice, st));
      uint32_t np = (uint32_t)(p.zero_pairs.size() / 2);
      { k_zero_buckets<<<std::min<uint32_t>(np, 1024), kThreads, 0, st>>>(t, d_pairs, np); g_launches.fetch_add(1, std::memory_order_relaxed); }
      CUDA_TRY(cudaFreeAsync(d_pairs, st));
      CUDA_TRY(cudaStreamSynchronize(st));
    }
  }
  return err;
}

int gg_new_bucket(gg_array *a, uint32_t s, uint32_t b, int32_t *h_won, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  *h_won = 0;
  if (s >= a->S) return fail(GG_EVALUE, "shard out of range");
  if (b >= a->MB) return fail(GG_ECAPACITY, "bucket outside the table");
  if (a->flags[s] >> b & 1) return GG_OK;
  Plan p;
  plan_init(a, p);
  if (!plan_alloc(a, p, s, b)) return fail(GG_ENOMEM, "bucket allocation failed");
  int rc = commit_plan(a, p, st);
  if (rc) return rc;
  Tables t = tables_for_launch(a, false);
  { k_new_bucket<<<1, 1, 0, st>>>(t, s, b, a->d_won); g_launches.fetch_add(1, std::memory_order_relaxed); }
  CUDA_TRY(cudaGetLastError());
  if (!p.zero_pairs.empty()) {
    uint32_t pair[2] = {s, b};
    uint32_t *d_pairs = (uint32_t *)a->d_scratch;
    CUDA_TRY(cudaMemcpyAsync(d_pairs, pair, 8, cudaMemcpyHostToDevice, st));
    { k_zero_buckets<<<1, kThreads, 0, st>>>(t, d_pairs, 1); g_launches.fetch_add(1, std::memory_order_relaxed); }
  }
  int won = 0;
  if (!a->h_scratch) CUDA_TRY(cudaMallocHost(&a->h_scratch, 64));   // pinned, on first use
  CUDA_TRY(cudaMemcpyAsync(a->h_scratch, a->d_won, sizeof(int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(&won, a->h_scratch, sizeof(int));
  *h_won = won > 0;
  return GG_OK;
}

int gg_fetch_add(gg_array *a, uint32_t s, uint64_t c, uint64_t *h_prev, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  if (s >= a->S) return fail(GG_EVALUE, "shard out of range");
  *h_prev = a->size[s];
  a->size[s] += c;
  a->ops[s] += 1;
  { k_fetch_add<<<1, 1, 0, S_(stream)>>>(a->t, s, c); g_launches.fetch_add(1, std::memory_order_relaxed); }
  CUDA_TRY(cudaGetLastError());
  return GG_OK;
}

int gg_shrink_ex(gg_array *a, const uint64_t *h_new_sizes, uint64_t keep_mapped_bytes,
                 void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  for (uint32_t s = 0; s < a->S; ++s)
    if (h_new_sizes[s] > a->size[s]) return fail(GG_EVALUE, "shrink cannot grow a shard");
  bool uni = true;                             // same size and buckets everywhere: class-batched
  for (uint32_t s = 0; s < a->S && uni; ++s)
    uni = h_new_sizes[s] == h_new_sizes[0] && a->flags[s] == a->flags[0];
  if (uni) {
    const uint32_t keep = min_buckets_for(a, h_new_sizes[0]);
    const uint64_t drop = keep >= 64 ? 0 : (a->flags[0] & ~((uint64_t(1) << keep) - 1));
    uint64_t elems = 0, bytes = 0;
    for (uint32_t b = 0; b < a->MB; ++b)
      if (drop >> b & 1) {
        elems += bucket_elems(a, b);
        bytes += bucket_bytes(a, b);
        a->slab.unback_range(b, 0, a->S);
      }
    for (uint32_t s = 0; s < a->S; ++s) {
      a->flags[s] &= ~drop;
      a->cap[s] -= elems;
      a->size[s] = h_new_sizes[s];
    }
    a->live -= bytes * a->S;
  } else {
    for (uint32_t s = 0; s < a->S; ++s) {
      uint32_t keep = min_buckets_for(a, h_new_sizes[s]);
      for (uint32_t b = keep; b < a->MB; ++b)
        if (a->flags[s] >> b & 1) {
          a->flags[s] &= ~(uint64_t(1) << b);
          a->cap[s] -= bucket_elems(a, b);
          a->live -= bucket_bytes(a, b);
          a->slab.unback(s, b);
        }
      a->size[s] = h_new_sizes[s];
    }
  }
  void *dst[1] = {a->t.count};
  const void *src[1] = {h_new_sizes};
  size_t bytes[1] = {a->S * 8};
  int rc = a->up.upload(st, 1, dst, src, bytes);
  if (rc) return rc;
  Tables t = tables_for_launch(a, false);
  CUDA_TRY(launch_k(k_shrink, 1, std::min<uint32_t>(1024, (a->S + 31) / 32 * 32), 0, st, t,
                    (const uint64_t *)a->t.count));
  uint64_t acc = 0;
  for (uint32_t s = 0; s < a->S; ++s) { acc += a->size[s]; a->prefix[s + 1] = acc; }
  // unmap emptied chunks down to keep_mapped_bytes (waits for the device:
  // queued work may still read the released buckets).  Never under graph
  // capture, where the chunks stay cached until gg_trim.
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  cudaStreamIsCapturing(st, &cap);
  if (cap == cudaStreamCaptureStatusNone && a->slab.cached && a->slab.mapped > keep_mapped_bytes) {
    CUDA_TRY(cudaDeviceSynchronize());
    a->slab.trim_to(keep_mapped_bytes);
  }
  return GG_OK;
}

int gg_shrink(gg_array *a, const uint64_t *h_new_sizes, void *stream) {
  return gg_shrink_ex(a, h_new_sizes, 0, stream);
}

int gg_trim(gg_array *a) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  if (!a->slab.cached) return GG_OK;
  CUDA_TRY(cudaDeviceSynchronize());
  a->slab.trim();
  return GG_OK;
}

int gg_insert_lanes(gg_array *a, const void *d_values, const uint32_t *d_counts,
                    const uint64_t *h_lane_offsets, uint64_t values_per_lane,
                    int32_t *h_status, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  if (h_lane_offsets[0] != 0) return fail(GG_EVALUE, "lane offsets must start at 0");
  for (uint32_t s = 0; s < a->S; ++s)
    if (h_lane_offsets[s + 1] < h_lane_offsets[s]) return fail(GG_EVALUE, "lane offsets must be non-decreasing");
  if (values_per_lane == 0 || values_per_lane > 0xffffffffu) return fail(GG_EVALUE, "bad values_per_lane");
  void *dst[1] = {a->t.offsets};
  const void *src[1] = {h_lane_offsets};
  size_t bytes[1] = {(a->S + 1) * 8};
  int rc = a->up.upload(st, 1, dst, src, bytes);
  if (rc) return rc;
  // pass 1: per-shard totals -> host (one sync per launch, not per insert)
  { k_lanes_count<<<a->S, 1024, 0, st>>>(a->t, d_counts); g_launches.fetch_add(1, std::memory_order_relaxed); }
  CUDA_TRY(cudaGetLastError());
  std::vector<uint64_t> counts(a->S);
  CUDA_TRY(cudaMemcpyAsync(counts.data(), a->t.count, a->S * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  for (uint32_t s = 0; s < a->S; ++s)
    if (counts[s] > (h_lane_offsets[s + 1] - h_lane_offsets[s]) * values_per_lane)
      return fail(GG_EVALUE, "a lane count exceeds values_per_lane");
  Plan p;
  plan_init(a, p);
  plan_append(a, p, counts.data(), nullptr);
  if ((rc = commit_plan(a, p, st))) return rc;
  Tables t = tables_for_launch(a, p.any_ctl);
  if (p.any_ctl) {
    void *d2[1] = {a->t.ctl};
    const void *s2[1] = {p.ctl.data()};
    size_t b2[1] = {a->S * sizeof(uint32_t)};
    if ((rc = a->up.upload(st, 1, d2, s2, b2))) return rc;
  }
  if (!p.zero_pairs.empty()) return fail(GG_EVALUE, "lane insert into a shard with failed reservations");
  switch (a->esz) {
    case 1: { k_lanes_insert<1><<<a->S, 1024, 0, st>>>(t, (const char *)d_values, d_counts, (uint32_t)values_per_lane); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 2: { k_lanes_insert<2><<<a->S, 1024, 0, st>>>(t, (const char *)d_values, d_counts, (uint32_t)values_per_lane); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 4: { k_lanes_insert<4><<<a->S, 1024, 0, st>>>(t, (const char *)d_values, d_counts, (uint32_t)values_per_lane); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 8: { k_lanes_insert<8><<<a->S, 1024, 0, st>>>(t, (const char *)d_values, d_counts, (uint32_t)values_per_lane); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
  }
  CUDA_TRY(cudaGetLastError());
  for (uint32_t s = 0; s < a->S; ++s) if (counts[s]) a->ops[s] += 1;
  return finish_status(a, p, h_status);
}

int gg_rw_add(gg_array *a, const void *h_addend, uint32_t passes, int32_t mode, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  int rc = check_committed_published(a);
  if (rc) return rc;
  const uint64_t total = a->prefix[a->S];
  if (total == 0 || passes == 0) return GG_OK;
  Tables t = tables_for_launch(a, false);
  DISPATCH_DTYPE(a->dtype, T, {
    T v; memcpy(&v, h_addend, sizeof(T));
    rc = launch_rw<T>(a, t, v, passes, mode, total, S_(stream));
  });
  return rc;
}

int gg_flatten(gg_array *a, void *d_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  int rc = check_committed_published(a);
  if (rc) return rc;
  Tables t = tables_for_launch(a, false);
  return launch_walk<W_FLATTEN>(a, t, nullptr, (char *)d_out, a->prefix[a->S], S_(stream));
}

int gg_flatten_range(gg_array *a, uint64_t lo, uint64_t hi, void *d_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  if (lo > hi || hi > a->prefix[a->S]) return fail(GG_EINDEX, "flatten range outside the committed size");
  if (lo == hi) return GG_OK;
  int rc = check_committed_published(a);
  if (rc) return rc;
  Tables t = tables_for_launch(a, false);
  Fuse fz{0, 0};
  fz.g0 = lo;
  // the walk stores element g at flat_dst + g * esz: shift the base so that
  // element lo lands at d_out (never dereferenced below lo)
  char *base = (char *)d_out - lo * a->esz;
  return walk_copy<W_FLATTEN, false>(a, t, nullptr, base, hi, fz, S_(stream));
}

int gg_gather(gg_array *a, const int64_t *d_idx, uint64_t n, void *d_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  if (n == 0) return GG_OK;
  Tables t = tables_for_launch(a, false);
  int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count(a->dev) * 8);
  switch (a->esz) {
    case 1: { k_gather<1><<<grid, 256, 0, S_(stream)>>>(t, d_idx, n, (char *)d_out, nullptr, 0); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 2: { k_gather<2><<<grid, 256, 0, S_(stream)>>>(t, d_idx, n, (char *)d_out, nullptr, 0); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 4: { k_gather<4><<<grid, 256, 0, S_(stream)>>>(t, d_idx, n, (char *)d_out, nullptr, 0); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 8: { k_gather<8><<<grid, 256, 0, S_(stream)>>>(t, d_idx, n, (char *)d_out, nullptr, 0); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
  }
  CUDA_TRY(cudaGetLastError());
  return GG_OK;
}

int gg_scatter(gg_array *a, const int64_t *d_idx, uint64_t n, const void *d_vals, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  if (n == 0) return GG_OK;
  Tables t = tables_for_launch(a, false);
  int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count(a->dev) * 8);
  switch (a->esz) {
    case 1: { k_gather<1><<<grid, 256, 0, S_(stream)>>>(t, d_idx, n, nullptr, (const char *)d_vals, 1); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 2: { k_gather<2><<<grid, 256, 0, S_(stream)>>>(t, d_idx, n, nullptr, (const char *)d_vals, 1); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 4: { k_gather<4><<<grid, 256, 0, S_(stream)>>>(t, d_idx, n, nullptr, (const char *)d_vals, 1); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 8: { k_gather<8><<<grid, 256, 0, S_(stream)>>>(t, d_idx, n, nullptr, (const char *)d_vals, 1); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
  }
  CUDA_TRY(cudaGetLastError());
  return GG_OK;
}

namespace {
int elem_addr(gg_array *a, uint32_t s, uint64_t i, char **out, cudaStream_t st) {
  if (s >= a->S) return fail(GG_EVALUE, "shard out of range");
  if (i >= a->size[s]) return fail(GG_EINDEX, "index outside size");
  uint32_t b; uint64_t o;
  host_locate(a, i, b, o);
  if (b >= a->MB || !(a->flags[s] >> b & 1))
    return fail(GG_EUNPUBLISHED, "index is reserved but its bucket is unpublished");
  char *p = nullptr;
  if (!a->h_scratch) CUDA_TRY(cudaMallocHost(&a->h_scratch, 64));   // pinned, on first use
  CUDA_TRY(cudaMemcpyAsync(a->h_scratch, a->t.ptr + (size_t)s * a->MB + b, sizeof(char *),
                           cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(&p, a->h_scratch, sizeof(char *));
  *out = p + o * a->esz;
  return GG_OK;
}
}  // namespace

int gg_get(gg_array *a, uint32_t s, uint64_t i, void *h_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  char *p;
  int rc = elem_addr(a, s, i, &p, st);
  if (rc) return rc;
  if (!a->h_scratch) CUDA_TRY(cudaMallocHost(&a->h_scratch, 64));   // pinned, on first use
  CUDA_TRY(cudaMemcpyAsync(a->h_scratch, p, a->esz, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  memcpy(h_out, a->h_scratch, a->esz);
  return GG_OK;
}

int gg_set(gg_array *a, uint32_t s, uint64_t i, const void *h_val, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  char *p;
  int rc = elem_addr(a, s, i, &p, st);
  if (rc) return rc;
  if (!a->h_scratch) CUDA_TRY(cudaMallocHost(&a->h_scratch, 64));   // pinned, on first use
  memcpy(a->h_scratch, h_val, a->esz);
  CUDA_TRY(cudaMemcpyAsync(p, a->h_scratch, a->esz, cudaMemcpyHostToDevice, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  return GG_OK;
}

uint64_t gg_device_view_bytes(void) { return sizeof(gg_device_view); }

int gg_device_view_get(gg_array *a, const uint64_t *h_max_sizes, void *h_view, uint64_t view_bytes) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  if (view_bytes != sizeof(gg_device_view)) return fail(GG_EVALUE, "view size mismatch (ggarray_device.cuh)");
  if (!a->headroom.empty()) return fail(GG_EVALUE, "a device view is outstanding (call gg_device_view_sync)");
  // back every slot the launch may take: buckets [0, min_buckets_for(max)) per
  // shard, in shard then bucket order, while the live-bytes cap allows
  std::vector<unsigned long long> am(a->S);
  uint64_t live = a->live;
  bool stop = false;
  for (uint32_t s = 0; s < a->S; ++s) {
    am[s] = a->flags[s];
    if (!h_max_sizes || stop) continue;
    const uint32_t k = std::min<uint32_t>(min_buckets_for(a, h_max_sizes[s]), a->MB);
    for (uint32_t b = 0; b < k; ++b) {
      if (a->flags[s] >> b & 1) continue;
      const uint64_t nb = bucket_bytes(a, b);
      if ((a->limit && live + nb > a->limit) || back_bucket(a, s, b) != GG_OK) { stop = true; break; }
      live += nb;
      am[s] |= 1ull << b;
      a->headroom.push_back(s);
      a->headroom.push_back(b);
    }
  }
  int rc = push_cbase(a, 0);
  if (rc) return rc;
  CUDA_TRY(cudaMemcpy(a->t.amask, am.data(), a->S * 8, cudaMemcpyHostToDevice));
  CUDA_TRY(cudaDeviceSynchronize());
  gg_device_view v = a->t;
  v.ctl = nullptr;                          // amask gates the device allocator
  memcpy(h_view, &v, sizeof v);
  return GG_OK;
}

// refresh the host mirrors from the device after user kernels appended
int gg_device_view_sync(gg_array *a, int32_t *h_status, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  CUDA_TRY(cudaStreamSynchronize(st));
  const size_t S = a->S;
  std::vector<uint32_t> f(S * a->MB), status(S);
  std::vector<unsigned long long> misc(MISC_N);
  CUDA_TRY(cudaMemcpy(a->size.data(), a->t.size, S * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(a->cap.data(), a->t.cap, S * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(a->ops.data(), a->t.ops, S * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(f.data(), a->t.flag, f.size() * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(status.data(), a->t.status, S * 4, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemcpy(misc.data(), a->t.misc, MISC_N * 8, cudaMemcpyDeviceToHost));
  CUDA_TRY(cudaMemset(a->t.status, 0, S * 4));
  bool any = false;
  for (size_t s = 0; s < S; ++s) {
    uint64_t m = 0;
    for (uint32_t b = 0; b < a->MB; ++b)
      if (f[s * a->MB + b] == kFlagPublished) m |= uint64_t(1) << b;
    a->flags[s] = m;
    if (h_status) h_status[s] = (int32_t)status[s];
    if (status[s]) { any = true; a->dirty[s] = 1; }
  }
  a->alloc_calls = misc[MISC_ALLOCS];
  // headroom the kernel took becomes live; the rest is unmapped again
  for (size_t i = 0; i < a->headroom.size(); i += 2) {
    const uint32_t s = a->headroom[i], b = a->headroom[i + 1];
    if (a->flags[s] >> b & 1) a->live += bucket_bytes(a, b);
    else a->slab.unback(s, b);
  }
  a->headroom.clear();
  if (a->slab.cached) a->slab.trim();
  return any ? fail(GG_EPARTIAL, "device-side appends failed on some shards") : GG_OK;
}

int gg_push_if(gg_array *a, const void *d_vals, const uint8_t *d_pred, uint64_t n, int32_t mode,
               uint32_t grid, int32_t *h_status, void *stream) {
  cudaStream_t st = S_(stream);
  if (n == 0) return GG_OK;
  const uint32_t B = 256;
  if (!grid) grid = (uint32_t)std::min<uint64_t>((n + B - 1) / B, (uint64_t)a->S * 64);
  // worst case: every candidate of shard s appended
  std::vector<uint64_t> maxsz(a->S, 0);
  {
    std::lock_guard<std::mutex> g(a->mu);
    const uint64_t per_round = (uint64_t)grid * B;
    for (uint32_t blk = 0; blk < grid; ++blk) {
      uint64_t lo = (uint64_t)blk * B, c = 0;
      for (uint64_t base = lo; base < n; base += per_round) c += std::min<uint64_t>(B, n - base);
      maxsz[blk % a->S] += c;
    }
    for (uint32_t s = 0; s < a->S; ++s) maxsz[s] += a->size[s];
  }
  gg_device_view v;
  int rc = gg_device_view_get(a, maxsz.data(), &v, sizeof v);
  if (rc) return rc;
  switch (a->esz) {
    case 1: { k_push_if<1, 256><<<grid, B, 0, st>>>(v, (const char *)d_vals, d_pred, n, mode); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 2: { k_push_if<2, 256><<<grid, B, 0, st>>>(v, (const char *)d_vals, d_pred, n, mode); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 4: { k_push_if<4, 256><<<grid, B, 0, st>>>(v, (const char *)d_vals, d_pred, n, mode); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 8: { k_push_if<8, 256><<<grid, B, 0, st>>>(v, (const char *)d_vals, d_pred, n, mode); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
  }
  CUDA_TRY(cudaGetLastError());
  return gg_device_view_sync(a, h_status, stream);
}

int gg_set_tuning(int32_t ls, int32_t unroll, uint32_t tile_bytes, uint32_t threads) {
  (void)ls; (void)tile_bytes; (void)threads;
  if (unroll != -1 && unroll != 1 && unroll != 2 && unroll != 4 && unroll != 8)
    return fail(GG_EVALUE, "bad tuning");
  g_tune.unroll = unroll;
  return GG_OK;
}

int gg_set_pdl(int32_t on) {
  g_pdl = on != 0;
  return GG_OK;
}

int gg_set_defer(int32_t on) {
  g_defer = on != 0;
  return GG_OK;
}

int gg_capture_mode(gg_array *a, int32_t on) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  a->defer_in_capture = on == 2;
  if (on && !a->up.capturing) return a->up.begin_capture();
  if (!on) a->up.capturing = false;
  return GG_OK;
}

int gg_flush(gg_array *a) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  return flush_pending(a);
}

int gg_capture_release(gg_array *a) {
  std::lock_guard<std::mutex> g(a->mu);
  cudaDeviceSynchronize();
  a->up.release_captured();
  return GG_OK;
}

int gg_summary(gg_array *a, uint64_t *o) {
  std::lock_guard<std::mutex> g(a->mu);
  uint64_t sz = 0, cp = 0;
  for (uint32_t s = 0; s < a->S; ++s) { sz += a->size[s]; cp += a->cap[s]; }
  o[0] = a->prefix[a->S]; o[1] = sz; o[2] = cp;
  return GG_OK;
}

int gg_info(gg_array *a, uint32_t *o) {
  o[0] = a->S; o[1] = a->fb; o[2] = a->dtype; o[3] = a->MB;
  return GG_OK;
}

int gg_host_state(gg_array *a, uint64_t *sz, uint64_t *cp, uint64_t *fl, uint64_t *pre,
                  uint64_t *ops) {
  std::lock_guard<std::mutex> g(a->mu);
  const size_t S = a->S;
  if (sz) memcpy(sz, a->size.data(), S * 8);
  if (cp) memcpy(cp, a->cap.data(), S * 8);
  if (fl) memcpy(fl, a->flags.data(), S * 8);
  if (pre) memcpy(pre, a->prefix.data(), (S + 1) * 8);
  if (ops) memcpy(ops, a->ops.data(), S * 8);
  return GG_OK;
}

int gg_device_state(gg_array *a, uint64_t *sz, uint64_t *cp, uint64_t *fl, uint64_t *pre,
                    uint64_t *ops, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  cudaStream_t st = S_(stream);
  CUDA_TRY(cudaStreamSynchronize(st));
  const size_t S = a->S;
  if (sz) CUDA_TRY(cudaMemcpy(sz, a->t.size, S * 8, cudaMemcpyDeviceToHost));
  if (cp) CUDA_TRY(cudaMemcpy(cp, a->t.cap, S * 8, cudaMemcpyDeviceToHost));
  if (pre) CUDA_TRY(cudaMemcpy(pre, a->t.prefix, (S + 1) * 8, cudaMemcpyDeviceToHost));
  if (ops) CUDA_TRY(cudaMemcpy(ops, a->t.ops, S * 8, cudaMemcpyDeviceToHost));
  if (fl) {
    std::vector<uint32_t> f(S * a->MB);
    CUDA_TRY(cudaMemcpy(f.data(), a->t.flag, f.size() * 4, cudaMemcpyDeviceToHost));
    for (size_t s = 0; s < S; ++s) {
      uint64_t m = 0;
      for (uint32_t b = 0; b < a->MB; ++b)
        if (f[s * a->MB + b] == kFlagPublished) m |= uint64_t(1) << b;
      fl[s] = m;
    }
  }
  return GG_OK;
}

int gg_prefix_copy(gg_array *a, void *d_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  CUDA_TRY(cudaMemcpyAsync(d_out, a->t.prefix, (a->S + 1) * 8, cudaMemcpyDeviceToDevice, S_(stream)));
  return GG_OK;
}

int gg_bucket_ptrs(gg_array *a, uint64_t *h_ptrs, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  CUDA_TRY(cudaStreamSynchronize(S_(stream)));
  CUDA_TRY(cudaMemcpy(h_ptrs, a->t.ptr, (size_t)a->S * a->MB * 8, cudaMemcpyDeviceToHost));
  return GG_OK;
}

int gg_mem_stats(gg_array *a, uint64_t *o, void *stream) {
  (void)stream;
  std::lock_guard<std::mutex> g(a->mu);
  uint64_t cap = 0, need = 0;
  for (uint32_t s = 0; s < a->S; ++s) { cap += a->cap[s]; need += a->size[s]; }
  o[0] = cap * a->esz; o[1] = a->slab.mapped; o[2] = a->live; o[3] = need * a->esz;
  o[4] = a->alloc_calls; o[5] = a->slab.cached;
  return GG_OK;
}

int gg_slab_stats(gg_array *a, uint64_t *o) {
  std::lock_guard<std::mutex> g(a->mu);
  const Slab &sl = a->slab;
  o[0] = sl.mapped; o[1] = sl.cached; o[2] = sl.n_map; o[3] = sl.n_unmap;
  o[4] = sl.ns_map; o[5] = sl.ns_unmap; o[6] = sl.n_regions; o[7] = sl.va_used;
  return GG_OK;
}

// ---------------------------------------------------------------- baselines
int gg_flat_insert(void *d_buf, uint64_t capacity, uint64_t *d_counter, const void *d_vals,
                   uint64_t n, uint32_t esz, int32_t algo, void *stream) {
  if (n == 0) return GG_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t st = S_(stream);
  if (algo == GG_ALGO_BATCH) {
    // contiguous append at the host-known counter value is done by the caller
    // with gg_buf_copy; here: device-side single reservation + copy
    return fail(GG_EVALUE, "BATCH algo is host-side (reserve + gg_buf_copy)");
  }
  int grid = (int)std::min<uint64_t>((n + 255) / 256, (uint64_t)sm_count(dev) * 16);
  switch (esz) {
    case 1: { k_flat_insert<1><<<grid, 256, 0, st>>>((char *)d_buf, capacity, (unsigned long long *)d_counter, (const char *)d_vals, n, algo, (uint64_t)0); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 2: { k_flat_insert<2><<<grid, 256, 0, st>>>((char *)d_buf, capacity, (unsigned long long *)d_counter, (const char *)d_vals, n, algo, (uint64_t)0); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 4: { k_flat_insert<4><<<grid, 256, 0, st>>>((char *)d_buf, capacity, (unsigned long long *)d_counter, (const char *)d_vals, n, algo, (uint64_t)0); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    case 8: { k_flat_insert<8><<<grid, 256, 0, st>>>((char *)d_buf, capacity, (unsigned long long *)d_counter, (const char *)d_vals, n, algo, (uint64_t)0); g_launches.fetch_add(1, std::memory_order_relaxed); } break;
    default: return fail(GG_EVALUE, "bad element size");
  }
  CUDA_TRY(cudaGetLastError());
  return GG_OK;
}

int gg_flat_add(void *d_buf, uint64_t n, uint32_t dtype, const void *h_addend, uint32_t passes,
                int32_t fused, void *stream) {
  int dev = 0;
  cudaGetDevice(&dev);
  int rc = GG_OK;
  DISPATCH_DTYPE(dtype, T, {
    T v; memcpy(&v, h_addend, sizeof(T));
    rc = launch_flat_add<T>((char *)d_buf, n, v, passes, fused, dev, S_(stream));
  });
  return rc;
}

// ---- peer memory for the multi-GPU gather (CUDA IPC over NVLink / NVSwitch)
int gg_ipc_alloc(uint64_t bytes, void **d_out) {
  *d_out = nullptr;
  CUDA_TRY(cudaMalloc(d_out, bytes ? bytes : 16));   // IPC needs a plain cudaMalloc allocation
  return GG_OK;
}
int gg_ipc_free(void *d_ptr) {
  CUDA_TRY(cudaFree(d_ptr));
  return GG_OK;
}
int gg_ipc_handle_bytes(void) { return (int)sizeof(cudaIpcMemHandle_t); }
int gg_ipc_get_handle(void *d_ptr, void *h_handle) {
  cudaIpcMemHandle_t h;
  CUDA_TRY(cudaIpcGetMemHandle(&h, d_ptr));
  memcpy(h_handle, &h, sizeof h);
  return GG_OK;
}
int gg_ipc_open(const void *h_handle, void **d_out) {
  cudaIpcMemHandle_t h;
  memcpy(&h, h_handle, sizeof h);
  *d_out = nullptr;
  CUDA_TRY(cudaIpcOpenMemHandle(d_out, h, cudaIpcMemLazyEnablePeerAccess));
  return GG_OK;
}
int gg_ipc_close(void *d_ptr) {
  CUDA_TRY(cudaIpcCloseMemHandle(d_ptr));
  return GG_OK;
}

int gg_buf_alloc(uint64_t bytes, void *stream, void **d_out) {
  CUDA_TRY(cudaMallocAsync(d_out, bytes ? bytes : 16, S_(stream)));
  return GG_OK;
}
int gg_buf_free(void *d_ptr, void *stream) {
  CUDA_TRY(cudaFreeAsync(d_ptr, S_(stream)));
  return GG_OK;
}
int gg_buf_copy(void *d_dst, const void *d_src, uint64_t bytes, void *stream) {
  if (!bytes) return GG_OK;
  CUDA_TRY(cudaMemcpyAsync(d_dst, d_src, bytes, cudaMemcpyDeviceToDevice, S_(stream)));
  return GG_OK;
}

}  // extern "C"

struct gg_vmm {
  Arena arena;
};

extern "C" {
int gg_vmm_create(int device, uint64_t va_bytes, gg_vmm **out) {
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaFree(0));
  gg_vmm *v = new gg_vmm();
  int rc = v->arena.init(device, va_bytes);
  if (rc) { delete v; return rc; }
  *out = v;
  return GG_OK;
}
int gg_vmm_ensure(gg_vmm *v, uint64_t bytes) { return v->arena.ensure(bytes); }
int gg_vmm_info(gg_vmm *v, uint64_t *b, uint64_t *m, uint64_t *g) {
  *b = (uint64_t)v->arena.base; *m = v->arena.mapped; *g = v->arena.gran;
  return GG_OK;
}
int gg_vmm_destroy(gg_vmm *v) {
  if (!v) return GG_OK;
  cudaDeviceSynchronize();
  v->arena.destroy();
  delete v;
  return GG_OK;
}
}  // extern "C"
