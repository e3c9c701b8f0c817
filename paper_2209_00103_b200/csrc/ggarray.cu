// ggarray.cu -- B200 (sm_100a) GGArray: the array handle, the host planner and
// the C ABI of include/ggarray.h over the kernels of gg_device.cuh and the
// slab / upload runtime of gg_host.cuh (one translation unit).
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
#include "gg_common.cuh"
#include "gg_device.cuh"
#include "gg_host.cuh"

using namespace gg;

// pending tiled lanes inserts that may chain before their sizes are read back
constexpr uint32_t kLanesChain = 8;

struct gg_array {
  int dev;
  uint32_t S, fb, log2fb, dtype, esz, MB;
  // exact host mirrors
  std::vector<uint64_t> size, cap, ops, prefix, flags;  // flags: bitmask per shard
  std::vector<uint8_t> dirty;                            // shard saw a failed reservation
  uint64_t live = 0;                                     // bytes of live buckets
  std::vector<uint32_t> headroom;                        // (b, s0, s1) runs backed for a device view
  bool cbase_dirty = false;                              // a class region appeared
  // metadata pass of the last planned append, not launched yet (eager issue
  // only): fused into the next grow, launched by any other device-touching call
  bool pend = false;
  Fuse pend_fz{0, 0};
  cudaStream_t pend_st = nullptr;
  bool defer_in_capture = false;                         // capture mode 2: caller flushes in-capture
  // double-buffered size / prefix (the planned walk's metadata CTA writes the
  // next pair while its copy CTAs read the current one); t.size / t.prefix
  // always point at the current pair
  uint64_t *sz_buf[2] = {nullptr, nullptr}, *pf_buf[2] = {nullptr, nullptr};
  int cur = 0;
  int cap_parity = 0;                                    // buffer parity when capture mode 2 began
  // a uniform grow not launched yet: published by the next planned walk's
  // metadata CTA, or launched (k_grow) by any other device-touching call
  uint32_t pend_grow = 0;
  cudaStream_t pend_grow_st = nullptr;
  uint64_t alloc_calls = 0;
  uint64_t limit = 0;                                    // live-bytes cap (0 = none)
  gg_alloc_hook hook = nullptr;
  void *hook_ctx = nullptr;
  Slab slab;
  Uploader up;
  Tables t;          // device pointers (kernel argument)
  void *dmem = nullptr;
  // stream order between calls: every device-touching call on stream st waits
  // for the previous call's stream when it differs (one event), so deferred
  // passes and a later call on another stream never run concurrently
  cudaStream_t last_st = nullptr;
  bool have_last = false;
  bool captured = false;                                 // ever issued under stream capture
  cudaEvent_t ord_ev = nullptr;
  bool view_out = false;                                 // gg_device_view_get without a sync yet
  // A tiled lanes insert (paper Alg. 1) is planned on the upper bound lanes x
  // values_per_lane; the sizes it reached come back through a pinned buffer
  // behind an event and are applied by resolve_lanes (at the next call that
  // reads the host mirrors), which also unbacks the headroom no bucket took.
  // Consecutive tiled lanes inserts chain without that round trip: the next
  // one plans on the pending upper bounds (lanes_ub, buckets already backed
  // for them in lanes_hb) and queues its own readback (up to kLanesChain
  // pending calls; resolve_lanes applies them in order).
  bool lanes_pend = false;
  uint32_t lanes_n = 0;                                  // pending tiled lanes calls
  std::vector<uint64_t> lanes_ub, lanes_hb;              // [S] pending upper bounds / backed-bucket masks
  bool view_pend = false;                                // push_if mirrors pending behind lanes_ev
  uint32_t view_n = 0;                                   // pending push_if calls (they chain like lanes)
  std::vector<uint64_t> view_ub, view_hb;                // [S] pending upper bounds / headroom-bucket masks
  cudaEvent_t lanes_ev = nullptr;
  uint64_t *h_lanes = nullptr;                           // pinned [kLanesChain x S]
  std::vector<uint32_t> lanes_head;                      // (b, s0, s1) runs backed for the upper bound
  uint64_t lanes_keep = 0;                               // mapped bytes before that backing
  uint64_t view_keep = 0;                                // mapped bytes before a device view's headroom
  char *h_view = nullptr;                                // pinned staging of view_finish
  char *d_vpack = nullptr;                               // device staging of view_finish (in dmem)
  size_t h_view_cap = 0;
  // the last shrink asked to keep released chunks cached (release=False):
  // headroom returned by lanes inserts / device views stays cached too
  bool keep_cached = false;
  void *lanes_dmem = nullptr;                            // arrive[S] | tpre[S+1] | tiles[]
  size_t lanes_tiles_cap = 0;
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

// Runs of consecutive shards that will allocate the same bucket class are
// mapped as extents up front (ragged plans otherwise map one grid chunk per
// driver call); the per-shard backing below then only takes references.
// Skipped with an allocator hook or an arena limit (exact per-shard failure
// semantics first).  GG_PREMAP_CHUNKS caps an extent (default 8 grid chunks
// = 1/2..1 class region; 0 = off).
void plan_premap(gg_array *a, const std::vector<uint64_t> &need, uint64_t any) {
  static const size_t cap = [] { const char *e = getenv("GG_PREMAP_CHUNKS"); return e ? (size_t)atol(e) : (size_t)8; }();
  if (!cap || a->hook || a->limit) return;
  for (uint64_t mm = any; mm; mm &= mm - 1) {
    const uint32_t b = (uint32_t)__builtin_ctzll(mm);
    bool created = false;
    if (a->slab.ensure_region(b, &created)) continue;
    if (created) a->cbase_dirty = true;
    for (uint32_t s = 0; s < a->S;) {
      if (!(need[s] >> b & 1)) { ++s; continue; }
      uint32_t e = s;
      while (e + 1 < a->S && (need[e + 1] >> b & 1)) ++e;
      a->slab.premap_range(b, s, e + 1, cap);
      s = e + 1;
    }
  }
}

// Batched (run) backing of new bucket classes: 1 = on (default), 0 = one
// slab call per bucket, 2 = runs path with every run treated as unbackable
// (exercises the per-shard fallback; test hook).  gg_set_batch_backing.
int g_batch_backing = 1;
bool run_backed(gg_array *a, uint32_t b, uint32_t s0, uint32_t s1) {
  return g_batch_backing != 2 && a->slab.back_range(b, s0, s1) == GG_OK;
}

// Plan an append of counts[s] at starts (explicit) or at size[s] (reserve).
void plan_append(gg_array *a, Plan &p, const uint64_t *counts, const uint64_t *starts) {
  // no allocator hook / arena limit: the new buckets are backed class by
  // class in runs of consecutive shards (one batched refcount pass per run
  // instead of one slab call per bucket; a run that cannot be backed falls
  // back to per-shard backing, which fails exactly the shards concerned),
  // and each shard's plan is updated once from the mask of classes it took
  const bool runs = g_batch_backing && !a->hook && !a->limit;
  std::vector<uint64_t> need(runs ? a->S : 0, 0);
  uint64_t any = 0;
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
    if (runs) {
      need[s] = ((b1 >= 63 ? ~0ull : ((2ull << b1) - 1)) & ~((1ull << b0) - 1)) & ~p.flags[s];
      any |= need[s];
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
  if (!runs || !any) return;
  plan_premap(a, need, any);
  std::vector<uint32_t> fail_b(a->S, ~0u);
  for (uint64_t mm = any; mm; mm &= mm - 1) {   // ascending classes
    const uint32_t b = (uint32_t)__builtin_ctzll(mm);
    bool created = false;
    const bool region = a->slab.ensure_region(b, &created) == GG_OK;
    if (created) a->cbase_dirty = true;
    auto wants = [&](uint32_t x) { return (need[x] >> b & 1) && fail_b[x] == ~0u; };
    for (uint32_t s = 0; s < a->S;) {
      if (!wants(s)) { ++s; continue; }
      uint32_t e = s + 1;
      while (e < a->S && wants(e)) ++e;
      if (!region || !run_backed(a, b, s, e))
        for (uint32_t x = s; x < e; ++x)
          if (!region || a->slab.back(x, b) != GG_OK) fail_b[x] = b;
      s = e;
    }
  }
  // per-class element / byte prefix sums once, then one update per shard (a
  // contiguous run of classes -- the usual case -- in closed form)
  uint64_t pe[65], pb[65];
  pe[0] = pb[0] = 0;
  for (uint32_t b = 0; b < 64; ++b) {
    pe[b + 1] = pe[b] + (b < a->MB ? bucket_elems(a, b) : 0);
    pb[b + 1] = pb[b] + (b < a->MB ? bucket_bytes(a, b) : 0);
  }
  for (uint32_t s = 0; s < a->S; ++s) {
    if (!need[s]) continue;
    uint64_t took = need[s];
    if (fail_b[s] != ~0u) {                  // bucket_vector.py:194-201
      took &= (uint64_t(1) << fail_b[s]) - 1;
      p.status[s] = GG_ENOMEM;
      p.ctl[s] = fail_b[s] | kCtlZero;       // keep buckets < b; zero the reserved range
      p.any_fail = p.any_ctl = true;
    }
    if (!took) continue;
    p.flags[s] |= took;
    const uint32_t k = (uint32_t)__builtin_popcountll(took), lo = (uint32_t)__builtin_ctzll(took);
    p.alloc_calls += k;
    if ((took >> lo) == (k == 64 ? ~0ull : (1ull << k) - 1)) {     // classes lo .. lo + k - 1
      p.cap[s] += pe[lo + k] - pe[lo];
      p.live += pb[lo + k] - pb[lo];
    } else {
      for (uint64_t m = took; m; m &= m - 1) {
        const uint32_t b = (uint32_t)__builtin_ctzll(m);
        p.cap[s] += pe[b + 1] - pe[b];
        p.live += pb[b + 1] - pb[b];
      }
    }
    if (a->dirty[s])
      for (uint64_t m = took; m; m &= m - 1) { p.zero_pairs.push_back(s); p.zero_pairs.push_back((uint32_t)__builtin_ctzll(m)); }
  }
}

// class bases travel to the device when a new class region was reserved
int push_cbase(gg_array *a, cudaStream_t st) {
  int arc = a->slab.finalize_access();          // chunks mapped by this operation
  if (arc) return arc;
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
// Work spaces from 32 MiB use the U the sweeps measured best per walk
// (tools/sweep.py, tools/ab_unroll.sh, tools/rwb_probe.py, B200: copies into
// the slabs U = 8 -- 32 KiB tiles; flatten and in-place r/w U = 4, 6.92 vs
// 6.88 TB/s for r/w since the planned walks run 3 CTAs per SM); below, U = 2 so small rounds
// still spread over every SM.  gg_set_tuning / GG_U_SMALL / GG_U_MID override.
uint32_t walk_unroll(const gg_array *a, uint64_t total, int w, uint32_t reps = 1) {
  if (g_tune.unroll > 0) return (uint32_t)g_tune.unroll;
  static const uint32_t u_small = [] { const char *e = getenv("GG_U_SMALL"); return e ? (uint32_t)atoi(e) : 2u; }();
  static const uint32_t u_mid = [] { const char *e = getenv("GG_U_MID"); return e ? (uint32_t)atoi(e) : 0u; }();
  const uint64_t bytes = total * a->esz;
  uint32_t u;
  if (bytes < (uint64_t(32) << 20)) u = u_small;
  else if (bytes < (uint64_t(256) << 20) && u_mid) u = u_mid;
  // in-place passes fused in registers (reps > 1) are ALU-heavy: more vectors in flight
  else u = (w == W_FLATTEN || (w == W_RW && reps <= 1)) ? 4u : 8u;   // tools/ab_unroll.sh, tools/sweep.py
  // many short LFVectors: a tile no longer than the average LFVector's work,
  // so tiles stay inside one LFVector (the vector path) instead of stepping
  // through several pieces one after another (S = 16384 x 2048 int32: 292 ->
  // 80 us per walk, tools/bigS_probe.py)
  const uint64_t per = total / (a->S ? a->S : 1), unit = 256ull * (16u / a->esz);
  while (u > 1 && (uint64_t)u * unit > per) u >>= 1;
  return u;
}

template <int ESZ, int W, typename T, bool P, int U>
cudaError_t walk_u(const gg_array *a, const Tables &t, const char *src, char *dst, uint64_t total,
                   T add, uint32_t reps, Fuse fz, cudaStream_t st) {
  const uint32_t tile = (uint32_t)U * kThreads * (16 / ESZ);
  const uint64_t grid = (total - fz.g0 + tile - 1) / tile + ((P && fz.size_next) ? 1 : 0);
  // Residency: the large-tile copies into the slabs (planned insert /
  // duplicate, U = 8) stream best at 3 CTAs of 256 threads per SM -- 4 are
  // ~1% slower, 2 far slower (tools/reset_probe.py with GG_WALK_SMEM /
  // GG_WALK_CARVEOUT).  Enforced with 16 KiB of dynamic shared memory under a
  // 25% shared-memory carveout (57 KiB per SM fit 3 such CTAs, not 4), so it
  // does not hinge on the kernel's register count.  The U = 4 flatten too;
  // the U = 4 in-place r/w is best uncapped.  GG_WALK_SMEM / GG_WALK_CARVEOUT
  // override both (tuning sweeps).
  static const int env_smem = [] { const char *e = getenv("GG_WALK_SMEM"); return e ? atoi(e) : -1; }();
  static const int env_carve = [] { const char *e = getenv("GG_WALK_CARVEOUT"); return e ? atoi(e) : -1; }();
  int smem = -1, carve = -1;
  if (U == 8 && P) { smem = 16 * 1024; carve = 25; }
  if (U == 4 && W == W_FLATTEN) { smem = 12 * 1024; carve = 25; }   // flatten: 3 per SM too (+0.6%)
  if (env_smem >= 0 && (U == 8 || U == 4)) smem = env_smem;
  if (env_carve >= 0 && (U == 8 || U == 4)) carve = env_carve;
  if (smem > 0 || carve >= 0) {
    // function attributes live in each device's context: once per kernel
    // instantiation and device (a->dev < 64)
    static std::atomic<uint64_t> attr_set{0};
    const uint64_t bit = uint64_t(1) << (a->dev & 63);
    if (!(attr_set.load(std::memory_order_acquire) & bit)) {
      if (smem > 48 * 1024)
        cudaFuncSetAttribute(k_walk<ESZ, W, T, U, kDefLS, P>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
      if (carve >= 0)
        cudaFuncSetAttribute(k_walk<ESZ, W, T, U, kDefLS, P>, cudaFuncAttributePreferredSharedMemoryCarveout, carve);
      attr_set.fetch_or(bit, std::memory_order_acq_rel);
    }
  }
  return launch_k(k_walk<ESZ, W, T, U, kDefLS, P>, (unsigned)grid, kThreads, smem > 0 ? (size_t)smem : 0, st, t,
                  src, dst, total, add, reps, tile, fz);
}

// the shard-grid walk (k_walk_shard) for a non-uniform directory: planned
// appends, flatten and in-place r/w over whole shards, buckets of >= 16 B,
// enough work per shard for full tiles
bool shard_grid_ok(const gg_array *a, int w, bool planned, const Fuse &fz, uint64_t total) {
  static const bool on = [] { const char *e = getenv("GG_SHARD_GRID"); return !e || e[0] != '0'; }();
  return on && fz.maxlen && !fz.ulen && fz.g0 == 0 && !fz.size_next && a->S <= 65535 &&
         ((uint64_t)a->fb * a->esz) >= 16 && total / a->S >= 2048 && (w == W_FLATTEN || w == W_RW || planned);
}

// longest shard of a directory dir[S+1]
uint64_t dir_maxlen(const uint64_t *dir, uint32_t S) {
  uint64_t m = 0;
  for (uint32_t s = 0; s < S; ++s) m = std::max<uint64_t>(m, dir[s + 1] - dir[s]);
  return m;
}

template <int ESZ, int W, typename T, int U>
int walk_shard(const gg_array *a, const Tables &t, const char *src, char *dst, T add, uint32_t reps,
               uint64_t maxlen, cudaStream_t st) {
  constexpr uint64_t TL = (uint64_t)U * 256 * (16 / ESZ);
  const dim3 grid((unsigned)((maxlen + 16 + TL - 1) / TL), a->S);
  cudaError_t e;
  if constexpr (W == W_DUP) e = launch_k(k_walk_shard_dup<ESZ, W, T, U>, grid, kThreads, 0, st, t, src, dst, add, reps);
  else e = launch_k(k_walk_shard<ESZ, W, T, U>, grid, kThreads, 0, st, t, src, dst, add, reps);
  if (e != cudaSuccess) return fail(GG_ECUDA, std::string("walk launch: ") + cudaGetErrorString(e));
  return GG_OK;
}

template <int ESZ, int W, typename T, bool P = false>
int walk(const gg_array *a, const Tables &t, const char *src, char *dst, uint64_t total, T add,
         uint32_t reps, Fuse fz, cudaStream_t st) {
  if (total == 0) return GG_OK;
  if (shard_grid_ok(a, W, P, fz, total)) {
    // copies into the slabs move 32 KiB tiles, flatten / r/w 16 KiB (tools/sweep.py's split)
    static const int u_sg = [] { const char *e = getenv("GG_SG_U"); return e ? atoi(e) : 0; }();
    if constexpr (W == W_INSERT || W == W_DUP) {
      if (u_sg == 4) return walk_shard<ESZ, W, T, 4>(a, t, src, dst, add, reps, fz.maxlen, st);
      return walk_shard<ESZ, W, T, 8>(a, t, src, dst, add, reps, fz.maxlen, st);
    } else {
      if (u_sg == 8) return walk_shard<ESZ, W, T, 8>(a, t, src, dst, add, reps, fz.maxlen, st);
      return walk_shard<ESZ, W, T, 4>(a, t, src, dst, add, reps, fz.maxlen, st);
    }
  }
  cudaError_t e;
  switch (walk_unroll(a, total, W, reps)) {
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

// every shard's committed length when they are all equal (and nonzero), else
// 0: a uniform directory lets the walks find shards by division
uint64_t uniform_len(const gg_array *a) {
  const uint64_t c = a->prefix[1] - a->prefix[0];
  for (uint32_t s = 1; s < a->S; ++s)
    if (a->prefix[s + 1] - a->prefix[s] != c) return 0;
  return c;
}

template <int W>
int launch_walk(gg_array *a, const Tables &t, const char *src, char *dst, uint64_t total,
                cudaStream_t st) {
  Fuse fz{0, 0};
  if (W == W_FLATTEN) {
    fz.ulen = uniform_len(a);
    if (!fz.ulen) fz.maxlen = dir_maxlen(a->prefix.data(), a->S);
  }
  return walk_copy<W, false>(a, t, src, dst, total, fz, st);
}

bool g_defer = true;            // defer + fuse planned metadata (GG_DEFER=0 disables)

uint32_t meta_threads(const gg_array *a) { return std::min<uint32_t>(1024, (a->S + 31) / 32 * 32); }

bool g_fuse = true;             // metadata CTA inside the planned walk (GG_FUSE_META=0 disables)

// launch a deferred metadata pass, if any: on the calling stream `st`
// (already ordered after the stream the pass was deferred on, order_stream),
// or on the stream of its walk for calls without a stream
int flush_meta(gg_array *a, cudaStream_t st = nullptr, bool on_st = false) {
  if (!a->pend) return GG_OK;
  a->pend = false;
  Tables t = tables_for_launch(a, false);
  CUDA_TRY(launch_k(k_planned_meta, 1, meta_threads(a), 0, on_st ? st : a->pend_st, t, a->pend_fz));
  return GG_OK;
}

// launch a deferred uniform grow, if any (same stream rule)
int flush_grow(gg_array *a, cudaStream_t st = nullptr, bool on_st = false) {
  if (!a->pend_grow) return GG_OK;
  const uint32_t k = a->pend_grow;
  a->pend_grow = 0;
  Tables t = tables_for_launch(a, true);
  CUDA_TRY(launch_k(k_grow, (a->S + 255) / 256, 256, 0, on_st ? st : a->pend_grow_st, t, k));
  return GG_OK;
}

int resolve_lanes(gg_array *a);

int flush_pending(gg_array *a, cudaStream_t st = nullptr, bool on_st = false) {
  int rc = resolve_lanes(a);
  if (rc) return rc;
  rc = flush_meta(a, st, on_st);
  return rc ? rc : flush_grow(a, st, on_st);
}

void flip_buffers(gg_array *a) {
  a->cur ^= 1;
  a->t.size = a->sz_buf[a->cur];
  a->t.prefix = a->pf_buf[a->cur];
}

bool capturing_now(gg_array *a, cudaStream_t st) {
  cudaStreamCaptureStatus cap = cudaStreamCaptureStatusNone;
  return a->up.capturing ||
         (cudaStreamIsCapturing(st, &cap) == cudaSuccess && cap != cudaStreamCaptureStatusNone);
}

// Stream order between calls on one handle (stream-ordered semantics across
// streams): a call on stream st after a call on another stream makes st wait
// for that stream's work so far (one event).  Deferred passes are then
// launched on st.  Under stream capture the caller orders its streams (an
// event recorded outside a capture cannot be waited on inside it).
int order_stream(gg_array *a, cudaStream_t st) {
  if (capturing_now(a, st)) { a->captured = true; return GG_OK; }
  if (a->have_last && a->last_st != st) {
    if (!a->ord_ev) CUDA_TRY(cudaEventCreateWithFlags(&a->ord_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(a->ord_ev, a->last_st));
    CUDA_TRY(cudaStreamWaitEvent(st, a->ord_ev, 0));
  }
  a->last_st = st;
  a->have_last = true;
  return GG_OK;
}

// An array that adopted a cached slab (slab_adopt) starts with every chunk
// of the destroyed array mapped.  Once its first allocating operation has
// taken the chunks it needs (live > 0), the adopted chunks still without a
// live bucket are doomed down to 2x the needed bytes -- unmapped
// asynchronously behind an event, or taken back in place for free if a later
// operation needs them before the reap -- so the adopted cache never leaves
// the array above the footprint bound (the paper's <= 2x).
int settle_adopted(gg_array *a, cudaStream_t st) {
  if (!a->slab.adopt_guard || !a->live || capturing_now(a, st)) return GG_OK;
  a->slab.adopt_guard = false;
  uint64_t need = 0;
  for (uint32_t s = 0; s < a->S; ++s) need += a->size[s];
  const uint64_t keep = 2 * need * a->esz;
  if (a->slab.cached && a->slab.mapped - a->slab.doomed_bytes > keep) return a->slab.doom_to(keep, st);
  return GG_OK;
}

// entry of a device-touching call on stream st: order, then launch whatever
// was deferred (on st)
int enter(gg_array *a, cudaStream_t st) {
  int rc = order_stream(a, st);
  if (!rc) rc = settle_adopted(a, st);
  return rc ? rc : flush_pending(a, st, true);
}

// mutating calls are refused while a device view is out: a user kernel may
// be appending through it, and the host mirrors the planner reads are stale
// until gg_device_view_sync
int check_no_view(const gg_array *a) {
  return a->view_out ? fail(GG_EVALUE, "a device view is outstanding (call gg_device_view_sync first)") : GG_OK;
}

// wait for the work queued on this handle so far: an event behind its last
// call's stream (every earlier stream is ordered before it); a device
// synchronize for handles that were captured into graphs
int wait_last(gg_array *a) {
  if (a->captured || !a->have_last) { CUDA_TRY(cudaDeviceSynchronize()); return GG_OK; }
  if (!a->ord_ev) CUDA_TRY(cudaEventCreateWithFlags(&a->ord_ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(a->ord_ev, a->last_st));
  CUDA_TRY(cudaEventSynchronize(a->ord_ev));
  return GG_OK;
}

// the metadata pass may ride inside the planned walk (and take a deferred
// grow with it): eager issue, or capture through GrowableArray.capture
bool fuse_ok(gg_array *a, cudaStream_t st) {
  // the metadata CTA has the walk's 256 threads: beyond 4096 shards its loop
  // would outlast small copies -- take the separate 1024-thread kernel there
  return g_fuse && a->S <= 4096 && (!capturing_now(a, st) || a->defer_in_capture);
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
               uint64_t total, cudaStream_t st, uint32_t flags, bool *committed,
               const uint64_t *h_offsets = nullptr, uint64_t csr_ulen = 0, uint64_t csr_ustart = 0) {
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
    // a non-uniform directory with whole tiles per shard takes the shard-grid
    // walk (its metadata pass is deferred, like the unfused planned walk)
    Fuse gz{reserve_mode, commit ? 1 : 0};
    if (!csr_ulen && total) {
      if (wk == W_INSERT && h_offsets) gz.maxlen = dir_maxlen(h_offsets, a->S);
      else if (wk == W_DUP && !uniform_len(a)) gz.maxlen = dir_maxlen(a->prefix.data(), a->S);
    }
    const bool grid2d = shard_grid_ok(a, wk, true, gz, total);
    if (total && fuse_ok(a, st) && !grid2d) {
      // ONE launch: copy CTAs + a metadata CTA writing the next size/prefix
      // pair (and publishing a deferred grow)
      Fuse fz{reserve_mode, commit ? 1 : 0};
      fz.size_next = a->sz_buf[a->cur ^ 1];
      fz.prefix_next = a->pf_buf[a->cur ^ 1];
      fz.grow_k = a->pend_grow;
      fz.ulen = csr_ulen;                    // uniform CSR: no offsets on the device needed
      fz.ustart = csr_ustart;
      a->pend_grow = 0;
      rc = wk == W_INSERT ? walk_copy<W_INSERT, true>(a, t, src, nullptr, total, fz, st)
                          : walk_copy<W_DUP, true>(a, t, nullptr, nullptr, total, fz, st);
      if (rc) return rc;
      flip_buffers(a);
      if (commit) { host_commit(a); *committed = true; }
      return GG_OK;
    }
    if ((rc = flush_grow(a, st, true))) return rc;
    if (csr_ulen) {                          // the other paths read the offsets on the device
      void *dst[1] = {a->t.offsets};
      const void *srcs[1] = {h_offsets};
      size_t bytes[1] = {(a->S + 1) * 8};
      if ((rc = a->up.upload(st, 1, dst, srcs, bytes))) return rc;
    }
    if (total) {
      Fuse fz = gz;
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
  if ((rc = flush_grow(a, st, true))) return rc;
  if (csr_ulen) {
    void *dst[1] = {a->t.offsets};
    const void *srcs[1] = {h_offsets};
    size_t bytes[1] = {(a->S + 1) * 8};
    if ((rc = a->up.upload(st, 1, dst, srcs, bytes))) return rc;
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

// Apply a tiled lanes insert to the host mirrors once its sizes are back
// (the pinned copy behind lanes_ev): sizes, ops, the published buckets of
// every reserved range (a deterministic function of the old and new sizes),
// capacity and live bytes; the upper-bound headroom no bucket took is
// unbacked, and chunks the backing newly mapped beyond max(2 x needed, the
// mapped bytes before it) are released asynchronously (doomed behind an
// event, taken back in place if an operation needs them first).
// issue the readback: one packing kernel (which also clears the status
// words) + ONE copy into the pinned staging
int view_finish_issue(gg_array *a, cudaStream_t st) {
  const size_t S = a->S;
  const size_t nb = view_pack_bytes(S);
  if (!a->h_view || a->h_view_cap < nb) {
    if (a->h_view) CUDA_TRY(cudaFreeHost(a->h_view));
    a->h_view = nullptr;
    CUDA_TRY(cudaMallocHost(&a->h_view, nb));
    a->h_view_cap = nb;
  }
  { k_view_pack<<<(unsigned)((S + 255) / 256), 256, 0, st>>>(a->t, a->d_vpack); g_launches.fetch_add(1, std::memory_order_relaxed); }
  CUDA_TRY(cudaGetLastError());
  CUDA_TRY(cudaMemcpyAsync(a->h_view, a->d_vpack, nb, cudaMemcpyDeviceToHost, st));
  return GG_OK;
}

// the host half, once the copy landed: mirrors from the device tables,
// headroom the kernel took becomes live, the rest is unbacked
int view_finish_host(gg_array *a, int32_t *h_status, cudaStream_t st) {
  const size_t S = a->S;
  char *hb = a->h_view;
  uint64_t *hs = (uint64_t *)hb, *hc = hs + S, *ho = hc + S, *hp = ho + S;
  uint32_t *hst = (uint32_t *)(hp + S);
  unsigned long long *hm = (unsigned long long *)(hb + S * 32 + ((S * 4 + 7) & ~size_t(7)));
  bool any = false;
  for (size_t s = 0; s < S; ++s) {
    a->size[s] = hs[s];
    a->cap[s] = hc[s];
    a->ops[s] = ho[s];
    // pmask bits are set after the once-flag is published (and never for a
    // rolled-back allocation): at kernel completion they are the published set
    a->flags[s] = hp[s];
    if (h_status) h_status[s] = (int32_t)hst[s];
    if (hst[s]) { any = true; a->dirty[s] = 1; }
  }
  a->alloc_calls = hm[MISC_ALLOCS];
  for (size_t i = 0; i < a->headroom.size(); i += 3) {
    const uint32_t b = a->headroom[i];
    for (uint32_t s = a->headroom[i + 1]; s < a->headroom[i + 2]; ++s) {
      if (a->flags[s] >> b & 1) a->live += bucket_bytes(a, b);
      else a->slab.unback(s, b);
    }
  }
  a->headroom.clear();
  // headroom chunks no bucket took: released asynchronously down to
  // max(2 x needed, the mapped bytes before the view), unless the array
  // keeps its cache (release=False)
  uint64_t need = 0;
  for (size_t s = 0; s < S; ++s) need += a->size[s];
  const uint64_t keep = std::max<uint64_t>(2 * need * a->esz, a->view_keep);
  if (!a->keep_cached && a->slab.cached && a->slab.mapped - a->slab.doomed_bytes > keep) {
    int drc = a->slab.doom_to(keep, st);
    if (drc) return drc;
  }
  return any ? fail(GG_EPARTIAL, "device-side appends failed on some shards") : GG_OK;
}

int resolve_lanes(gg_array *a) {
  if (a->view_pend) {                 // a push_if whose appends could not fail (see gg_push_if)
    CUDA_TRY(cudaEventSynchronize(a->lanes_ev));
    a->view_pend = false;
    a->view_n = 0;
    std::fill(a->view_hb.begin(), a->view_hb.end(), 0);
    const int rc = view_finish_host(a, nullptr, a->have_last ? a->last_st : nullptr);
    if (rc && rc != GG_EPARTIAL) return rc;
  }
  if (!a->lanes_pend) return GG_OK;
  CUDA_TRY(cudaEventSynchronize(a->lanes_ev));
  a->lanes_pend = false;
  const uint32_t n = a->lanes_n;
  a->lanes_n = 0;
  std::fill(a->lanes_hb.begin(), a->lanes_hb.end(), 0);
  uint64_t need = 0;
  for (uint32_t s = 0; s < a->S; ++s) {
    const uint64_t os = a->size[s];
    uint64_t ns = os;
    for (uint32_t k = 0; k < n; ++k)            // the pending calls in order: one op each that appended
      if (a->h_lanes[(size_t)k * a->S + s] > ns) {
        ns = a->h_lanes[(size_t)k * a->S + s];
        a->ops[s] += 1;
      }
    if (ns > os) {
      uint32_t b0, b1; uint64_t o;
      host_locate(a, os, b0, o);
      host_locate(a, ns - 1, b1, o);
      for (uint32_t b = b0; b <= b1 && b < a->MB; ++b) {
        if (a->flags[s] >> b & 1) continue;
        a->flags[s] |= uint64_t(1) << b;
        a->cap[s] += bucket_elems(a, b);
        a->live += bucket_bytes(a, b);
        a->alloc_calls += 1;
      }
      a->size[s] = ns;
    }
    need += a->size[s];
  }
  for (size_t i = 0; i < a->lanes_head.size(); i += 3) {
    const uint32_t b = a->lanes_head[i];
    for (uint32_t s = a->lanes_head[i + 1]; s < a->lanes_head[i + 2]; ++s)
      if (!(a->flags[s] >> b & 1)) a->slab.unback(s, b);
  }
  a->lanes_head.clear();
  const uint64_t keep = std::max<uint64_t>(2 * need * a->esz, a->lanes_keep);
  if (!a->keep_cached && a->slab.cached && a->slab.mapped - a->slab.doomed_bytes > keep && a->have_last)
    return a->slab.doom_to(keep, a->last_st);
  return GG_OK;
}

template <typename T>
int launch_rw(gg_array *a, const Tables &t, T addend, uint32_t passes, int mode, uint64_t total,
              cudaStream_t st) {
  if (mode == GG_RW_GLOBAL) {
    const uint64_t nvec = (total * sizeof(T) + 15) / 16;
    // sweep (tools/sweep.py): rw_g peaks at U = 4 (U = 8 spills the per-vector
    // pointers / masks into a lower occupancy)
    static const uint32_t ucap = [] { const char *e = getenv("GG_RWG_U"); return e ? (uint32_t)atoi(e) : 4u; }();
    const uint32_t U = std::min<uint32_t>(walk_unroll(a, total, W_RW), ucap);
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
  Fuse none{0, 0};
  none.ulen = uniform_len(a);
  if (!none.ulen) none.maxlen = dir_maxlen(a->prefix.data(), a->S);
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
// candidates i of its slices with pred[i] != 0 to shard b % S, warp- or
// block-aggregated.  Slice = kPushSlice consecutive candidates: block b
// takes slice b of every round of grid x kPushSlice candidates.  Each thread
// loads G consecutive candidates at a time -- one 16 B vector of values
// (32 B for 8 B elements) and G predicate bytes (a 4 / 8 / 16 B vector) --
// K per append call, into registers with a K-bit keep mask, and appends them
// with ONE warp- or block-aggregated reservation per call (block mode: the
// run is staged in shared memory and leaves as 16 B vector stores); all
// indexing static (no local memory).  For 1 / 2 B elements G = 16 / 8, so a
// slice is covered by 64 / 128 threads and one load sweep of the block
// covers 4 / 2 rounds (the same 8 rounds per call as 4 B elements).
constexpr uint32_t kPushSlice = 1024;

template <int ESZ, int BLOCK>
struct PushShape {
  static constexpr uint32_t G = ESZ >= 4 ? 4 : 16 / ESZ;   // candidates per load
  static constexpr uint32_t K = ESZ == 8 ? 16 : 32;         // candidates per thread per append call
  static constexpr uint32_t J = K / G;                      // loads per thread per call
  static constexpr uint32_t TPS = kPushSlice / G;           // threads per slice
  static constexpr uint32_t RPL = BLOCK / TPS;              // rounds per load sweep
  static constexpr uint32_t RPC = J * RPL;                  // rounds per call
  static_assert(BLOCK % TPS == 0, "a block covers whole slices");
};

template <int ESZ, int BLOCK, bool BLOCK_MODE>
__global__ void __launch_bounds__(BLOCK, ESZ >= 4 ? 4 : 6) k_push_if(gg_device_view t, const char *vals,
                                                   const uint8_t *pred, uint64_t n, int aligned, uint32_t pf) {
  typedef typename ElemT<ESZ>::T E;
  typedef PushShape<ESZ, BLOCK> P;
  constexpr uint32_t G = P::G, J = P::J, RPL = P::RPL;
  constexpr int K = (int)P::K;
  __shared__ unsigned long long scratch[34];
  // block mode: one run of up to BLOCK*K staged; warp mode: a private slice
  // of 32*K + 32/ESZ elements per warp (16 B multiples)
  __shared__ __align__(16) E stage[BLOCK * K + (BLOCK_MODE ? 1 : BLOCK / 32) * (32 / ESZ)];
  const uint32_t s = blockIdx.x % t.S;
  const uint64_t round = (uint64_t)gridDim.x * kPushSlice;
  // this thread's candidates: load j of a call starting at round r0 covers
  // round r0 + j * RPL + sub, positions [pos, pos + G) of the block's slice
  const uint64_t sub = threadIdx.x / P::TPS, pos = (threadIdx.x % P::TPS) * G;
  // the next call's slices (values and predicates of RPC rounds) are
  // prefetched into L2 by TMA while this call loads and appends (pf = 1)
  auto pf_call = [&](uint64_t rc) {
    const uint32_t j = threadIdx.x >> 1;
    if (j < P::RPC) {
      const uint64_t i = (uint64_t)blockIdx.x * kPushSlice + (rc + j) * round;
      if (i + kPushSlice <= n) {
        if (threadIdx.x & 1) prefetch_l2(pred + i, kPushSlice);
        else prefetch_l2(vals + i * ESZ, kPushSlice * ESZ);
      }
    }
  };
  if (pf && aligned) pf_call(0);
  for (uint64_t r0 = 0; (uint64_t)blockIdx.x * kPushSlice + r0 * round < n; r0 += P::RPC) {
    if (pf && aligned) pf_call(r0 + P::RPC);
    E v[K];
    uint32_t mask = 0;
    const uint64_t i0 = (uint64_t)blockIdx.x * kPushSlice + (r0 + sub) * round + pos;
    if (aligned && i0 + (uint64_t)(J - 1) * RPL * round + G <= n) {
      // interior: every load in bounds -- all J loads are issued before any
      // is consumed (a per-load bounds branch around load + use would
      // serialise them: one load in flight per thread)
      uint32_t pw[J][G / 4];
#pragma unroll
      for (int j = 0; j < (int)J; ++j) {
        const uint64_t i = i0 + (uint64_t)j * RPL * round;
        if constexpr (G == 16) {
          const uint4 q = __ldcs(reinterpret_cast<const uint4 *>(pred + i));
          pw[j][0] = q.x; pw[j][1] = q.y; pw[j][2] = q.z; pw[j][3] = q.w;
        } else if constexpr (G == 8) {
          const uint2 q = __ldcs(reinterpret_cast<const uint2 *>(pred + i));
          pw[j][0] = q.x; pw[j][1] = q.y;
        } else {
          pw[j][0] = __ldcs(reinterpret_cast<const uint32_t *>(pred + i));
        }
        if constexpr (ESZ * G == 16) {
          const uint4 q = __ldcs(reinterpret_cast<const uint4 *>(vals + i * ESZ));
          memcpy(&v[j * G], &q, 16);
        } else {
          const uint4 q0 = __ldcs(reinterpret_cast<const uint4 *>(vals + i * ESZ));
          const uint4 q1 = __ldcs(reinterpret_cast<const uint4 *>(vals + i * ESZ) + 1);
          memcpy(&v[j * G], &q0, 16);
          memcpy(&v[j * G + 2], &q1, 16);
        }
      }
#pragma unroll
      for (int j = 0; j < (int)J; ++j)
#pragma unroll
        for (int g = 0; g < (int)G; ++g)
          mask |= ((pw[j][g >> 2] >> (8 * (g & 3))) & 0xffu ? 1u : 0u) << (j * G + g);
    } else {
      // the last rounds of the input (or an unaligned input): element loads
#pragma unroll
      for (int j = 0; j < (int)J; ++j) {
        const uint64_t i = i0 + (uint64_t)j * RPL * round;
#pragma unroll
        for (int g = 0; g < (int)G; ++g) {
          v[j * G + g] = E(0);
          if (i + g < n) {
            v[j * G + g] = __ldcs(reinterpret_cast<const E *>(vals) + i + g);
            mask |= (__ldcs(pred + i + g) ? 1u : 0u) << (j * G + g);
          }
        }
      }
    }
    if constexpr (BLOCK_MODE) block_push_back_staged<BLOCK, E, K>(t, s, mask, v, scratch, stage);
    else warp_push_back_staged<E, K>(t, s, mask, v, stage + (threadIdx.x >> 5) * (32 * K + 32 / ESZ));
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

// Per-device library initialisation, once per process: the CUDA context and
// the library's kernel image (lazy module loading would otherwise load it
// at the first launch, ~30 ms inside the first operation).  Called by
// gg_create; callable up front.
int gg_init(int device) {
  static std::mutex mu;
  static uint64_t done = 0;
  if (device < 0 || device >= 64) return fail(GG_EVALUE, "device out of range");
  std::lock_guard<std::mutex> g(mu);
  if (done >> device & 1) return GG_OK;
  CUDA_TRY(cudaSetDevice(device));
  CUDA_TRY(cudaFree(0));
  cudaFuncAttributes fa;
  CUDA_TRY(cudaFuncGetAttributes(&fa, k_shrink_uniform));
  done |= 1ull << device;
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
  { int rc = gg_init(device); if (rc) return rc; }
  CUDA_TRY(cudaSetDevice(device));
  reclaim(false);                          // chunks of arrays destroyed earlier -> the pool
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
  const bool adopted = slab_adopt(a->slab);   // a same-shape slab left by a destroyed array
  // metadata block
  const size_t S = shards, T = S * max_buckets;
  size_t bytes = 0;
  auto take = [&](size_t n) { size_t o = bytes; bytes += (n + 255) & ~size_t(255); return o; };
  size_t o_size = take(S * 8), o_cap = take(S * 8), o_ops = take(S * 8), o_start = take(S * 8),
         o_count = take(S * 8), o_prefix = take((S + 1) * 8), o_off = take((S + 1) * 8),
         o_ctl = take(S * 4), o_flag = take(T * 4), o_status = take(S * 4), o_ptr = take(T * 8),
         o_misc = take(MISC_N * 8), o_won = take(16), o_scr = take(64), o_am = take(S * 8),
         o_cb = take(max_buckets * 8), o_pm = take(S * 8), o_size2 = take(S * 8),
         o_prefix2 = take((S + 1) * 8), o_vpack = take(view_pack_bytes(S));
  cudaError_t e = cudaMallocAsync(&a->dmem, bytes, 0);   // driver mempool: no device-wide sync
  if (e != cudaSuccess) { a->slab.destroy(); delete a; return fail(GG_ECUDA, cudaGetErrorString(e)); }
  cudaMemsetAsync(a->dmem, 0, bytes, 0);
  char *base = (char *)a->dmem;
  Tables &t = a->t;
  t.size = (uint64_t *)(base + o_size); t.cap = (uint64_t *)(base + o_cap);
  t.ops = (uint64_t *)(base + o_ops); t.start = (uint64_t *)(base + o_start);
  t.count = (uint64_t *)(base + o_count); t.prefix = (uint64_t *)(base + o_prefix);
  t.offsets = (uint64_t *)(base + o_off); t.ctl = (uint32_t *)(base + o_ctl);
  t.flag = (uint32_t *)(base + o_flag); t.status = (uint32_t *)(base + o_status);
  t.ptr = (char **)(base + o_ptr); t.misc = (unsigned long long *)(base + o_misc);
  t.amask = (unsigned long long *)(base + o_am); t.cbase = (char **)(base + o_cb);
  a->sz_buf[0] = t.size; a->sz_buf[1] = (uint64_t *)(base + o_size2);
  a->pf_buf[0] = t.prefix; a->pf_buf[1] = (uint64_t *)(base + o_prefix2);
  t.pmask = (unsigned long long *)(base + o_pm);
  t.S = shards; t.log2fb = a->log2fb; t.MB = max_buckets; t.esz = esz;
  a->d_won = (int *)(base + o_won);
  a->d_vpack = base + o_vpack;
  a->d_scratch = base + o_scr;
  // creation work is queued on the legacy default stream (no device-wide
  // synchronize); the first call on another stream waits for it (order_stream)
  a->last_st = 0;
  a->have_last = true;
  if ((rc = a->up.init(device))) { gg_destroy(a); return rc; }
  if (a->slab.small.base || adopted) {  // the packed small-class region (and adopted regions) exist
    std::vector<uint64_t> cb(max_buckets);
    for (uint32_t b = 0; b < max_buckets; ++b) cb[b] = a->slab.class_base(b);
    void *dst[1] = {t.cbase};
    const void *src[1] = {cb.data()};
    size_t nb[1] = {max_buckets * sizeof(uint64_t)};
    if ((rc = a->up.upload(0, 1, dst, src, nb))) { gg_destroy(a); return rc; }
  }
  *out = a;
  return GG_OK;
}

// Stream-ordered teardown: the handle's memory (slab chunks, metadata, pinned
// buffers) is freed once an event recorded behind its last call's stream
// completes -- every earlier call's stream is ordered before that one
// (order_stream) -- so destroying an array never waits for the whole device
// and costs no driver call here; the chunks then go to the process pool.
// Arrays that were ever captured into a CUDA graph fall back to a device
// synchronize (a graph may still replay their kernels on any stream).
int gg_destroy(gg_array *a) {
  if (!a) return GG_OK;
  std::unique_lock<std::mutex> lk(a->mu);
  use_dev(a->dev);
  Grave *g = new Grave();
  g->dev = a->dev;
  if (a->captured || a->up.capturing) {
    cudaDeviceSynchronize();
  } else if (a->have_last) {
    if (cudaEventCreateWithFlags(&g->ev, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventRecord(g->ev, a->last_st) != cudaSuccess) {
      if (g->ev) cudaEventDestroy(g->ev);
      g->ev = nullptr;
      cudaDeviceSynchronize();            // the last stream is gone: wait for the device
    }
  }
  a->slab.pending.clear();                // (access of chunks never used needs no grant)
  a->slab.doomed.clear();
  a->slab.doomed_bytes = 0;
  g->slab = std::move(a->slab);
  g->up = std::move(a->up);
  g->dmem = a->dmem;
  g->h_scratch = a->h_scratch;
  g->h_lanes = a->h_lanes;
  g->h_view = a->h_view;
  g->lanes_dmem = a->lanes_dmem;
  g->lanes_ev = a->lanes_ev;
  g->ord_ev = a->ord_ev;
  lk.unlock();
  delete a;
  bury(g);
  reclaim(false);                         // frees this one at once if its work is done
  return GG_OK;
}

int gg_reclaim(int32_t wait) {
  reclaim(wait != 0);
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

// Uniform fast path shared by insert and duplicate: every shard appends the
// same count c at the same size with the same published buckets (no hook,
// cap, failed or dirty shard) -> plan shard 0 once, back each bucket class
// for all shards in one call, one fused walk.  *done = false (nothing
// changed) when the state is not uniform or backing ran out of memory: the
// caller takes the exact per-shard planner.
int uniform_append(gg_array *a, int wk, const char *src, uint64_t c, const uint64_t *h_offsets,
                   uint32_t flags, int32_t *h_status, cudaStream_t st, bool *done) {
  *done = false;
  if (a->hook || a->limit || (flags & GG_F_UNFUSED) || !c) return GG_OK;
  for (uint32_t s = 0; s < a->S; ++s)
    if (a->size[s] != a->size[0] || a->flags[s] != a->flags[0] || a->dirty[s]) return GG_OK;
  const uint64_t start = a->size[0];
  uint32_t b0, b1; uint64_t o;
  host_locate(a, start, b0, o);
  host_locate(a, start + c - 1, b1, o);
  if (b1 >= a->MB) return GG_OK;               // capacity error: the exact path reports it
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
  if (rc) {                                     // out of memory: undo, take the exact path
    for (uint32_t b = b0; b <= b1; ++b)
      if (got >> b & 1) a->slab.unback_range(b, 0, a->S);
    return GG_OK;
  }
  *done = true;
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
  const int rmode = wk == W_DUP ? 1 : 0;
  const uint64_t total = c * a->S;
  Tables t = tables_for_launch(a, false);
  if (fuse_ok(a, st)) {
    Fuse fz{rmode, commit ? 1 : 0};
    fz.ulen = c;                               // uniform directory / CSR and destination start
    fz.ustart = start;
    fz.size_next = a->sz_buf[a->cur ^ 1];
    fz.prefix_next = a->pf_buf[a->cur ^ 1];
    fz.grow_k = a->pend_grow;
    a->pend_grow = 0;
    rc = wk == W_DUP ? walk_copy<W_DUP, true>(a, t, nullptr, nullptr, total, fz, st)
                     : walk_copy<W_INSERT, true>(a, t, src, nullptr, total, fz, st);
    if (rc) return rc;
    flip_buffers(a);
  } else {
    if ((rc = flush_grow(a, st, true))) return rc;
    if (wk == W_INSERT) {                      // the unfused walk reads the offsets on the device
      void *dst[1] = {a->t.offsets};
      const void *srcs[1] = {h_offsets};
      size_t nb[1] = {(a->S + 1) * 8};
      if ((rc = a->up.upload(st, 1, dst, srcs, nb))) return rc;
    }
    Fuse fu{rmode, commit ? 1 : 0};
    fu.ulen = c;                               // uniform: no directory loads in the walk
    fu.ustart = start;
    rc = wk == W_DUP ? walk_copy<W_DUP, true>(a, t, nullptr, nullptr, total, fu, st)
                     : walk_copy<W_INSERT, true>(a, t, src, nullptr, total, fu, st);
    if (rc) return rc;
    if (a->S > 4096) {
      // store-only multi-CTA metadata: every value is known on the host
      const uint64_t work = (uint64_t)a->S * (want ? (64 - __builtin_clzll(want)) - __builtin_ctzll(want) : 1);
      const uint32_t grid = (uint32_t)std::min<uint64_t>((work + 255) / 256, (uint64_t)sm_count(a->dev) * 4);
      CUDA_TRY(launch_k(k_meta_uniform, std::max<uint32_t>(grid, 1), 256, 0, st, t, start, c, commit ? 1 : 0,
                        (unsigned long long)want, (unsigned long long)a->flags[0], (uint64_t)a->cap[0]));
    } else if ((rc = finish_planned(a, Fuse{rmode, commit ? 1 : 0}, st))) {
      return rc;
    }
  }
  if (commit) host_commit(a);
  if (h_status) memset(h_status, 0, a->S * sizeof(int32_t));
  return GG_OK;
}

int gg_insert_ex2(gg_array *a, const void *d_values, const uint64_t *h_offsets,
                  const uint64_t *h_starts, uint32_t flags, int32_t *h_status, uint64_t *h_reserved,
                  void *stream);

int gg_insert_ex(gg_array *a, const void *d_values, const uint64_t *h_offsets,
                 const uint64_t *h_starts, uint32_t flags, int32_t *h_status, void *stream) {
  return gg_insert_ex2(a, d_values, h_offsets, h_starts, flags, h_status, nullptr, stream);
}

int gg_insert_ex2(gg_array *a, const void *d_values, const uint64_t *h_offsets,
                  const uint64_t *h_starts, uint32_t flags, int32_t *h_status, uint64_t *h_reserved,
                  void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  cudaStream_t st = S_(stream);
  {   // a deferred grow may ride on this walk
    int frc_ = check_no_view(a);
    if (!frc_) frc_ = order_stream(a, st);
    if (!frc_) frc_ = flush_meta(a, st, true);
    if (frc_) return frc_;
  }
  if (h_offsets[0] != 0) return fail(GG_EVALUE, "offsets[0] must be 0");
  if (h_reserved)       // each shard's reservation start, read under the handle's lock
    for (uint32_t s = 0; s < a->S; ++s) h_reserved[s] = h_starts ? h_starts[s] : a->size[s];
  std::vector<uint64_t> counts(a->S);
  for (uint32_t s = 0; s < a->S; ++s) {
    if (h_offsets[s + 1] < h_offsets[s]) return fail(GG_EVALUE, "offsets must be non-decreasing");
    counts[s] = h_offsets[s + 1] - h_offsets[s];
  }
  const uint64_t total = h_offsets[a->S];
  if (!h_starts && h_offsets[1] > 0) {        // uniform CSR over uniform shards
    bool u = true;
    for (uint32_t s = 0; s < a->S && u; ++s) u = counts[s] == h_offsets[1];
    if (u) {
      bool done = false;
      int rc = uniform_append(a, W_INSERT, (const char *)d_values, h_offsets[1], h_offsets, flags,
                              h_status, st, &done);
      if (rc || done) return rc;
    }
  }
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
  }
  // uniform CSR over uniform shards (every batch c elements, every shard the
  // same size): the fused walk derives the offsets and starts itself
  uint64_t ulen = 0, ustart = 0;
  if (!h_starts && h_offsets[1] > 0) {
    bool u = true;
    const uint64_t c = h_offsets[1];
    for (uint32_t s = 0; s < a->S && u; ++s)
      u = h_offsets[s + 1] - h_offsets[s] == c && a->size[s] == a->size[0];
    if (u) { ulen = c; ustart = a->size[0]; }
  }
  if (!h_starts && !ulen) {
    void *dst[1] = {a->t.offsets};
    const void *src[1] = {h_offsets};
    size_t bytes[1] = {(a->S + 1) * 8};
    if ((rc = a->up.upload(st, 1, dst, src, bytes))) return rc;
  }
  bool committed;
  if ((rc = run_append(a, p, h_starts ? 2 : 0, W_INSERT, (const char *)d_values, total, st, flags,
                       &committed, h_offsets, ulen, ustart)))
    return rc;
  if (!h_starts)
    for (uint32_t s = 0; s < a->S; ++s) if (counts[s]) a->ops[s] += 1;
  return finish_status(a, p, h_status);
}

int gg_insert_duplicate_ex(gg_array *a, uint32_t flags, int32_t *h_status, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  cudaStream_t st = S_(stream);
  {   // a deferred grow may ride on this walk
    int frc_ = check_no_view(a);
    if (!frc_) frc_ = order_stream(a, st);
    if (!frc_) frc_ = flush_meta(a, st, true);
    if (frc_) return frc_;
  }
  {
    // uniform fast path: every shard has the same committed length, size and
    // buckets, no hook / cap / failed shard -> plan shard 0 once
    const uint64_t c = a->prefix[1] - a->prefix[0];
    bool uni = c != 0;
    for (uint32_t s = 0; s < a->S && uni; ++s) uni = a->prefix[s + 1] - a->prefix[s] == c;
    if (uni) {
      const uint32_t kc = min_buckets_for(a, c);
      const uint64_t need = kc >= 64 ? ~uint64_t(0) : ((uint64_t(1) << kc) - 1);
      if ((a->flags[0] & need) != need)
        return fail(GG_EUNPUBLISHED, "bucket unpublished while walking shard 0");
      bool done = false;
      int rc = uniform_append(a, W_DUP, nullptr, c, nullptr, flags, h_status, st, &done);
      if (rc || done) return rc;
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
  { int frc_ = check_no_view(a); if (!frc_) frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
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
  {   // a deferred metadata pass / grow is fused below (on this, ordered, stream)
    int frc_ = check_no_view(a);
    if (!frc_) frc_ = order_stream(a, st);
    if (frc_) return frc_;
  }
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
        if (!a->pend && fuse_ok(a, st)) {     // published by the next planned walk's metadata CTA
          a->pend_grow = std::max(a->pend_grow, k);
          a->pend_grow_st = st;
          return GG_OK;
        }
        if ((rc = flush_grow(a, st, true))) return rc;
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
  { int frc_ = flush_pending(a, st, true); if (frc_) return frc_; }
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
  { int frc_ = check_no_view(a); if (!frc_) frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
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
  { int frc_ = check_no_view(a); if (!frc_) frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  if (s >= a->S) return fail(GG_EVALUE, "shard out of range");
  *h_prev = a->size[s];
  a->size[s] += c;
  a->ops[s] += 1;
  { k_fetch_add<<<1, 1, 0, S_(stream)>>>(a->t, s, c); g_launches.fetch_add(1, std::memory_order_relaxed); }
  CUDA_TRY(cudaGetLastError());
  if (c) {
    // indices reserved here may never be written (a reserver that fails
    // between reserve and write) and then read back after commit: they must
    // read 0 like the reference's np.zeros buckets, but slab memory is
    // recycled.  Zero the reserved range where its buckets already exist,
    // and mark the shard so buckets it allocates later are zeroed.
    a->dirty[s] = 1;
    const uint64_t lo = *h_prev, hi = lo + c;
    uint32_t b0, b1; uint64_t o;
    host_locate(a, lo, b0, o);
    host_locate(a, hi - 1, b1, o);
    for (uint32_t b = b0; b <= b1 && b < a->MB; ++b) {
      if (!(a->flags[s] >> b & 1)) continue;
      const uint64_t bs = ((uint64_t(1) << b) - 1) << a->log2fb, be = bs + bucket_elems(a, b);
      const uint64_t x0 = std::max(lo, bs), x1 = std::min(hi, be);
      char *p = (char *)a->slab.class_base(b) + (uint64_t)s * bucket_bytes(a, b) + (x0 - bs) * a->esz;
      CUDA_TRY(cudaMemsetAsync(p, 0, (x1 - x0) * a->esz, S_(stream)));
    }
  }
  return GG_OK;
}

int gg_shrink_ex(gg_array *a, const uint64_t *h_new_sizes, uint64_t keep_mapped_bytes,
                 void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = check_no_view(a); if (!frc_) frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  a->keep_cached = keep_mapped_bytes == ~uint64_t(0);
  cudaStream_t st = S_(stream);
  for (uint32_t s = 0; s < a->S; ++s)
    if (h_new_sizes[s] > a->size[s]) return fail(GG_EVALUE, "shrink cannot grow a shard");
  bool uni = true;                             // same size and buckets everywhere: class-batched
  for (uint32_t s = 0; s < a->S && uni; ++s)
    uni = h_new_sizes[s] == h_new_sizes[0] && a->flags[s] == a->flags[0];
  const uint64_t old_flags0 = a->flags[0];
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
  const uint64_t *d_sizes = nullptr;      // a uniform shrink passes its size as a scalar
  if (!uni) {
    void *dst[1] = {a->t.count};
    const void *src[1] = {h_new_sizes};
    size_t bytes[1] = {a->S * 8};
    int rc = a->up.upload(st, 1, dst, src, bytes);
    if (rc) return rc;
    d_sizes = a->t.count;
  }
  Tables t = tables_for_launch(a, false);
  if (uni) {
    const uint64_t keep_b = min_buckets_for(a, h_new_sizes[0]);
    const uint64_t drop = keep_b >= 64 ? 0 : (old_flags0 & ~((uint64_t(1) << keep_b) - 1));
    const uint64_t work = (uint64_t)a->S * (drop ? (64 - __builtin_clzll(drop)) - __builtin_ctzll(drop) : 1);
    const uint32_t grid = (uint32_t)std::min<uint64_t>((work + 255) / 256, (uint64_t)sm_count(a->dev) * 4);
    CUDA_TRY(launch_k(k_shrink_uniform, std::max<uint32_t>(grid, 1), 256, 0, st, t,
                      (uint64_t)h_new_sizes[0], (unsigned long long)drop,
                      (unsigned long long)a->flags[0], (uint64_t)a->cap[0]));
  } else {
    CUDA_TRY(launch_k(k_shrink, 1, std::min<uint32_t>(1024, (a->S + 31) / 32 * 32), 0, st, t, d_sizes,
                      (uint64_t)h_new_sizes[0]));
  }
  uint64_t acc = 0;
  for (uint32_t s = 0; s < a->S; ++s) { acc += a->size[s]; a->prefix[s + 1] = acc; }
  // unmap emptied chunks down to keep_mapped_bytes -- asynchronously: queued
  // work may still read the released buckets, so they are unmapped once an
  // event behind this shrink completed (Slab::doom_to / reap_doomed), not
  // after a device-wide synchronize.  Never under graph capture, where the
  // chunks stay cached until gg_trim.
  if (!capturing_now(a, st) && a->slab.cached && a->slab.mapped - a->slab.doomed_bytes > keep_mapped_bytes) {
    int rc = a->slab.doom_to(keep_mapped_bytes, st);
    if (rc) return rc;
  }
  a->slab.reap_doomed(false);               // earlier shrinks' chunks whose work is done
  return GG_OK;
}

int gg_shrink(gg_array *a, const uint64_t *h_new_sizes, void *stream) {
  return gg_shrink_ex(a, h_new_sizes, 0, stream);
}

int gg_trim(gg_array *a) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = check_no_view(a); if (!frc_) frc_ = flush_pending(a); if (frc_) return frc_; }
  a->keep_cached = false;
  if (!a->slab.cached) return GG_OK;
  int rc = wait_last(a);
  if (rc) return rc;
  a->slab.trim();
  return GG_OK;
}

// unmap what earlier shrinks released, waiting for the work queued before
// them (the footprint a caller reads next is then settled)
int gg_settle(gg_array *a) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int rc = resolve_lanes(a); if (rc) return rc; }
  { int rc = settle_adopted(a, a->have_last ? a->last_st : nullptr); if (rc) return rc; }
  a->slab.reap_doomed(true);
  return GG_OK;
}

namespace {
constexpr int GG_ENOTSUP = -1;      // internal: take the exact path

// The tiled lanes insert (paper Alg. 1 at throughput): the host backs every
// shard's slots for the upper bound lanes x values_per_lane (no device round
// trip), the device reserves (one atomicAdd per LFVector), publishes and
// scatters; the reached sizes come back asynchronously (resolve_lanes).
int lanes_tiled(gg_array *a, const void *d_values, const uint32_t *d_counts, const uint64_t *off,
                uint64_t K, cudaStream_t st) {
  static const bool on = [] { const char *e = getenv("GG_LANES_TILED"); return !e || e[0] != '0'; }();
  const uint64_t KB = K * a->esz;
  // register-resident lanes: KB a power of two in [4, 64], 16 B-aligned values
  if (!on || a->hook || a->limit || KB < 4 || KB > 64 || (KB & (KB - 1)) ||
      ((uintptr_t)d_values % 16) || capturing_now(a, st))
    return GG_ENOTSUP;
  const uint32_t S = a->S;
  for (uint32_t s = 0; s < S; ++s)
    if (off[s + 1] > off[s] && a->dirty[s]) return GG_ENOTSUP;
  // back the upper bound (all or nothing), class by class in runs of
  // consecutive shards that need the class (one batched refcount pass per
  // run instead of one slab call per bucket: uniform lanes are one run)
  const uint64_t mapped0 = a->slab.mapped;
  std::vector<uint32_t> head;               // (b, s0, s1) runs backed
  std::vector<uint32_t> nb0(S, 1), nb1(S, 0);
  uint32_t bmin = a->MB, bmax = 0;
  // the sizes this call starts from: exact, or the upper bounds of the
  // pending (chained) calls
  if (a->lanes_ub.size() != S) { a->lanes_ub.assign(S, 0); a->lanes_hb.assign(S, 0); }
  const uint64_t *base = a->lanes_pend ? a->lanes_ub.data() : a->size.data();
  const uint64_t *hb = a->lanes_hb.data();  // buckets the pending calls backed (zero when none)
  for (uint32_t s = 0; s < S; ++s) {
    const uint64_t U = (off[s + 1] - off[s]) * K;
    if (!U) continue;
    uint64_t o;
    host_locate(a, base[s], nb0[s], o);
    host_locate(a, base[s] + U - 1, nb1[s], o);
    if (nb1[s] >= a->MB) return GG_ENOTSUP;
    bmin = std::min(bmin, nb0[s]);
    bmax = std::max(bmax, nb1[s]);
  }
  bool ok = true;
  for (uint32_t b = bmin; b <= bmax && b < a->MB && ok; ++b) {
    bool have_region = false;
    for (uint32_t s = 0; s < S && ok;) {
      auto need = [&](uint32_t x) { return nb0[x] <= b && b <= nb1[x] && !((a->flags[x] | hb[x]) >> b & 1); };
      if (!need(s)) { ++s; continue; }
      uint32_t e = s + 1;
      while (e < S && need(e)) ++e;
      if (!have_region) {
        bool created = false;
        if (a->slab.ensure_region(b, &created) != GG_OK) { ok = false; break; }
        if (created) a->cbase_dirty = true;
        have_region = true;
      }
      if (g_batch_backing == 1 ? a->slab.back_range(b, s, e) != GG_OK : g_batch_backing == 2) { ok = false; break; }
      if (!g_batch_backing) {                    // one slab call per bucket (A/B)
        uint32_t x = s;
        for (; x < e && a->slab.back(x, b) == GG_OK; ++x) { head.push_back(b); head.push_back(x); head.push_back(x + 1); }
        if (x < e) { ok = false; break; }
        s = e;
        continue;
      }
      head.push_back(b); head.push_back(s); head.push_back(e);
      s = e;
    }
  }
  if (!ok) {
    for (size_t i = 0; i < head.size(); i += 3) a->slab.unback_range(head[i], head[i + 1], head[i + 2]);
    return GG_ENOTSUP;
  }
  int rc = push_cbase(a, st);
  if (rc) return rc;
  // tiles: 8 warps x (64 / KB) rows of 32 lanes (64 B of values per thread)
  // one pass (default): chunks of C lanes, a CTA each; 3-pass A/B
  // (GG_LANES_CHAIN=0): tiles of T lanes for k_lanes_sum / k_lanes_scatter
  static const bool chain = [] { const char *e = getenv("GG_LANES_CHAIN"); return !e || e[0] != '0'; }();
  const uint32_t T = (uint32_t)(256 * (64 / KB));
  // lanes per chunk (GG_LANES_C: A/B, a multiple of the tile)
  static const uint32_t chunk_lanes = [] {
    const char *e = getenv("GG_LANES_C");
    const long v = e ? atol(e) : 0;
    return v >= 4096 && v <= (1 << 20) && (v & (v - 1)) == 0 ? (uint32_t)v : kLanesChunk;
  }();
  const uint32_t C = std::max<uint32_t>(chunk_lanes, T);
  const uint32_t unit = chain ? C : T;
  std::vector<uint32_t> tpre(S + 1);
  uint64_t nt = 0;
  for (uint32_t s = 0; s < S; ++s) {
    tpre[s] = (uint32_t)nt;
    nt += (off[s + 1] - off[s] + unit - 1) / unit;
  }
  if (nt > 0x7fffffffu) return fail(GG_EVALUE, "too many lanes");
  tpre[S] = (uint32_t)nt;
  // scratch: tpre[S+1] | tiles[nt] (3-pass) or chain[nt] status words (one
  // pass) (grown on demand, stream ordered)
  const size_t o_tiles = ((size_t)(S + 1) * 4 + 31) & ~size_t(31);
  if (!a->lanes_dmem || a->lanes_tiles_cap < nt) {
    if (a->lanes_dmem) CUDA_TRY(cudaFreeAsync(a->lanes_dmem, st));
    const size_t cap = std::max<uint64_t>(nt, 1024);
    CUDA_TRY(cudaMallocAsync(&a->lanes_dmem, o_tiles + cap * sizeof(LaneTile), st));
    a->lanes_tiles_cap = cap;
  }
  char *dm = (char *)a->lanes_dmem;
  uint32_t *d_tpre = (uint32_t *)dm;
  LaneTile *d_tiles = (LaneTile *)(dm + o_tiles);
  void *dst[2] = {a->t.offsets, d_tpre};
  const void *src[2] = {off, tpre.data()};
  size_t bytes[2] = {(size_t)(S + 1) * 8, (size_t)(S + 1) * 4};
  if ((rc = a->up.upload(st, 2, dst, src, bytes))) return rc;
  if (!a->h_lanes) CUDA_TRY(cudaMallocHost(&a->h_lanes, (size_t)kLanesChain * S * 8));
  if (!a->lanes_ev) CUDA_TRY(cudaEventCreateWithFlags(&a->lanes_ev, cudaEventDisableTiming));
  Tables t = tables_for_launch(a, false);
  if (chain) {
    unsigned long long *d_chain = (unsigned long long *)(dm + o_tiles);
    CUDA_TRY(cudaMemsetAsync(d_chain, 0, nt * sizeof(unsigned long long), st));
    cudaError_t e = cudaSuccess;
    const char *dv = (const char *)d_values;
    const uint32_t *tp = (const uint32_t *)d_tpre;
    // TMA-streamed value blocks (k_lanes_bulk, a 2-stage ring) where they
    // measured faster than the register path (tools/lanes_probe.py A/B, two
    // runs: KB = 8 +5-7%, 32 +0-2%, 64 +4%; KB = 4 -12%, 16 -2..-8%: those
    // keep k_lanes_chunk).  GG_LANES_BULK=0 / 1: never / always.
    // L2 bulk prefetch distance (tiles) of the register-path lanes walk: one
    // tile ahead for 4 / 8 B elements (K1 int32 0.75 -> 0.79, K4 0.82 -> 0.86
    // of HBM), off for 1 / 2 B elements (instruction-bound: 0.46 -> 0.44);
    // profiles/r02_prefetch_ab.json.  A/B: GG_LANES_PF = distance
    static const int lanes_pf_env = [] { const char *e = getenv("GG_LANES_PF"); return e ? atoi(e) : -1; }();
    static const int bulk_env = [] {
      const char *e = getenv("GG_LANES_BULK");
      return e ? (e[0] == '0' ? 0 : 1) : -1;
    }();
    const bool bulk = bulk_env == 1 || (bulk_env < 0 && (KB == 8 || KB == 32 || KB == 64));
#define GG_CHAIN_CASE(ESZ_, KB_) \
  case KB_: \
    if (bulk) { \
      static std::atomic<uint64_t> attr{0}; \
      const uint64_t bit = uint64_t(1) << (a->dev & 63); \
      if (!(attr.load(std::memory_order_acquire) & bit)) { \
        cudaFuncSetAttribute(k_lanes_bulk<ESZ_, KB_, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 2 * 16384); \
        attr.fetch_or(bit, std::memory_order_acq_rel); \
      } \
      e = launch_k(k_lanes_bulk<ESZ_, KB_, 2>, (unsigned)nt, 256, (size_t)2 * 16384, st, t, dv, d_counts, tp, d_chain, \
                   C); \
    } else { \
      e = launch_k(k_lanes_chunk<ESZ_, KB_>, (unsigned)nt, 256, 0, st, t, dv, d_counts, tp, d_chain, C, \
                   lanes_pf_env >= 0 ? (uint32_t)lanes_pf_env : (ESZ_ >= 4 ? 1u : 0u)); \
    } \
    break;
    switch (a->esz) {
      case 1: switch (KB) { GG_CHAIN_CASE(1, 4) GG_CHAIN_CASE(1, 8) GG_CHAIN_CASE(1, 16) GG_CHAIN_CASE(1, 32) GG_CHAIN_CASE(1, 64) } break;
      case 2: switch (KB) { GG_CHAIN_CASE(2, 4) GG_CHAIN_CASE(2, 8) GG_CHAIN_CASE(2, 16) GG_CHAIN_CASE(2, 32) GG_CHAIN_CASE(2, 64) } break;
      case 4: switch (KB) { GG_CHAIN_CASE(4, 4) GG_CHAIN_CASE(4, 8) GG_CHAIN_CASE(4, 16) GG_CHAIN_CASE(4, 32) GG_CHAIN_CASE(4, 64) } break;
      default: switch (KB) { GG_CHAIN_CASE(8, 8) GG_CHAIN_CASE(8, 16) GG_CHAIN_CASE(8, 32) GG_CHAIN_CASE(8, 64) } break;
    }
#undef GG_CHAIN_CASE
    CUDA_TRY(e);
  } else {
  CUDA_TRY(launch_k(k_lanes_sum, (unsigned)((nt + 7) / 8), 256, 0, st, t, d_counts, (const uint32_t *)d_tpre,
                    d_tiles, (uint32_t)nt, T, (uint32_t)K));
  CUDA_TRY(launch_k(k_lanes_reserve, S, 256, 0, st, t, (const uint32_t *)d_tpre, d_tiles));
  cudaError_t e = cudaSuccess;
  const char *dv = (const char *)d_values;
  const LaneTile *ct = d_tiles;
#define GG_LANES_CASE(ESZ_, KB_) \
  case KB_: e = launch_k(k_lanes_scatter<ESZ_, KB_>, (unsigned)nt, 256, 0, st, t, dv, d_counts, ct); break;
  switch (a->esz) {
    case 1: switch (KB) { GG_LANES_CASE(1, 4) GG_LANES_CASE(1, 8) GG_LANES_CASE(1, 16) GG_LANES_CASE(1, 32) GG_LANES_CASE(1, 64) } break;
    case 2: switch (KB) { GG_LANES_CASE(2, 4) GG_LANES_CASE(2, 8) GG_LANES_CASE(2, 16) GG_LANES_CASE(2, 32) GG_LANES_CASE(2, 64) } break;
    case 4: switch (KB) { GG_LANES_CASE(4, 4) GG_LANES_CASE(4, 8) GG_LANES_CASE(4, 16) GG_LANES_CASE(4, 32) GG_LANES_CASE(4, 64) } break;
    default: switch (KB) { GG_LANES_CASE(8, 8) GG_LANES_CASE(8, 16) GG_LANES_CASE(8, 32) GG_LANES_CASE(8, 64) } break;
  }
#undef GG_LANES_CASE
  CUDA_TRY(e);
  }
  const uint32_t k = a->lanes_pend ? a->lanes_n : 0;
  CUDA_TRY(cudaMemcpyAsync(a->h_lanes + (size_t)k * S, a->t.size, S * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaEventRecord(a->lanes_ev, st));
  if (!a->lanes_pend) {
    a->lanes_head.swap(head);
    a->lanes_keep = mapped0;
  } else {
    a->lanes_head.insert(a->lanes_head.end(), head.begin(), head.end());
  }
  for (size_t i = 0; i < head.size(); i += 3)
    for (uint32_t s = head[i + 1]; s < head[i + 2]; ++s) a->lanes_hb[s] |= uint64_t(1) << head[i];
  for (uint32_t s = 0; s < S; ++s) a->lanes_ub[s] = base[s] + (off[s + 1] - off[s]) * K;
  a->lanes_pend = true;
  a->lanes_n = k + 1;
  return GG_OK;
}
}  // namespace

int gg_insert_lanes(gg_array *a, const void *d_values, const uint32_t *d_counts,
                    const uint64_t *h_lane_offsets, uint64_t values_per_lane,
                    int32_t *h_status, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  cudaStream_t st = S_(stream);
  // a tiled lanes insert pending (and nothing else): chain behind it without
  // waiting for its sizes (lanes_tiled plans on its upper bounds); any other
  // path resolves it first
  const bool chain = a->lanes_pend && !a->view_pend && a->lanes_n < kLanesChain;
  {
    int frc_ = check_no_view(a);
    if (!frc_) frc_ = chain ? order_stream(a, st) : enter(a, st);
    if (!frc_ && chain) frc_ = flush_meta(a, st, true);
    if (!frc_ && chain) frc_ = flush_grow(a, st, true);
    if (frc_) return frc_;
  }
  if (h_lane_offsets[0] != 0) return fail(GG_EVALUE, "lane offsets must start at 0");
  for (uint32_t s = 0; s < a->S; ++s)
    if (h_lane_offsets[s + 1] < h_lane_offsets[s]) return fail(GG_EVALUE, "lane offsets must be non-decreasing");
  if (values_per_lane == 0 || values_per_lane > 0xffffffffu) return fail(GG_EVALUE, "bad values_per_lane");
  if (h_lane_offsets[a->S] == 0) {
    if (h_status) memset(h_status, 0, a->S * sizeof(int32_t));
    return GG_OK;
  }
  {
    int frc = lanes_tiled(a, d_values, d_counts, h_lane_offsets, values_per_lane, st);
    if (frc != GG_ENOTSUP) {
      if (!frc && h_status) memset(h_status, 0, a->S * sizeof(int32_t));
      return frc;
    }
    // the exact path plans on exact sizes: finish what the chain skipped
    if (chain && (frc = enter(a, st))) return frc;
  }
  // exact two-pass path (allocator hook, live-bytes limit, shards with a
  // failed reservation, capacity exhaustion possible within the upper bound,
  // > 32 KiB of values per lane): counts summed on the device, brought back,
  // planned exactly like an insert
  void *dst[1] = {a->t.offsets};
  const void *src[1] = {h_lane_offsets};
  size_t bytes[1] = {(a->S + 1) * 8};
  int rc = a->up.upload(st, 1, dst, src, bytes);
  if (rc) return rc;
  // pass 1: per-shard totals -> host (one sync per launch, not per insert)
  { k_lanes_count<<<a->S, 1024, 0, st>>>(a->t, d_counts, (uint32_t)values_per_lane); g_launches.fetch_add(1, std::memory_order_relaxed); }
  CUDA_TRY(cudaGetLastError());
  std::vector<uint64_t> counts(a->S);
  CUDA_TRY(cudaMemcpyAsync(counts.data(), a->t.count, a->S * 8, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
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
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
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
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  int rc = check_committed_published(a);
  if (rc) return rc;
  Tables t = tables_for_launch(a, false);
  return launch_walk<W_FLATTEN>(a, t, nullptr, (char *)d_out, a->prefix[a->S], S_(stream));
}

int gg_flatten_range(gg_array *a, uint64_t lo, uint64_t hi, void *d_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  if (lo > hi || hi > a->prefix[a->S]) return fail(GG_EINDEX, "flatten range outside the committed size");
  if (lo == hi) return GG_OK;
  int rc = check_committed_published(a);
  if (rc) return rc;
  Tables t = tables_for_launch(a, false);
  Fuse fz{0, 0};
  fz.g0 = lo;
  fz.ulen = uniform_len(a);
  // the walk stores element g at flat_dst + g * esz: shift the base so that
  // element lo lands at d_out (never dereferenced below lo)
  char *base = (char *)d_out - lo * a->esz;
  return walk_copy<W_FLATTEN, false>(a, t, nullptr, base, hi, fz, S_(stream));
}

namespace {
// one launch of k_gather for get_many (scatter = 0) / set_many (1)
int launch_gather(gg_array *a, const int64_t *d_idx, uint64_t n, char *out, const char *vals, int scatter,
                  cudaStream_t st, uint64_t lim = 0, unsigned int *bad = nullptr) {
  Tables t = tables_for_launch(a, false);
  const bool smem = a->S < 4096;
  const size_t sb = smem ? (size_t)(a->S + 1) * 8 : 0;
  // one tile of 256 x kGatherU indices per CTA (no grid-stride cap): CTAs at different
  // phases (index loads, bisects, random element accesses) overlap on an SM
  // (8 indices per thread measured slower: 0.467 -> 0.493 ms, profiles/r02_prefetch_ab.json)
  const uint64_t per_cta = 256ull * kGatherU;
  const int grid = (int)std::min<uint64_t>((n + per_cta - 1) / per_cta, 0x7fffffffull);
  // cache policy of the random element reads (A/B: GG_GATHER_LD, see ld_rand)
  // (.L1::no_allocate by default: a random element is read once; 2% faster under ncu than the
  // L1-allocating load, profiles/r02_gather_ld_ab.json)
  static const int ldm = [] { const char *e = getenv("GG_GATHER_LD"); return e ? atoi(e) : 2; }();
  cudaError_t e = cudaSuccess;
#define GG_GATHER(ESZ_) \
  e = smem ? launch_k(k_gather<ESZ_, true>, grid, 256, sb, st, t, d_idx, n, out, vals, scatter, ldm, lim, bad) \
           : launch_k(k_gather<ESZ_, false>, grid, 256, 0, st, t, d_idx, n, out, vals, scatter, ldm, lim, bad);
  switch (a->esz) {
    case 1: GG_GATHER(1) break;
    case 2: GG_GATHER(2) break;
    case 4: GG_GATHER(4) break;
    default: GG_GATHER(8) break;
  }
#undef GG_GATHER
  CUDA_TRY(e);
  return GG_OK;
}
}  // namespace

int gg_gather(gg_array *a, const int64_t *d_idx, uint64_t n, void *d_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  if (n == 0) return GG_OK;
  return launch_gather(a, d_idx, n, (char *)d_out, nullptr, 0, S_(stream));
}

int gg_gather_checked(gg_array *a, const int64_t *d_idx, uint64_t n, void *d_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  cudaStream_t st = S_(stream);
  { int frc_ = enter(a, st); if (frc_) return frc_; }
  if (n == 0) return GG_OK;
  const uint64_t lim = a->prefix[a->S];
  if (lim == 0) return fail(GG_EINDEX, "index outside the committed size");
  // the bounds check rides in the gather (no separate pass over the
  // indices): a flag word in the device scratch, cleared first, read back
  unsigned int *d_bad = (unsigned int *)(a->d_scratch + 48);
  CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(unsigned int), st));
  int rc = launch_gather(a, d_idx, n, (char *)d_out, nullptr, 0, st, lim, d_bad);
  if (rc) return rc;
  if (!a->h_scratch) CUDA_TRY(cudaMallocHost(&a->h_scratch, 64));   // pinned, on first use
  CUDA_TRY(cudaMemcpyAsync(a->h_scratch + 48, d_bad, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  unsigned int badv;
  memcpy(&badv, a->h_scratch + 48, sizeof badv);
  if (badv) return fail(GG_EINDEX, "index outside the committed size");
  return GG_OK;
}

int gg_scatter_checked(gg_array *a, const int64_t *d_idx, uint64_t n, const void *d_vals, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  cudaStream_t st = S_(stream);
  { int frc_ = enter(a, st); if (frc_) return frc_; }
  if (n == 0) return GG_OK;
  const uint64_t lim = a->prefix[a->S];
  if (lim == 0) return fail(GG_EINDEX, "index outside the committed size");
  // bounds pass -> flag; the scatter behind it writes nothing if the flag is
  // set (no partial update on error); the flag is read back at the end
  unsigned int *d_bad = (unsigned int *)(a->d_scratch + 48);
  CUDA_TRY(cudaMemsetAsync(d_bad, 0, sizeof(unsigned int), st));
  const int grid = (int)std::min<uint64_t>((n + 1023) / 1024, (uint64_t)sm_count(a->dev) * 8);
  CUDA_TRY(launch_k(k_check_idx, std::max(grid, 1), 256, 0, st, d_idx, n, lim, d_bad));
  int rc = launch_gather(a, d_idx, n, nullptr, (const char *)d_vals, 1, st, lim, d_bad);
  if (rc) return rc;
  if (!a->h_scratch) CUDA_TRY(cudaMallocHost(&a->h_scratch, 64));   // pinned, on first use
  CUDA_TRY(cudaMemcpyAsync(a->h_scratch + 48, d_bad, sizeof(unsigned int), cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  unsigned int badv;
  memcpy(&badv, a->h_scratch + 48, sizeof badv);
  if (badv) return fail(GG_EINDEX, "index outside the committed size");
  return GG_OK;
}

int gg_scatter(gg_array *a, const int64_t *d_idx, uint64_t n, const void *d_vals, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  if (n == 0) return GG_OK;
  return launch_gather(a, d_idx, n, nullptr, (const char *)d_vals, 1, S_(stream));
}

namespace {
int elem_addr(gg_array *a, uint32_t s, uint64_t i, char **out, cudaStream_t st) {
  if (s >= a->S) return fail(GG_EVALUE, "shard out of range");
  if (i >= a->size[s]) return fail(GG_EINDEX, "index outside size");
  uint32_t b; uint64_t o;
  host_locate(a, i, b, o);
  if (b >= a->MB || !(a->flags[s] >> b & 1))
    return fail(GG_EUNPUBLISHED, "index is reserved but its bucket is unpublished");
  (void)st;
  // the bucket's slot is host-known (class base + s * bucket bytes): no
  // device round trip for the address
  char *p = (char *)a->slab.class_base(b) + (uint64_t)s * bucket_bytes(a, b);
  *out = p + o * a->esz;
  return GG_OK;
}
}  // namespace

int gg_get(gg_array *a, uint32_t s, uint64_t i, void *h_out, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
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
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
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

namespace {
// Back every slot a device-side append may take (buckets [0,
// min_buckets_for(max)) per shard, in shard then bucket order, while the
// live-bytes cap allows) and publish the backed-slot masks on stream st.
// sync: wait for the device (the public entry point, whose user kernel may
// run on any stream); the library's own push_if stays stream-ordered.
// pend_hb: buckets pending (chained) push_if calls already backed as headroom
// -- allowed in the mask, not backed again
int view_prepare(gg_array *a, const uint64_t *h_max_sizes, cudaStream_t st, bool sync, gg_device_view *out,
                 bool *complete = nullptr, const uint64_t *pend_hb = nullptr) {
  if (a->view_out) return fail(GG_EVALUE, "a device view is outstanding (call gg_device_view_sync)");
  std::vector<unsigned long long> am(a->S);
  uint64_t live = a->live;
  if (!pend_hb) a->view_keep = a->slab.mapped;
  bool stop = false;
  for (uint32_t s = 0; s < a->S; ++s) am[s] = a->flags[s] | (pend_hb ? pend_hb[s] : 0);
  if (h_max_sizes && !a->limit && g_batch_backing) {
    // no live-bytes cap: class by class in runs of consecutive shards (one
    // batched refcount pass per run; a run that cannot be backed goes slot by
    // slot); best effort, stops at the first slot that cannot be backed
    std::vector<uint32_t> k(a->S);
    uint32_t kmax = 0;
    for (uint32_t s = 0; s < a->S; ++s) {
      k[s] = std::min<uint32_t>(min_buckets_for(a, h_max_sizes[s]), a->MB);
      kmax = std::max(kmax, k[s]);
    }
    for (uint32_t b = 0; b < kmax && !stop; ++b) {
      bool have_region = false;
      for (uint32_t s = 0; s < a->S && !stop;) {
        auto need = [&](uint32_t x) { return b < k[x] && !(am[x] >> b & 1); };
        if (!need(s)) { ++s; continue; }
        uint32_t e = s + 1;
        while (e < a->S && need(e)) ++e;
        if (!have_region) {
          bool created = false;
          if (a->slab.ensure_region(b, &created) != GG_OK) { stop = true; break; }
          if (created) a->cbase_dirty = true;
          have_region = true;
        }
        if (run_backed(a, b, s, e)) {
          for (uint32_t x = s; x < e; ++x) am[x] |= 1ull << b;
          a->headroom.push_back(b); a->headroom.push_back(s); a->headroom.push_back(e);
        } else {                                 // slot by slot, up to the first that fails
          for (uint32_t x = s; x < e && !stop; ++x) {
            if (a->slab.back(x, b) != GG_OK) { stop = true; break; }
            am[x] |= 1ull << b;
            a->headroom.push_back(b); a->headroom.push_back(x); a->headroom.push_back(x + 1);
          }
        }
        s = e;
      }
    }
  } else if (h_max_sizes) {
    // live-bytes cap (or per-bucket backing): shard then bucket order, while
    // the cap allows
    for (uint32_t s = 0; s < a->S && !stop; ++s) {
      const uint32_t k = std::min<uint32_t>(min_buckets_for(a, h_max_sizes[s]), a->MB);
      for (uint32_t b = 0; b < k; ++b) {
        if (am[s] >> b & 1) continue;
        const uint64_t nb = bucket_bytes(a, b);
        if ((a->limit && live + nb > a->limit) || back_bucket(a, s, b) != GG_OK) { stop = true; break; }
        live += nb;
        am[s] |= 1ull << b;
        a->headroom.push_back(b); a->headroom.push_back(s); a->headroom.push_back(s + 1);
      }
    }
  }
  if (complete) *complete = !stop;
  int rc = push_cbase(a, st);
  if (rc) return rc;
  void *dst[1] = {a->t.amask};
  const void *src[1] = {am.data()};
  size_t bytes[1] = {a->S * 8};
  if ((rc = a->up.upload(st, 1, dst, src, bytes))) return rc;
  if (sync) CUDA_TRY(cudaDeviceSynchronize());
  gg_device_view v = a->t;
  v.ctl = nullptr;                          // amask gates the device allocator
  *out = v;
  a->view_out = true;                       // mutating calls refused until the view is synced
  return GG_OK;
}

// refresh the host mirrors from the device after device-side appends: one
// asynchronous copy of sizes / capacities / ops / published masks / status /
// counters into a pinned buffer and ONE stream synchronize
int view_finish(gg_array *a, int32_t *h_status, cudaStream_t st) {
  int rc = view_finish_issue(a, st);
  if (rc) return rc;
  CUDA_TRY(cudaStreamSynchronize(st));
  a->view_out = false;
  return view_finish_host(a, h_status, st);
}
}  // namespace

int gg_device_view_get(gg_array *a, const uint64_t *h_max_sizes, void *h_view, uint64_t view_bytes) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = flush_pending(a); if (frc_) return frc_; }
  if (view_bytes != sizeof(gg_device_view)) return fail(GG_EVALUE, "view size mismatch (ggarray_device.cuh)");
  gg_device_view v;
  // the view's user kernel may run on any stream: prepared on the legacy
  // stream and waited for
  int rc = view_prepare(a, h_max_sizes, 0, true, &v);
  if (rc) return rc;
  memcpy(h_view, &v, sizeof v);
  return GG_OK;
}

// refresh the host mirrors from the device after user kernels appended
int gg_device_view_sync(gg_array *a, int32_t *h_status, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  return view_finish(a, h_status, S_(stream));
}

int gg_push_if(gg_array *a, const void *d_vals, const uint8_t *d_pred, uint64_t n, int32_t mode,
               uint32_t grid, int32_t *h_status, void *stream) {
  cudaStream_t st = S_(stream);
  if (n == 0) return GG_OK;
  const uint32_t B = 256;
  // default grid: exactly the resident CTAs (one wave: each CTA then loops
  // over many rounds and each append call reserves up to R rounds at once; a
  // grid above residency leaves a half-empty second wave), at least one CTA
  // per shard
  if (!grid) {
    int per_sm = 0;
#define GG_PUSH_OCC(ESZ_) \
  (mode ? cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_push_if<ESZ_, 256, true>, B, 0) \
        : cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_push_if<ESZ_, 256, false>, B, 0))
    switch (a->esz) {
      case 1: GG_PUSH_OCC(1); break;
      case 2: GG_PUSH_OCC(2); break;
      case 4: GG_PUSH_OCC(4); break;
      default: GG_PUSH_OCC(8); break;
    }
#undef GG_PUSH_OCC
    if (per_sm <= 0) per_sm = 4;
    grid = (uint32_t)std::max<uint64_t>(
        a->S, std::min<uint64_t>((n + kPushSlice * 8 - 1) / (kPushSlice * 8),
                                 (uint64_t)sm_count(a->dev) * per_sm));
  }
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  // a deferred push_if pending (and nothing else): chain behind it, planning
  // on its upper bounds, without waiting for its readback
  const bool chain = a->view_pend && !a->lanes_pend && !a->limit && g_batch_backing &&
                     a->view_n < kLanesChain && !capturing_now(a, st);
  {
    int frc_ = check_no_view(a);
    if (!frc_) frc_ = chain ? order_stream(a, st) : enter(a, st);
    if (!frc_ && chain) frc_ = flush_meta(a, st, true);
    if (!frc_ && chain) frc_ = flush_grow(a, st, true);
    if (frc_) return frc_;
  }
  if (a->view_ub.size() != a->S) { a->view_ub.assign(a->S, 0); a->view_hb.assign(a->S, 0); }
  // worst case: every candidate of shard s appended (block blk takes slice
  // blk of every round of grid * kPushSlice candidates)
  std::vector<uint64_t> maxsz(a->S, 0);
  const uint64_t per_round = (uint64_t)grid * kPushSlice, full = n / per_round, rem = n % per_round;
  for (uint32_t blk = 0; blk < grid; ++blk) {
    const uint64_t lo = (uint64_t)blk * kPushSlice;
    maxsz[blk % a->S] += full * kPushSlice + (rem > lo ? std::min<uint64_t>(kPushSlice, rem - lo) : 0);
  }
  const uint64_t *base = chain ? a->view_ub.data() : a->size.data();
  for (uint32_t s = 0; s < a->S; ++s) maxsz[s] += base[s];
  gg_device_view v;
  bool backed = false;
  const size_t h0 = a->headroom.size();
  int rc = view_prepare(a, maxsz.data(), st, false, &v, &backed, chain ? a->view_hb.data() : nullptr);
  if (rc) return rc;
  // every slot the launch can reach is backed and within max_buckets: no
  // append can fail, so the host mirrors are refreshed lazily (the readback
  // is queued behind an event and resolved by the next call that needs the
  // mirrors, like the lanes insert) instead of waiting for the kernel here
  bool can_fail = !backed;
  for (uint32_t s = 0; s < a->S && !can_fail; ++s) can_fail = min_buckets_for(a, maxsz[s]) > a->MB;
  // vector loads: 16 B of values (8 B elements: 32 B) and G predicate bytes
  const uint32_t pg = a->esz >= 4 ? 4 : 16 / a->esz;
  const int al = ((uintptr_t)d_vals % (pg * a->esz) == 0 && (uintptr_t)d_pred % pg == 0) ? 1 : 0;
  // L2 bulk prefetch of the next append call's slices: on in block mode for
  // 4 / 8 B elements (block int32 0.73 -> 0.76, int64 0.79 -> 0.87 of HBM),
  // off in warp mode (int32 0.79 -> 0.72 with it) and for 1 / 2 B elements;
  // profiles/r02_prefetch_ab.json.  A/B: GG_PUSH_PF = 0 | 1
  static const int push_pf_env = [] { const char *e = getenv("GG_PUSH_PF"); return e ? atoi(e) : -1; }();
  const uint32_t push_pf = push_pf_env >= 0 ? (uint32_t)push_pf_env : (mode && a->esz >= 4 ? 1u : 0u);
  switch (a->esz) {
#define GG_PUSH_CASE(ESZ_) \
    case ESZ_: \
      if (mode) k_push_if<ESZ_, 256, true><<<grid, B, 0, st>>>(v, (const char *)d_vals, d_pred, n, al, push_pf); \
      else k_push_if<ESZ_, 256, false><<<grid, B, 0, st>>>(v, (const char *)d_vals, d_pred, n, al, push_pf); \
      g_launches.fetch_add(1, std::memory_order_relaxed); \
      break;
    GG_PUSH_CASE(1) GG_PUSH_CASE(2) GG_PUSH_CASE(4) GG_PUSH_CASE(8)
#undef GG_PUSH_CASE
  }
  CUDA_TRY(cudaGetLastError());
  if (can_fail || capturing_now(a, st)) {
    // synchronous readback: the device tables it copies are exact, so it
    // also settles any chained calls before this one (all their headroom)
    a->view_pend = false;
    a->view_n = 0;
    std::fill(a->view_hb.begin(), a->view_hb.end(), 0);
    return view_finish(a, h_status, st);
  }
  if ((rc = view_finish_issue(a, st))) return rc;
  if (!a->lanes_ev) CUDA_TRY(cudaEventCreateWithFlags(&a->lanes_ev, cudaEventDisableTiming));
  CUDA_TRY(cudaEventRecord(a->lanes_ev, st));
  for (size_t i = h0; i < a->headroom.size(); i += 3)
    for (uint32_t s = a->headroom[i + 1]; s < a->headroom[i + 2]; ++s) a->view_hb[s] |= uint64_t(1) << a->headroom[i];
  for (uint32_t s = 0; s < a->S; ++s) a->view_ub[s] = maxsz[s];
  a->view_pend = true;
  a->view_n += 1;
  a->view_out = false;
  if (h_status) memset(h_status, 0, a->S * sizeof(int32_t));
  return GG_OK;
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

int gg_set_batch_backing(int32_t mode) {
  if (mode < 0 || mode > 2) return fail(GG_EVALUE, "batch backing mode must be 0, 1 or 2");
  g_batch_backing = mode;
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
  a->cap_parity = a->cur;
  if (on && !a->up.capturing) return a->up.begin_capture();
  if (!on) a->up.capturing = false;
  return GG_OK;
}

int gg_flush(gg_array *a) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  return flush_pending(a);
}

int gg_capture_end(gg_array *a, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  int rc = enter(a, S_(stream));
  if (rc) return rc;
  if (a->cur != a->cap_parity) {     // an odd number of fused walks: copy back, restore the parity
    const int o = a->cur ^ 1;
    CUDA_TRY(launch_k(k_copy_db, (a->S + 256) / 256, 256, 0, S_(stream), a->sz_buf[o],
                      (const uint64_t *)a->sz_buf[a->cur], a->pf_buf[o],
                      (const uint64_t *)a->pf_buf[a->cur], a->S));
    flip_buffers(a);
  }
  return GG_OK;
}

int gg_set_fuse(int32_t on) {
  g_fuse = on != 0;
  return GG_OK;
}

int gg_capture_release(gg_array *a) {
  std::lock_guard<std::mutex> g(a->mu);
  cudaDeviceSynchronize();
  a->up.release_captured();
  return GG_OK;
}

int gg_summary(gg_array *a, uint64_t *o) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int rc = resolve_lanes(a); if (rc) return rc; }
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
  use_dev(a->dev);
  { int rc = resolve_lanes(a); if (rc) return rc; }
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
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
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
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  CUDA_TRY(cudaMemcpyAsync(d_out, a->t.prefix, (a->S + 1) * 8, cudaMemcpyDeviceToDevice, S_(stream)));
  return GG_OK;
}

int gg_bucket_ptrs(gg_array *a, uint64_t *h_ptrs, void *stream) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int frc_ = enter(a, S_(stream)); if (frc_) return frc_; }
  CUDA_TRY(cudaStreamSynchronize(S_(stream)));
  CUDA_TRY(cudaMemcpy(h_ptrs, a->t.ptr, (size_t)a->S * a->MB * 8, cudaMemcpyDeviceToHost));
  return GG_OK;
}

int gg_mem_stats(gg_array *a, uint64_t *o, void *stream) {
  (void)stream;
  std::lock_guard<std::mutex> g(a->mu);
  uint64_t cap = 0, need = 0;
  for (uint32_t s = 0; s < a->S; ++s) { cap += a->cap[s]; need += a->size[s]; }
  use_dev(a->dev);
  { int rc = resolve_lanes(a); if (rc) return rc; }
  { int rc = settle_adopted(a, a->have_last ? a->last_st : nullptr); if (rc) return rc; }
  a->slab.reap_doomed(false);
  o[0] = cap * a->esz; o[1] = a->slab.mapped; o[2] = a->live; o[3] = need * a->esz;
  o[4] = a->alloc_calls; o[5] = a->slab.cached; o[6] = a->slab.doomed_bytes;
  return GG_OK;
}

int gg_pool_stats(int device, uint64_t *o) {
  if (device < 0 || device >= 64) return fail(GG_EVALUE, "bad device");
  reclaim(false);
  size_t nslabs = 0;
  uint64_t slab_hits = 0;
  {
    SlabCache &C = slab_cache();
    std::lock_guard<std::mutex> g(C.mu);
    for (Slab *x : C.slabs) nslabs += x->dev == device;
    slab_hits = C.hits;
  }
  ChunkPool &p = chunk_pool();
  std::lock_guard<std::mutex> g(p.mu);
  o[0] = p.bytes[device]; o[1] = p.free[device].size(); o[2] = p.hits; o[3] = p.misses; o[4] = p.cap(device);
  o[7] = p.slab_bytes[device]; o[8] = nslabs; o[9] = slab_hits;
  Reclaimer &R = reclaimer();
  std::lock_guard<std::mutex> l(R.mu);
  o[5] = R.graves.size(); o[6] = p.refused;
  return GG_OK;
}

int gg_pool_trim(int device) {
  if (device < 0 || device >= 64) return fail(GG_EVALUE, "bad device");
  reclaim(true);
  slab_cache_evict(device);
  chunk_pool().trim(device);
  return GG_OK;
}

int gg_slab_stats(gg_array *a, uint64_t *o) {
  std::lock_guard<std::mutex> g(a->mu);
  use_dev(a->dev);
  { int rc = resolve_lanes(a); if (rc) return rc; }
  const Slab &sl = a->slab;
  o[0] = sl.mapped; o[1] = sl.cached; o[2] = sl.n_map; o[3] = sl.n_unmap;
  o[4] = sl.ns_map; o[5] = sl.ns_unmap; o[6] = sl.n_regions; o[7] = sl.va_used;
  o[8] = sl.n_create; o[9] = sl.n_pool; o[10] = sl.doomed_bytes;
  return GG_OK;
}

// ---------------------------------------------------------------- baselines
int gg_flat_insert(void *d_buf, uint64_t capacity, uint64_t *d_counter, const void *d_vals,
                   uint64_t n, uint32_t esz, int32_t algo, void *stream) {
  if (n == 0) return GG_OK;
  int dev = 0;
  cudaGetDevice(&dev);
  cudaStream_t st = S_(stream);
  if (algo == GG_ALGO_BATCH)
    return fail(GG_EVALUE, "BATCH: one host-side reservation, then gg_flat_append");
  if (algo == GG_ALGO_BLOCK) {
    // vectorised block reservation: tile = 256 threads x 8 x 16 B (tools/sweep.py U)
    const uint64_t tile = 256ull * 8 * (16 / esz);
    const unsigned grid_b = (unsigned)std::max<uint64_t>(1, (n + tile - 1) / tile);
    cudaError_t e;
    switch (esz) {
      case 1: e = launch_k(k_flat_insert_block<1, 8>, grid_b, 256, 0, st, (char *)d_buf, capacity, (unsigned long long *)d_counter, (const char *)d_vals, n, tile); break;
      case 2: e = launch_k(k_flat_insert_block<2, 8>, grid_b, 256, 0, st, (char *)d_buf, capacity, (unsigned long long *)d_counter, (const char *)d_vals, n, tile); break;
      case 4: e = launch_k(k_flat_insert_block<4, 8>, grid_b, 256, 0, st, (char *)d_buf, capacity, (unsigned long long *)d_counter, (const char *)d_vals, n, tile); break;
      case 8: e = launch_k(k_flat_insert_block<8, 8>, grid_b, 256, 0, st, (char *)d_buf, capacity, (unsigned long long *)d_counter, (const char *)d_vals, n, tile); break;
      default: return fail(GG_EVALUE, "bad element size");
    }
    CUDA_TRY(e);
    return GG_OK;
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

int gg_flat_append(void *d_buf, uint64_t capacity, uint64_t *d_counter, uint64_t start,
                   const void *d_vals, uint64_t n, uint32_t esz, void *stream) {
  if (n == 0) return GG_OK;
  if (start > capacity || n > capacity - start) return fail(GG_ECAPACITY, "batch exceeds the capacity");
  cudaStream_t st = S_(stream);
  const uint64_t tile = 256ull * 8 * (16 / (esz ? esz : 1));
  const unsigned grid = (unsigned)std::max<uint64_t>(1, (n + tile - 1) / tile);
  cudaError_t e;
  switch (esz) {
    case 1: e = launch_k(k_flat_append<1, 8>, grid, 256, 0, st, (char *)d_buf, start, (unsigned long long *)d_counter, (const char *)d_vals, n, tile); break;
    case 2: e = launch_k(k_flat_append<2, 8>, grid, 256, 0, st, (char *)d_buf, start, (unsigned long long *)d_counter, (const char *)d_vals, n, tile); break;
    case 4: e = launch_k(k_flat_append<4, 8>, grid, 256, 0, st, (char *)d_buf, start, (unsigned long long *)d_counter, (const char *)d_vals, n, tile); break;
    case 8: e = launch_k(k_flat_append<8, 8>, grid, 256, 0, st, (char *)d_buf, start, (unsigned long long *)d_counter, (const char *)d_vals, n, tile); break;
    default: return fail(GG_EVALUE, "bad element size");
  }
  CUDA_TRY(e);
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
