// gg_host.cuh -- host-side runtime of the B200 GGArray library: the CUDA-VMM
// arena (memMap baseline) and bucket slabs (refcounted chunk mapping), the
// PDL kernel launcher, and the pinned upload ring.
#ifndef GG_HOST_CUH
#define GG_HOST_CUH

#include "gg_device.cuh"

namespace gg {

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

// Process-wide cache of physical chunks released by DESTROYED arrays, per
// device and chunk size: a new array maps a cached handle (cuMemMap +
// cuMemSetAccess) instead of creating one, which avoids the driver's
// allocate / scrub / free churn when arrays come and go (config 1 builds an
// array per call).  Bounded (GG_POOL_BYTES, default 4 GiB per device) and
// reported by gg_pool_stats / emptied by gg_pool_trim; a shrink's release
// and trim() always return memory to the driver, so a live array's mapped
// bytes are its whole footprint.
struct ChunkPool {
  std::mutex mu;
  std::vector<std::pair<size_t, CUmemGenericAllocationHandle>> free[64];
  uint64_t bytes[64] = {0};
  uint64_t hits = 0, misses = 0;
  uint64_t cap() {
    static uint64_t c = [] {
      const char *e = getenv("GG_POOL_BYTES");
      return e ? strtoull(e, nullptr, 10) : (uint64_t(4) << 30);
    }();
    return c;
  }
  bool take(int dev, size_t size, CUmemGenericAllocationHandle *h) {
    if (dev < 0 || dev >= 64) return false;
    std::lock_guard<std::mutex> g(mu);
    auto &v = free[dev];
    for (size_t i = v.size(); i-- > 0;)
      if (v[i].first == size) {
        *h = v[i].second;
        v.erase(v.begin() + i);
        bytes[dev] -= size;
        ++hits;
        return true;
      }
    ++misses;
    return false;
  }
  bool give(int dev, size_t size, CUmemGenericAllocationHandle h) {
    if (dev < 0 || dev >= 64) return false;
    std::lock_guard<std::mutex> g(mu);
    if (bytes[dev] + size > cap()) return false;
    free[dev].push_back({size, h});
    bytes[dev] += size;
    return true;
  }
  void trim(int dev) {
    std::lock_guard<std::mutex> g(mu);
    for (auto &e : free[dev]) drv().release(e.second);
    free[dev].clear();
    bytes[dev] = 0;
  }
};

inline ChunkPool &chunk_pool() {
  static ChunkPool p;
  return p;
}

// Slab store of one GGArray: a VA region per bucket class, slot s of class b
// = bucket (s, b).  Physical memory is mapped per chunk (a gran-multiple
// piece of a region) and refcounted by the live buckets overlapping it, so
// releasing buckets returns memory as soon as a chunk empties.  Classes whose
// region is smaller than one granule share one packed region ("small"), so a
// tiny array costs one granule, not one per class.
struct Slab {
  struct Chunk { uint32_t refs = 0; bool mapped = false; CUmemGenericAllocationHandle h = 0; };
  struct Region { CUdeviceptr base = 0; size_t va = 0, chunk = 0; std::vector<Chunk> chunks; };
  static constexpr size_t kChunk = size_t(1) << 30;    // largest mapping unit of a region
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
  // one bucket, 1/8..1/16 of the region, at most kChunk.  Each cuMemCreate /
  // Map / SetAccess call costs ~1.5-2 ms of driver time almost regardless of
  // size (tools/vmm_fresh_probe.py: 8 GiB as 128 x 64 MiB 250-1450 ms, as
  // 8 x 1 GiB 36 ms), so chunks are large; a partly live top class (an
  // uneven split) strands at most one chunk, <= 1/8 of its region.
  uint64_t chunk_for(uint32_t b) const {
    if (bytes[b] >= kChunk) return bytes[b];
    const uint64_t R = S * bytes[b];
    uint64_t c = gran;
    while (c < kChunk && c * 16 <= R) c <<= 1;
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
    if (!chunk_pool().take(dev, r.chunk, &k.h)) {
      CUmemAllocationProp prop = props();
      CU_TRY(drv().create(&k.h, r.chunk, &prop, 0));
    }
    const CUdeviceptr at = r.base + c * r.chunk;
    if (drv().map(at, r.chunk, 0, k.h, 0) != CUDA_SUCCESS) {
      drv().release(k.h);
      return fail(GG_ENOMEM, "cuMemMap failed");
    }
    // access rights are granted in finalize_access(), one cuMemSetAccess per
    // contiguous run of chunks mapped by the same operation (the call costs
    // about as much as the mapping itself)
    pending.push_back({&r, c});
    static const bool batch = [] { const char *e = getenv("GG_BATCH_ACCESS"); return !e || e[0] != '0'; }();
    if (!batch) {
      int rc = finalize_access();
      if (rc) return rc;
    }
    k.mapped = true;
    mapped += r.chunk;
    n_map += 1;
    ns_map += now_ns() - t0;
    return GG_OK;
  }
  std::vector<std::pair<Region *, size_t>> pending;   // mapped, access not granted yet
  // grant read/write access to every chunk mapped since the last call; must
  // run before a kernel can touch them (push_cbase calls it)
  int finalize_access() {
    if (pending.empty()) return GG_OK;
    const uint64_t t0 = now_ns();
    std::sort(pending.begin(), pending.end());
    CUmemAccessDesc acc = {};
    acc.location.type = CU_MEM_LOCATION_TYPE_DEVICE;
    acc.location.id = dev;
    acc.flags = CU_MEM_ACCESS_FLAGS_PROT_READWRITE;
    int rc = GG_OK;
    for (size_t i = 0; i < pending.size();) {
      Region *r = pending[i].first;
      size_t j = i + 1;
      while (j < pending.size() && pending[j].first == r && pending[j].second == pending[j - 1].second + 1) ++j;
      const CUdeviceptr at = r->base + pending[i].second * r->chunk;
      if (drv().set_access(at, (j - i) * r->chunk, &acc, 1) != CUDA_SUCCESS && !rc)
        rc = fail(GG_ENOMEM, "cuMemSetAccess failed");
      i = j;
    }
    pending.clear();
    ns_map += now_ns() - t0;
    return rc;
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
    finalize_access();
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
    finalize_access();
    auto go = [&](Region &r) {
      for (size_t c = 0; c < r.chunks.size(); ++c)
        if (r.chunks[c].mapped && r.chunks[c].refs == 0) unmap_chunk(r, c);
    };
    go(small);
    for (auto &r : big) go(r);
  }
  // the array is going away: unmap everything, keep physical chunks in the
  // process pool while it has room (the caller synchronised the device)
  void destroy() {
    pending.clear();
    auto go = [&](Region &r) {
      for (size_t c = 0; c < r.chunks.size(); ++c)
        if (r.chunks[c].mapped) {
          drv().unmap(r.base + c * r.chunk, r.chunk);
          if (!chunk_pool().give(dev, r.chunk, r.chunks[c].h)) drv().release(r.chunks[c].h);
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

#endif  // GG_HOST_CUH
