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

// Process-wide cache of physical chunks, per device and chunk size (the
// chunk size is a function of the bucket class and S, so the lists are
// per-class free lists in effect): chunks of destroyed arrays and chunks a
// shrink / trim unmaps go here, and a slab maps a cached handle (cuMemMap +
// cuMemSetAccess) before asking the driver for a new one (cuMemCreate scrubs
// pages; cuMemRelease frees them -- the expensive half of the VMM calls).
// Bounded by GG_POOL_BYTES (default: a quarter of the device's memory, so an
// array of up to that size is rebuilt entirely from cached chunks), reported
// by gg_pool_stats, emptied by gg_pool_trim -- and emptied on demand when a
// cuMemCreate runs out of memory.  A live array's mapped bytes are its
// footprint; pooled chunks belong to no array.
struct ChunkPool {
  std::mutex mu;
  std::vector<std::pair<size_t, CUmemGenericAllocationHandle>> free[64];
  uint64_t bytes[64] = {0};
  uint64_t slab_bytes[64] = {0};           // mapped bytes of cached slabs (SlabCache), same cap
  uint64_t caps[64] = {0};
  uint64_t hits = 0, misses = 0, refused = 0;
  uint64_t cap(int dev) {                  // caller holds mu
    if (!caps[dev]) {
      const char *e = getenv("GG_POOL_BYTES");
      if (e) {
        caps[dev] = strtoull(e, nullptr, 10);
        if (!caps[dev]) caps[dev] = 1;     // 0 = no pooling
      } else {
        size_t fr = 0, tot = 0;
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != dev) cudaSetDevice(dev);
        if (cudaMemGetInfo(&fr, &tot) != cudaSuccess || !tot) tot = size_t(16) << 30;
        if (cur != dev && cur >= 0) cudaSetDevice(cur);
        caps[dev] = tot / 4;
      }
    }
    return caps[dev];
  }
  bool take(int dev, size_t size, CUmemGenericAllocationHandle *h) {
    if (dev < 0 || dev >= 64) return false;
    std::lock_guard<std::mutex> g(mu);
    auto &v = free[dev];
    for (size_t i = v.size(); i-- > 0;)
      if (v[i].first == size) {
        *h = v[i].second;
        v[i] = v.back();
        v.pop_back();
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
    if (bytes[dev] + slab_bytes[dev] + size > cap(dev)) { ++refused; return false; }
    free[dev].push_back({size, h});
    bytes[dev] += size;
    return true;
  }
  // release cached handles to the driver (all of them, or until `want` bytes
  // were freed)
  uint64_t trim(int dev, uint64_t want = ~uint64_t(0)) {
    std::lock_guard<std::mutex> g(mu);
    uint64_t got = 0;
    auto &v = free[dev];
    while (!v.empty() && got < want) {
      drv().release(v.back().second);
      got += v.back().first;
      bytes[dev] -= v.back().first;
      v.pop_back();
    }
    return got;
  }
};

inline ChunkPool &chunk_pool() {
  static ChunkPool p;
  return p;
}

// deferred teardown (defined below): free what destroyed arrays left once the
// work queued on them completed; wait = block until all of it has
inline void reclaim(bool wait);

// Slab store of one GGArray: a VA region per bucket class, slot s of class b
// = bucket (s, b).  Physical memory is refcounted per grid chunk (a
// gran-multiple piece of a region) by the live buckets overlapping it, and
// mapped in EXTENTS -- runs of consecutive grid chunks backed by ONE
// physical handle: a uniform operation that backs all S slots of a class
// maps the whole region with one cuMemCreate + cuMemMap and one
// cuMemSetAccess per operation (the driver charges ~0.5-1 ms per call almost
// regardless of size: B200 probe, 8 GiB as one handle 1.0 ms, as 8 x 1 GiB
// 4.8 ms, as 80 chunks ~21-111 ms), while per-shard backing (ragged plans)
// maps single grid chunks, so an uneven split strands at most one grid
// chunk (<= 1/8 of the region).  An extent is unmapped when none of its
// chunks holds a live bucket.  Classes whose region is smaller than one
// granule share one packed region ("small"), so a tiny array costs one
// granule, not one per class.
struct Slab {
  struct Chunk {
    uint32_t refs = 0;
    bool mapped = false, doomed = false;
    uint32_t head = 0;                      // first grid chunk of its extent
    uint32_t len = 0;                       // (head only) grid chunks in the extent
    CUmemGenericAllocationHandle h = 0;     // (head only) the extent's handle
  };
  struct Region { CUdeviceptr base = 0; size_t va = 0, chunk = 0; std::vector<Chunk> chunks; };
  static constexpr size_t kChunk = size_t(1) << 30;    // largest grid chunk of a region
  int dev = 0;
  size_t gran = 0;
  uint32_t S = 0, MB = 0;
  uint64_t va_budget = 0, va_used = 0, mapped = 0, cached = 0;  // cached: mapped, 0 refs
  uint64_t n_map = 0, n_unmap = 0, ns_map = 0, ns_unmap = 0, n_regions = 0;  // cost counters
  uint64_t n_create = 0, n_pool = 0;   // handles from the driver / from the process pool
  uint64_t adopted = 0;                // bytes mapped when this slab was adopted (slab cache)
  bool adopt_guard = false;            // adopted chunks not yet settled against the footprint bound
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
  // refcount grid of class b's region: a power of two >= one granule and >=
  // one bucket, 1/8..1/16 of the region, at most kChunk (uniform backing maps
  // whole runs of grid chunks as one extent, so the grid only bounds what an
  // uneven split strands)
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
  // a physical handle of `size` bytes: the process pool first (after freeing
  // whatever destroyed arrays left behind), else the driver; on the driver's
  // out-of-memory, wait for deferred teardown and empty the caches, then retry
  int new_handle(size_t size, CUmemGenericAllocationHandle *h);
  // map grid chunks [c0, c0 + n) of r (all unmapped) as one extent
  int map_run(Region &r, size_t c0, size_t n) {
    const uint64_t t0 = now_ns();
    const size_t bytes_ = n * r.chunk;
    Chunk &hd = r.chunks[c0];
    { int rc = new_handle(bytes_, &hd.h); if (rc) return rc; }
    const CUdeviceptr at = r.base + c0 * r.chunk;
    if (drv().map(at, bytes_, 0, hd.h, 0) != CUDA_SUCCESS) {
      give_or_release(bytes_, hd.h);
      hd.h = 0;
      return fail(GG_ENOMEM, "cuMemMap failed");
    }
    // access rights are granted in finalize_access(), one cuMemSetAccess per
    // contiguous run of extents mapped by the same operation (the call costs
    // about as much as the mapping itself)
    pending.push_back({&r, c0});
    hd.len = (uint32_t)n;
    for (size_t c = c0; c < c0 + n; ++c) {
      r.chunks[c].mapped = true;
      r.chunks[c].head = (uint32_t)c0;
      cached += r.chunk;                      // refs are added by the caller
    }
    mapped += bytes_;
    n_map += 1;
    ns_map += now_ns() - t0;
    static const bool batch = [] { const char *e = getenv("GG_BATCH_ACCESS"); return !e || e[0] != '0'; }();
    if (!batch) return finalize_access();
    return GG_OK;
  }
  void give_or_release(size_t size, CUmemGenericAllocationHandle h);
  // a mapped chunk about to gain a reference: un-doom its extent
  void revive(Region &r, size_t c) {
    Chunk &k = r.chunks[c];
    if (!k.doomed) return;
    const Chunk &hd = r.chunks[k.head];
    for (size_t i = k.head; i < k.head + hd.len; ++i) r.chunks[i].doomed = false;
    doomed_bytes -= hd.len * r.chunk;
  }
  void add_ref(Region &r, size_t c, uint32_t n) {
    Chunk &k = r.chunks[c];
    revive(r, c);
    if (!k.refs) cached -= r.chunk;
    k.refs += n;
  }
  int map_chunk(Region &r, size_t c) {
    if (r.chunks[c].mapped) return GG_OK;
    return map_run(r, c, 1);
  }
  std::vector<std::pair<Region *, size_t>> pending;   // extents mapped, access not granted yet
  // grant read/write access to every extent mapped since the last call; must
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
      size_t end = pending[i].second + r->chunks[pending[i].second].len;
      size_t j = i + 1;
      while (j < pending.size() && pending[j].first == r && pending[j].second == end) {
        end += r->chunks[pending[j].second].len;
        ++j;
      }
      const CUdeviceptr at = r->base + pending[i].second * r->chunk;
      if (drv().set_access(at, (end - pending[i].second) * r->chunk, &acc, 1) != CUDA_SUCCESS && !rc)
        rc = fail(GG_ENOMEM, "cuMemSetAccess failed");
      i = j;
    }
    pending.clear();
    ns_map += now_ns() - t0;
    return rc;
  }
  bool extent_free(const Region &r, size_t head) const {
    const Chunk &hd = r.chunks[head];
    for (size_t c = head; c < head + hd.len; ++c)
      if (r.chunks[c].refs) return false;
    return true;
  }
  // unmap an extent without live buckets; its physical handle goes to the
  // process pool (released to the driver only when the pool is full)
  void unmap_extent(Region &r, size_t head) {
    const uint64_t t0 = now_ns();
    drv().unmap(r.base + head * r.chunk, r.chunks[head].len * r.chunk);
    unmapped(r, head);
    ns_unmap += now_ns() - t0;
  }
  // bookkeeping of an extent whose mapping is gone: handle to the pool
  void unmapped(Region &r, size_t head) {
    Chunk &hd = r.chunks[head];
    const size_t n = hd.len, bytes_ = n * r.chunk;
    give_or_release(bytes_, hd.h);
    if (hd.doomed) doomed_bytes -= bytes_;
    for (size_t c = head; c < head + n; ++c) {
      Chunk &k = r.chunks[c];
      k.mapped = k.doomed = false;
      k.len = 0;
      k.h = 0;
    }
    mapped -= bytes_;
    cached -= bytes_;
    n_unmap += 1;
  }
  // unmap a set of extents without live buckets, adjacent extents of a
  // region with ONE cuMemUnmap (the driver charges per call -- ~1-10 ms on
  // some boxes -- far more than per byte); an unmap the driver refuses over
  // several mappings is retried extent by extent
  void unmap_extents(std::vector<std::pair<Region *, size_t>> &v) {
    if (v.empty()) return;
    const uint64_t t0 = now_ns();
    std::sort(v.begin(), v.end());
    for (size_t i = 0; i < v.size();) {
      Region &r = *v[i].first;
      size_t end = v[i].second + r.chunks[v[i].second].len, j = i + 1;
      while (j < v.size() && v[j].first == &r && v[j].second == end) {
        end += r.chunks[v[j].second].len;
        ++j;
      }
      const size_t c0 = v[i].second;
      if (j - i > 1 && drv().unmap(r.base + c0 * r.chunk, (end - c0) * r.chunk) == CUDA_SUCCESS) {
        for (size_t k = i; k < j; ++k) unmapped(r, v[k].second);
      } else {
        for (size_t k = i; k < j; ++k) {
          drv().unmap(r.base + v[k].second * r.chunk, r.chunks[v[k].second].len * r.chunk);
          unmapped(r, v[k].second);
        }
      }
      i = j;
    }
    ns_unmap += now_ns() - t0;
  }
  // Asynchronous trim: extents that lose their last live bucket in a shrink
  // stay mapped until the work queued before the shrink completed (an event
  // on its stream, no device-wide synchronize); they are unmapped by the
  // next reap_doomed -- or taken back in place for free if a later operation
  // needs them first.
  std::vector<std::pair<Region *, size_t>> doomed;
  uint64_t doomed_bytes = 0;
  cudaEvent_t doom_ev = nullptr;
  template <typename F>
  void for_free_extents(Region &r, F f) {      // highest first
    for (size_t c = r.chunks.size(); c-- > 0;) {
      Chunk &k = r.chunks[c];
      if (k.mapped && k.head == c && extent_free(r, c) && !f(r, c)) return;
    }
  }
  int doom_to(uint64_t keep, cudaStream_t st) {
    finalize_access();
    auto pick = [&](Region &r, size_t head) {
      if (mapped - doomed_bytes <= keep) return false;
      Chunk &hd = r.chunks[head];
      if (hd.doomed) return true;
      for (size_t c = head; c < head + hd.len; ++c) r.chunks[c].doomed = true;
      doomed_bytes += hd.len * r.chunk;
      doomed.push_back({&r, head});
      return true;
    };
    for (int b = (int)MB - 1; b >= 0 && mapped - doomed_bytes > keep && cached; --b)
      if (small_off[b] == ~uint64_t(0)) for_free_extents(big[b], pick);
    if (mapped - doomed_bytes > keep) for_free_extents(small, pick);
    if (doomed.empty()) return GG_OK;
    if (!doom_ev) CUDA_TRY(cudaEventCreateWithFlags(&doom_ev, cudaEventDisableTiming));
    CUDA_TRY(cudaEventRecord(doom_ev, st));    // everything queued so far (incl. the shrink)
    return GG_OK;
  }
  // unmap the doomed extents once their event completed (wait = block on it)
  void reap_doomed(bool wait) {
    if (doomed.empty()) return;
    if (wait) cudaEventSynchronize(doom_ev);
    else if (cudaEventQuery(doom_ev) != cudaSuccess) return;
    std::vector<std::pair<Region *, size_t>> go;
    for (auto &d : doomed) {
      Chunk &hd = d.first->chunks[d.second];
      if (hd.doomed && hd.mapped && hd.head == d.second && extent_free(*d.first, d.second)) go.push_back(d);
    }
    unmap_extents(go);
    doomed.clear();
    doomed_bytes = 0;
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
      add_ref(*r, c, 1);
    }
    return GG_OK;
  }
  void drop(Region &r, size_t c) {
    Chunk &k = r.chunks[c];
    if (--k.refs == 0) cached += r.chunk;      // stays mapped until trimmed
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
  // back slots [s0, s1) of class b (region must exist); all-or-nothing.
  // Maximal runs of unmapped grid chunks are mapped as one extent each.
  int back_range(uint32_t b, uint32_t s0, uint32_t s1) {
    if (s1 <= s0) return GG_OK;
    Region &r = region(b);
    const uint64_t base = small_off[b] != ~uint64_t(0) ? small_off[b] : 0, bb = bytes[b];
    const size_t lo = (base + (uint64_t)s0 * bb) / r.chunk, hi = (base + (uint64_t)s1 * bb - 1) / r.chunk;
    for (size_t c = lo; c <= hi;) {
      if (r.chunks[c].mapped) { ++c; continue; }
      size_t e = c;
      while (e + 1 <= hi && !r.chunks[e + 1].mapped) ++e;
      int rc = map_run(r, c, e - c + 1);       // (a failure leaves earlier runs cached, refs 0)
      if (rc) return rc;
      c = e + 1;
    }
    for_range(b, s0, s1, [&](Region &rr, size_t c, uint32_t n) { add_ref(rr, c, n); });
    return GG_OK;
  }
  // map (without references) the unmapped grid chunks slots [s0, s1) of
  // class b overlap, maximal runs as one extent each but at most `cap` grid
  // chunks per extent (release granularity); best effort: a failure leaves
  // the rest to per-slot backing, which fails exactly the shard concerned
  void premap_range(uint32_t b, uint32_t s0, uint32_t s1, size_t cap) {
    if (s1 <= s0) return;
    Region &r = region(b);
    const uint64_t base = small_off[b] != ~uint64_t(0) ? small_off[b] : 0, bb = bytes[b];
    const size_t lo = (base + (uint64_t)s0 * bb) / r.chunk, hi = (base + (uint64_t)s1 * bb - 1) / r.chunk;
    for (size_t c = lo; c <= hi;) {
      if (r.chunks[c].mapped) { ++c; continue; }
      size_t e = c;
      while (e + 1 <= hi && e + 1 - c < cap && !r.chunks[e + 1].mapped) ++e;
      if (e == c) { ++c; continue; }              // a single chunk: per-slot backing maps it
      if (map_run(r, c, e - c + 1)) return;
      c = e + 1;
    }
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
  // unmap extents without live buckets, largest class first, until at most
  // `keep` bytes stay mapped (caller synchronised the work that used them)
  void trim_to(uint64_t keep) {
    finalize_access();
    reap_doomed(true);
    std::vector<std::pair<Region *, size_t>> sel;
    uint64_t left = mapped;
    auto go = [&](Region &r, size_t head) {
      if (left <= keep) return false;
      sel.push_back({&r, head});
      left -= r.chunks[head].len * r.chunk;
      return true;
    };
    for (int b = (int)MB - 1; b >= 0 && left > keep && cached; --b)
      if (small_off[b] == ~uint64_t(0)) for_free_extents(big[b], go);
    if (left > keep) for_free_extents(small, go);
    unmap_extents(sel);
  }
  // unmap every extent without live buckets (caller synchronised)
  void trim() { trim_to(0); }
  // the array is going away: unmap everything, physical handles to the
  // process pool while it has room (the caller synchronised the work)
  void destroy() {
    pending.clear();
    doomed.clear();
    doomed_bytes = 0;
    if (doom_ev) cudaEventDestroy(doom_ev), doom_ev = nullptr;
    auto go = [&](Region &r) {
      // runs of adjacent mapped extents: one cuMemUnmap each (per-extent
      // calls if the driver refuses the run), handles to the pool
      for (size_t c = 0; c < r.chunks.size();) {
        if (!(r.chunks[c].mapped && r.chunks[c].head == c)) { ++c; continue; }
        size_t e = c;
        while (e < r.chunks.size() && r.chunks[e].mapped && r.chunks[e].head == e) e += r.chunks[e].len;
        const bool one = e - c > r.chunks[c].len &&
                         drv().unmap(r.base + c * r.chunk, (e - c) * r.chunk) == CUDA_SUCCESS;
        for (size_t h = c; h < e; h += r.chunks[h].len) {
          if (!one) drv().unmap(r.base + h * r.chunk, r.chunks[h].len * r.chunk);
          give_or_release(r.chunks[h].len * r.chunk, r.chunks[h].h);
        }
        c = e;
      }
      if (r.base) drv().addr_free(r.base, r.va);
      r = Region();
    };
    go(small);
    for (auto &r : big) go(r);
    mapped = cached = va_used = 0;
  }
  // the same slab for a new array (slab cache): no live buckets, every
  // mapped chunk cached in place
  void adopt_reset() {
    pending.clear();
    doomed.clear();
    doomed_bytes = 0;
    auto go = [&](Region &r) {
      for (auto &k : r.chunks) { k.refs = 0; k.doomed = false; }
    };
    go(small);
    for (auto &r : big) go(r);
    cached = mapped;
    adopted = mapped;
    adopt_guard = mapped > 0;
    n_map = n_unmap = ns_map = ns_unmap = n_create = n_pool = 0;
  }
  // shape key of the slab cache: same S, classes, bucket bytes and budget
  bool same_shape(const Slab &o) const {
    return dev == o.dev && S == o.S && MB == o.MB && bytes == o.bytes && va_budget == o.va_budget &&
           gran == o.gran;
  }
};

// Slab cache: the slab of a destroyed array -- VA regions with their
// extents still mapped -- kept whole for the next array of the same shape
// (S, element size, first bucket size, max_buckets), which adopts it with
// every chunk cached in place: rebuilding an array (from_flat into a fresh
// GGArray, the paper's two-phase pattern) then costs no driver call at all.
// Its mapped bytes count against the process pool's cap; least recently
// cached slabs are evicted first (their handles go to the chunk pool).
struct SlabCache {
  std::mutex mu;
  std::vector<Slab *> slabs;                 // oldest first
  uint64_t hits = 0, offered = 0;
};

inline SlabCache &slab_cache() {
  static SlabCache c;
  return c;
}

inline void destroy_slabs(std::vector<Slab *> &v) {
  for (Slab *x : v) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != x->dev) cudaSetDevice(x->dev);
    x->destroy();
    if (cur != x->dev && cur >= 0) cudaSetDevice(cur);
    delete x;
  }
  v.clear();
}

// drop every cached slab of `dev` (-1: all devices)
inline void slab_cache_evict(int dev) {
  std::vector<Slab *> out;
  {
    SlabCache &C = slab_cache();
    std::lock_guard<std::mutex> g(C.mu);
    ChunkPool &P = chunk_pool();
    std::lock_guard<std::mutex> g2(P.mu);
    for (size_t i = 0; i < C.slabs.size();) {
      if (dev < 0 || C.slabs[i]->dev == dev) {
        P.slab_bytes[C.slabs[i]->dev] -= C.slabs[i]->mapped;
        out.push_back(C.slabs[i]);
        C.slabs.erase(C.slabs.begin() + i);
      } else {
        ++i;
      }
    }
  }
  destroy_slabs(out);
}

// keep `sl` (moved in) for a later array of the same shape; false = not
// kept (the caller destroys it)
inline bool slab_offer(Slab &sl) {
  if (!sl.mapped || sl.dev < 0 || sl.dev >= 64) return false;
  static const bool on = [] { const char *e = getenv("GG_SLAB_CACHE"); return !e || e[0] != '0'; }();
  if (!on) return false;
  std::vector<Slab *> out;
  bool kept = false;
  {
    SlabCache &C = slab_cache();
    std::lock_guard<std::mutex> g(C.mu);
    ChunkPool &P = chunk_pool();
    std::lock_guard<std::mutex> g2(P.mu);
    const int d = sl.dev;
    const uint64_t cap = P.cap(d);
    if (sl.mapped <= cap) {
      // make room: oldest cached slabs of this device first, then pooled handles
      for (size_t i = 0; i < C.slabs.size() && P.bytes[d] + P.slab_bytes[d] + sl.mapped > cap;) {
        if (C.slabs[i]->dev == d) {
          P.slab_bytes[d] -= C.slabs[i]->mapped;
          out.push_back(C.slabs[i]);
          C.slabs.erase(C.slabs.begin() + i);
        } else {
          ++i;
        }
      }
      while (!P.free[d].empty() && P.bytes[d] + P.slab_bytes[d] + sl.mapped > cap) {
        drv().release(P.free[d].back().second);
        P.bytes[d] -= P.free[d].back().first;
        P.free[d].pop_back();
      }
      if (P.bytes[d] + P.slab_bytes[d] + sl.mapped <= cap) {
        Slab *x = new Slab(std::move(sl));
        x->pending.clear();
        x->doomed.clear();
        x->doomed_bytes = 0;
        if (x->doom_ev) cudaEventDestroy(x->doom_ev), x->doom_ev = nullptr;
        C.slabs.push_back(x);
        P.slab_bytes[d] += x->mapped;
        ++C.offered;
        kept = true;
      }
    }
  }
  destroy_slabs(out);                        // evicted slabs' handles -> the chunk pool
  return kept;
}

// replace `sl` (freshly initialised, nothing mapped) by a cached slab of the
// same shape, if any (most recent first)
inline bool slab_adopt(Slab &sl) {
  Slab *x = nullptr;
  {
    SlabCache &C = slab_cache();
    std::lock_guard<std::mutex> g(C.mu);
    for (size_t i = C.slabs.size(); i-- > 0;)
      if (C.slabs[i]->same_shape(sl)) {
        x = C.slabs[i];
        C.slabs.erase(C.slabs.begin() + i);
        ++C.hits;
        break;
      }
    if (x) {
      ChunkPool &P = chunk_pool();
      std::lock_guard<std::mutex> g2(P.mu);
      P.slab_bytes[x->dev] -= x->mapped;
    }
  }
  if (!x) return false;
  sl.destroy();                              // the fresh slab's (empty) regions
  sl = std::move(*x);
  delete x;
  sl.adopt_reset();
  return true;
}

inline void Slab::give_or_release(size_t size, CUmemGenericAllocationHandle h) {
  if (!chunk_pool().give(dev, size, h)) drv().release(h);
}

inline int Slab::new_handle(size_t size, CUmemGenericAllocationHandle *h) {
  if (chunk_pool().take(dev, size, h)) { ++n_pool; return GG_OK; }
  reclaim(false);
  if (chunk_pool().take(dev, size, h)) { ++n_pool; return GG_OK; }
  CUmemAllocationProp prop = props();
  CUresult r = drv().create(h, size, &prop, 0);
  if (r == CUDA_ERROR_OUT_OF_MEMORY) {       // free what the process caches, then retry once
    reclaim(true);
    if (chunk_pool().take(dev, size, h)) { ++n_pool; return GG_OK; }
    slab_cache_evict(dev);
    if (chunk_pool().take(dev, size, h)) { ++n_pool; return GG_OK; }
    chunk_pool().trim(dev);
    r = drv().create(h, size, &prop, 0);
  }
  if (r != CUDA_SUCCESS) return fail(GG_ENOMEM, "cuMemCreate failed (device memory exhausted)");
  ++n_create;
  return GG_OK;
}

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

// What a destroyed array leaves behind, freed once an event recorded behind
// the array's last queued work completes (gg_destroy costs an event record,
// not a device-wide synchronize).  Its slab chunks go to the process pool.
struct Grave {
  int dev = 0;
  cudaEvent_t ev = nullptr;           // nullptr: nothing queued any more
  Slab slab;
  Uploader up;
  void *dmem = nullptr;               // cudaMallocAsync'd metadata block
  char *h_scratch = nullptr;          // pinned
  uint64_t *h_lanes = nullptr;        // pinned
  char *h_view = nullptr;             // pinned
  void *lanes_dmem = nullptr;         // cudaMallocAsync'd lanes scratch
  cudaEvent_t lanes_ev = nullptr;
  cudaEvent_t ord_ev = nullptr;
  void free_all() {
    if (!slab_offer(slab)) slab.destroy();   // kept whole for the next same-shape array
    up.destroy();
    if (h_scratch) cudaFreeHost(h_scratch);
    if (h_lanes) cudaFreeHost(h_lanes);
    if (h_view) cudaFreeHost(h_view);
    if (lanes_dmem) cudaFreeAsync(lanes_dmem, 0);
    if (lanes_ev) cudaEventDestroy(lanes_ev);
    if (dmem) cudaFreeAsync(dmem, 0);
    if (ord_ev) cudaEventDestroy(ord_ev);
    if (ev) cudaEventDestroy(ev);
  }
};

struct Reclaimer {
  std::mutex mu;
  std::vector<Grave *> graves;
  uint64_t buried = 0, freed = 0;
};

inline Reclaimer &reclaimer() {
  static Reclaimer r;
  return r;
}

inline void bury(Grave *g) {
  Reclaimer &R = reclaimer();
  std::lock_guard<std::mutex> l(R.mu);
  R.graves.push_back(g);
  ++R.buried;
}

inline void reclaim(bool wait) {
  Reclaimer &R = reclaimer();
  std::vector<Grave *> ready;
  {
    std::lock_guard<std::mutex> l(R.mu);
    if (R.graves.empty()) return;
    for (size_t i = 0; i < R.graves.size();) {
      Grave *g = R.graves[i];
      bool done = !g->ev;
      if (!done) {
        int cur = -1;
        cudaGetDevice(&cur);
        if (cur != g->dev) cudaSetDevice(g->dev);
        done = wait ? cudaEventSynchronize(g->ev) == cudaSuccess : cudaEventQuery(g->ev) == cudaSuccess;
        if (cur != g->dev && cur >= 0) cudaSetDevice(cur);
      }
      if (done) {
        ready.push_back(g);
        R.graves[i] = R.graves.back();
        R.graves.pop_back();
      } else {
        ++i;
      }
    }
    R.freed += ready.size();
  }
  for (Grave *g : ready) {
    int cur = -1;
    cudaGetDevice(&cur);
    if (cur != g->dev) cudaSetDevice(g->dev);
    g->free_all();
    if (cur != g->dev && cur >= 0) cudaSetDevice(cur);
    delete g;
  }
}

}  // namespace gg

#endif  // GG_HOST_CUH
