/*
 * ggarray.h -- C ABI of the B200-native GGArray (arXiv 2209.00103).
 *
 * A GGArray is S LFVectors ("shards"); shard s stores its elements in
 * power-of-two buckets, bucket b holding fb*2^b elements, allocated on the
 * device (CAS once-flag) in a per-class slab -- bucket (s, b) sits in slot s of
 * class b's CUDA-VMM region -- and never moved.  Physical memory is mapped
 * in refcounted chunks as buckets appear and unmapped when a shrink empties
 * them.  A committed exclusive prefix over the shard sizes is the global
 * directory.
 *
 * This header is the drop-in boundary.  The reference has no FFI: its
 * boundary is the Python class API of growarray.GrowableArray /
 * ShardVector / baselines.  Each entry point below names the reference
 * member it replaces (paths relative to /root/reference/pkg/src/growarray).
 * Pointers named d_* are device pointers, h_* host pointers; `stream` is a
 * cudaStream_t (NULL = legacy default stream).  No torch types cross the ABI.
 *
 * Return codes map to the reference's Python exceptions (errors.py):
 *   GG_OK 0, GG_EVALUE 1 (ValueError), GG_ECAPACITY 2 (CapacityError),
 *   GG_EINDEX 3 (IndexError), GG_ENOMEM 4 (MemoryError), GG_ECUDA 5,
 *   GG_EUNPUBLISHED 6 (RuntimeError: bucket unpublished), GG_EPARTIAL 7
 *   (some shards failed: per-shard codes in h_status -> ShardInsertError).
 * gg_last_error() returns a message for the calling thread's last failure.
 */
#ifndef GGARRAY_H
#define GGARRAY_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  GG_OK = 0, GG_EVALUE = 1, GG_ECAPACITY = 2, GG_EINDEX = 3, GG_ENOMEM = 4,
  GG_ECUDA = 5, GG_EUNPUBLISHED = 6, GG_EPARTIAL = 7
};

/* element types (arithmetic of the r/w passes; copies are byte-exact) */
enum {
  GG_I8 = 0, GG_U8 = 1, GG_I16 = 2, GG_U16 = 3, GG_I32 = 4, GG_U32 = 5,
  GG_I64 = 6, GG_U64 = 7, GG_F16 = 8, GG_F32 = 9, GG_F64 = 10
};

/* r/w traversal modes */
enum { GG_RW_PER_SHARD = 0, GG_RW_GLOBAL = 1, GG_RW_FUSED = 2 };

/* static-array insertion algorithms (paper section 3-B) */
enum { GG_ALGO_ATOMIC = 0, GG_ALGO_WARP = 1, GG_ALGO_BLOCK = 2, GG_ALGO_BATCH = 3 };

typedef struct gg_array gg_array;

/* Allocator hook: called on the host, in shard then bucket order, once per
 * bucket an operation is about to allocate; nonzero = allocation failure.
 * Replaces the `allocator` callable of ShardVector (bucket_vector.py:130-134,
 * 194-201) for counting and failure injection; storage always comes from
 * the device slabs. */
typedef int (*gg_alloc_hook)(void *ctx, uint32_t shard, uint32_t bucket, uint64_t elems);

const char *gg_last_error(void);
int gg_version(void);

/* Per-device library initialisation (CUDA context + the library's kernel
 * image), once per process; gg_create calls it.  Exposed so a host can pay
 * it up front.  No reference counterpart (the reference has no device). */
int gg_init(int device);
/* number of kernels this library has launched (process-wide counter) */
uint64_t gg_kernel_launches(void);

/* GrowableArray(shards, first_bucket_size, dtype, max_buckets, allocator)
 * sharded_array.py:85-100, bucket_vector.py:84-93,124-137.
 * arena_va_bytes = virtual-address budget of the bucket slabs (0 = 16 TiB;
 * class regions are reserved lazily, S * bucket bytes each).  max_buckets
 * <= 64. */
int gg_create(int device, uint32_t shards, uint32_t first_bucket_size, uint32_t dtype,
              uint32_t max_buckets, uint64_t arena_va_bytes, gg_array **out);
int gg_destroy(gg_array *a);
int gg_set_alloc_hook(gg_array *a, gg_alloc_hook hook, void *ctx);
/* Cap on live bucket bytes (failure injection: allocations past it fail
 * with MemoryError, like a failing allocator). 0 = no cap. */
int gg_set_arena_limit(gg_array *a, uint64_t bytes);

/* insert_parallel / push_back_batch (sharded_array.py:190-211,
 * bucket_vector.py:216-247): shard s appends d_values[h_offsets[s] ..
 * h_offsets[s+1]) in argument order.  h_starts == NULL: each non-empty shard
 * reserves its range with one device atomicAdd on its size; otherwise the
 * ranges were reserved earlier (ShardVector.size_counter.fetch_add) and only
 * allocation + write happen.  h_status[S] (may be NULL) receives per-shard
 * codes; a failing shard keeps its reservation, as in the reference.  Does
 * not commit. */
int gg_insert(gg_array *a, const void *d_values, const uint64_t *h_offsets,
              const uint64_t *h_starts, int32_t *h_status, void *stream);
/* flags of the _ex variants: GG_F_COMMIT commits (prefix rebuild) in the same
 * launch when no shard fails -- insert_parallel's insert-then-commit
 * (sharded_array.py:207-211); GG_F_UNFUSED forces the separate
 * reserve / copy kernels.  By default reservation, bucket allocation and the
 * copy run as ONE persistent launch. */
enum { GG_F_COMMIT = 1, GG_F_UNFUSED = 2 };
int gg_insert_ex(gg_array *a, const void *d_values, const uint64_t *h_offsets,
                 const uint64_t *h_starts, uint32_t flags, int32_t *h_status, void *stream);
/* gg_insert_ex that also returns each shard's reservation start in
 * h_reserved[S] (may be NULL): the ReservedRange push_back_batch returns
 * (bucket_vector.py:229-232), read under the handle's lock so concurrent
 * callers on one shard get the ranges they actually reserved. */
int gg_insert_ex2(gg_array *a, const void *d_values, const uint64_t *h_offsets,
                  const uint64_t *h_starts, uint32_t flags, int32_t *h_status, uint64_t *h_reserved,
                  void *stream);
int gg_insert_duplicate_ex(gg_array *a, uint32_t flags, int32_t *h_status, void *stream);
/* bench_cli.py:298-307 _insert_duplicate: every shard appends a copy of its
 * committed contents, read straight from its buckets (no snapshot). */
int gg_insert_duplicate(gg_array *a, int32_t *h_status, void *stream);
/* Paper Alg. 1 with per-lane counts (insert_index.py:84-143 LanePlan /
 * scan_reserve semantics): lanes [h_lane_offsets[s], h_lane_offsets[s+1])
 * belong to shard s; lane j appends its first d_counts[j] <= values_per_lane
 * values d_values[j*values_per_lane ...] (values_per_lane = 1, counts in
 * {0,1} is the paper's predicated push_back).  Shard s's batch lands in lane
 * order.  Pass 1 sums the counts per shard (CTA per shard) so the host maps
 * the slabs exactly; pass 2 reserves with ONE atomicAdd per shard, allocates
 * the buckets, block-scans the counts and scatters. */
int gg_insert_lanes(gg_array *a, const void *d_values, const uint32_t *d_counts,
                    const uint64_t *h_lane_offsets, uint64_t values_per_lane,
                    int32_t *h_status, void *stream);
/* commit (sharded_array.py:213-222): prefix = exclusive_scan(sizes)+[total] */
int gg_commit(gg_array *a, void *stream);
/* grow / reserve (sharded_array.py:224-240, bucket_vector.py:249-257):
 * shard by shard, allocate the minimal bucket prefix covering
 * h_min_capacity[s]; stops at the first failing shard (*h_failed_shard). */
int gg_reserve(gg_array *a, const uint64_t *h_min_capacity, int64_t *h_failed_shard,
               void *stream);
/* ShardVector.new_bucket (bucket_vector.py:170-205): *h_won = 1 iff this
 * call allocated bucket b of shard s. */
int gg_new_bucket(gg_array *a, uint32_t shard, uint32_t bucket, int32_t *h_won, void *stream);
/* AtomicCounter.fetch_add on a shard's size (insert_index.py:52-58) */
int gg_fetch_add(gg_array *a, uint32_t shard, uint64_t count, uint64_t *h_prev, void *stream);
/* shrink (extension, no reference semantics): size[s] = h_new_sizes[s] <=
 * size[s]; buckets b >= min_buckets_for(new size) are released.  Slab chunks
 * left without a live bucket stay mapped ("cached", reused in place when the
 * buckets come back) except that, largest class first, they are unmapped
 * until at most keep_mapped_bytes remain mapped (0 = unmap them all,
 * UINT64_MAX = keep them all); unmapping waits for the device.  The Python
 * layer's default keeps the footprint <= 2x the needed bytes.
 * gg_shrink = gg_shrink_ex(.., 0, ..).  Commits. */
int gg_shrink_ex(gg_array *a, const uint64_t *h_new_sizes, uint64_t keep_mapped_bytes,
                 void *stream);
int gg_shrink(gg_array *a, const uint64_t *h_new_sizes, void *stream);
/* unmap every cached chunk (waits for the device) */
int gg_trim(gg_array *a);

/* Device-side appends from user kernels (include/ggarray_device.cuh, paper
 * Alg. 1/2).  gg_device_view_get backs the slots of every bucket shard s
 * needs to reach h_max_sizes[s] elements (NULL = no headroom: appends only
 * into published buckets) and copies the device tables' view (a
 * gg::gg_device_view, view_bytes = sizeof) to h_view for passing to a kernel
 * by value; gg_device_view_sync waits for `stream`, refreshes the host
 * mirrors from the device (sizes, capacities, flags), unmaps the headroom no
 * bucket took and reports per-shard failures (GG_EPARTIAL).  Neither
 * commits; one view at a time per array. */
uint64_t gg_device_view_bytes(void);
int gg_device_view_get(gg_array *a, const uint64_t *h_max_sizes, void *h_view, uint64_t view_bytes);
int gg_device_view_sync(gg_array *a, int32_t *h_status, void *stream);
/* Example user kernel of that API: block b of a `grid`-block launch (0 =
 * auto) appends d_vals[i] for every i of its slices with d_pred[i] != 0 to
 * shard b % S; mode 0 = warp_push_back (one atomicAdd per warp), 1 =
 * block_push_back (block scan, one atomicAdd per block). */
int gg_push_if(gg_array *a, const void *d_vals, const uint8_t *d_pred, uint64_t n, int32_t mode,
               uint32_t grid, int32_t *h_status, void *stream);

/* for_each_shard(+c) x passes (sharded_array.py:165-186, bench_cli.py:
 * 180-183, 323-366).  h_addend points to one element of the array dtype.
 * mode GG_RW_PER_SHARD walks shard segments (rw_b), GG_RW_GLOBAL resolves
 * every global index through the directory (rw_g), GG_RW_FUSED applies all
 * passes in one sweep (reported separately). */
int gg_rw_add(gg_array *a, const void *h_addend, uint32_t passes, int32_t mode, void *stream);
/* flatten (sharded_array.py:244-257): d_out[prefix[s]+i] = shard_s[i]. */
int gg_flatten(gg_array *a, void *d_out, void *stream);
/* the committed elements with global index in [lo, hi) to d_out[0 .. hi-lo)
 * (a slice of flatten(): pieces of a rebalance, bounded staging) */
int gg_flatten_range(gg_array *a, uint64_t lo, uint64_t hi, void *d_out, void *stream);
/* get_global / set_global for index arrays (sharded_array.py:139-158) */
int gg_gather(gg_array *a, const int64_t *d_idx, uint64_t n, void *d_out, void *stream);
int gg_scatter(gg_array *a, const int64_t *d_idx, uint64_t n, const void *d_vals, void *stream);
/* gg_gather with the bounds check of get_global (sharded_array.py:152-155:
 * IndexError outside the committed size) fused into the gather: returns
 * GG_EINDEX if any index is outside [0, committed size) (d_out then holds
 * no meaningful values); synchronizes the stream to read the check back */
int gg_gather_checked(gg_array *a, const int64_t *d_idx, uint64_t n, void *d_out, void *stream);
/* gg_scatter with set_global's bounds check (sharded_array.py:156-158): a
 * bounds pass over the indices, then the scatter, which writes nothing if
 * any index is outside [0, committed size) (GG_EINDEX, no partial update);
 * synchronizes the stream to read the check back */
int gg_scatter_checked(gg_array *a, const int64_t *d_idx, uint64_t n, const void *d_vals, void *stream);
/* single-element ShardVector.get / set (bucket_vector.py:259-277) */
int gg_get(gg_array *a, uint32_t shard, uint64_t i, void *h_out, void *stream);
int gg_set(gg_array *a, uint32_t shard, uint64_t i, const void *h_val, void *stream);

/* CUDA-graph capture support: while on != 0, per-op host->device uploads use
 * pinned buffers owned by the captured graph (released by
 * gg_capture_release) and no call synchronises, so a stream capture of any
 * op sequence is legal.  A captured sequence that starts and ends in the same
 * state (e.g. reset + inserts) may be replayed; the host mirrors keep the
 * state after the captured sequence. */
int gg_capture_mode(gg_array *a, int32_t on);
/* on = 2: as 1, and the deferred metadata pass (gg_set_defer) stays enabled
 * under capture -- the caller must gg_flush() before the capture ends (the
 * Python GrowableArray.capture helper does). */
/* launch a deferred metadata pass / grow now, if one is pending (stream-ordered) */
int gg_flush(gg_array *a);
/* end of a capture-mode-2 sequence, called INSIDE the capture: flushes what
 * is deferred and restores the size/prefix buffer parity the capture began
 * with, so the graph can be replayed. */
int gg_capture_end(gg_array *a, void *stream);
/* Metadata pass inside the planned walk (default on): one launch per append,
 * double-buffered size / prefix, and uniform grows deferred into the next
 * append.  Process-wide; for A/B measurements. */
int gg_set_fuse(int32_t on);
int gg_capture_release(gg_array *a);
/* Tuning of the streaming kernels (sweeps): unroll U in {1,2,4,8} = 16 B
 * vectors per thread per tile (tile = 256 threads x U vectors); -1 = the
 * built-in choice.  ls / tile_bytes / threads are accepted and ignored
 * (kept for ABI stability).  Process-wide. */
int gg_set_tuning(int32_t ls, int32_t unroll, uint32_t tile_bytes, uint32_t threads);
/* Programmatic dependent launch of the library's kernels (default on): a
 * kernel may start while its stream predecessor drains.  Process-wide; for
 * A/B measurements. */
int gg_set_pdl(int32_t on);
/* Deferred metadata (default on): the metadata pass of an append issued
 * eagerly is launched with the next device-touching call, fused into the
 * next grow when that comes first (one launch instead of two).  Host-only
 * queries (summary, host state, memory stats) see the up-to-date host
 * mirrors either way.  Process-wide; for A/B measurements. */
int gg_set_defer(int32_t on);
/* Batched backing of new bucket classes (default 1): append plans, lanes
 * inserts and device views back each class in runs of consecutive shards
 * (one refcount pass per run).  0 = one slab call per bucket; 2 = every run
 * treated as unbackable, so the per-shard fallback (exact failure semantics)
 * runs -- a test hook.  Process-wide. */
int gg_set_batch_backing(int32_t mode);
/* committed size, total (reserved) size, total capacity -- host mirrors */
int gg_summary(gg_array *a, uint64_t *h_out3);

/* Host views of the state (mirrors kept exact by the planner). */
int gg_info(gg_array *a, uint32_t *h_out4 /* shards, fb, dtype, max_buckets */);
int gg_host_state(gg_array *a, uint64_t *h_sizes, uint64_t *h_caps, uint64_t *h_flags,
                  uint64_t *h_prefix, uint64_t *h_ops);
/* Same quantities read back from DEVICE memory (synchronises `stream`). */
int gg_device_state(gg_array *a, uint64_t *h_sizes, uint64_t *h_caps, uint64_t *h_flags,
                    uint64_t *h_prefix, uint64_t *h_ops, void *stream);
/* committed directory prefix[S+1] (u64) copied to device memory d_out,
 * stream-ordered (capture-safe; the global-index map of the array) */
int gg_prefix_copy(gg_array *a, void *d_out, void *stream);
/* bucket base device pointers [S*max_buckets] (0 = unallocated); syncs */
int gg_bucket_ptrs(gg_array *a, uint64_t *h_ptrs, void *stream);
/* footprint: [0]=capacity bytes (elements of allocated buckets x element
 * size, the reference's capacity), [1]=mapped slab bytes (physical),
 * [2]=live bucket bytes (16 B rounded), [3]=needed bytes (sum of sizes),
 * [4]=device alloc calls, [5]=cached bytes (mapped chunks without a live
 * bucket), [6]=bytes a shrink released that are still mapped until the work
 * queued before it completes (see gg_settle) */
int gg_mem_stats(gg_array *a, uint64_t *h_out7, void *stream);
/* unmap the chunks earlier shrinks released, waiting (event) for the work
 * queued before them; after it mem_stats[1] is the settled footprint */
int gg_settle(gg_array *a);
/* slab mapping cost: [0]=mapped bytes, [1]=cached bytes, [2]=chunks mapped
 * (cumulative), [3]=chunks unmapped, [4]=ns in cuMemCreate/Map/SetAccess,
 * [5]=ns in cuMemUnmap/Release, [6]=class regions reserved, [7]=VA bytes,
 * [8]=physical handles created by the driver, [9]=handles taken from the
 * process pool, [10]=bytes pending an asynchronous unmap */
int gg_slab_stats(gg_array *a, uint64_t *h_out11);

/* Process-wide cache of physical slab chunks (per device and chunk size):
 * chunks of destroyed arrays and chunks a shrink / trim unmaps, reused by any
 * array before the driver is asked for new memory.  Bounded by GG_POOL_BYTES
 * (default: a quarter of the device's memory); emptied on a cuMemCreate
 * out-of-memory.  Besides loose handles it keeps whole slabs of destroyed
 * arrays (VA regions with their extents still mapped) for the next array of
 * the same shape, which adopts one with no driver call (GG_SLAB_CACHE=0
 * disables).  stats: [0]=cached handle bytes, [1]=handles, [2]=hits,
 * [3]=misses (process-wide), [4]=cap bytes (handles + slabs), [5]=destroyed
 * arrays whose memory is not freed yet (their queued work is still
 * running), [6]=handles the full pool refused (released to the driver),
 * [7]=mapped bytes of cached slabs, [8]=cached slabs, [9]=slab adoptions
 * (process-wide).  trim: wait for those, release everything to the driver. */
int gg_pool_stats(int device, uint64_t *h_out10);
int gg_pool_trim(int device);
/* Free what destroyed arrays left behind once their queued work completed
 * (gg_destroy records an event instead of synchronising the device);
 * wait != 0 blocks until all of it is freed. */
int gg_reclaim(int32_t wait);

/* ---- baselines (baselines.py) on raw device buffers ---- */
/* StaticArray/DoublingArray/ChunkTableArray.insert_batch (baselines.py:
 * 63-77, 143-157, 224-236): append d_vals[0..n) at *d_counter using `algo`
 * (ATOMIC: one atomicAdd per element; WARP: one per warp; BLOCK: one per
 * CTA after a block scan; BATCH: one reservation, argument order). Elements
 * landing at index >= capacity are dropped and counted in *d_counter. */
int gg_flat_insert(void *d_buf, uint64_t capacity, uint64_t *d_counter, const void *d_vals,
                   uint64_t n, uint32_t elem_bytes, int32_t algo, void *stream);
/* insert_batch with the reference's default semantics (one reservation,
 * argument order; baselines.py:59-72): the caller reserved [start, start+n)
 * on its host counter; the kernel copies d_vals there with 16 B vectors and
 * adds n to *d_counter (may be NULL).  CapacityError past the capacity. */
int gg_flat_append(void *d_buf, uint64_t capacity, uint64_t *d_counter, uint64_t start,
                   const void *d_vals, uint64_t n, uint32_t elem_bytes, void *stream);
/* contiguous +c passes over d_buf[0..n) (static r/w, flattened r/w) */
int gg_flat_add(void *d_buf, uint64_t n, uint32_t dtype, const void *h_addend,
                uint32_t passes, int32_t fused, void *stream);
/* stream-ordered device buffers (semi-static DoublingArray.resize,
 * baselines.py:127-141: new buffer + D2D copy + free) */
int gg_buf_alloc(uint64_t bytes, void *stream, void **d_out);
int gg_buf_free(void *d_ptr, void *stream);
int gg_buf_copy(void *d_dst, const void *d_src, uint64_t bytes, void *stream);
/* ---- multi-GPU gather: the root allocates the global flat
 * buffer with gg_ipc_alloc, publishes its handle (gg_ipc_get_handle, 64 B),
 * every other rank maps it with gg_ipc_open and runs gg_flatten straight
 * into it at its global base -- the flatten kernel's stores cross NVLink /
 * NVSwitch, so the gather is fused into the flatten (no staging copy, no
 * NCCL call on the data path). */
int gg_ipc_alloc(uint64_t bytes, void **d_out);
int gg_ipc_free(void *d_ptr);
int gg_ipc_handle_bytes(void);
int gg_ipc_get_handle(void *d_ptr, void *h_handle);
int gg_ipc_open(const void *h_handle, void **d_out);
int gg_ipc_close(void *d_ptr);
/* memMap baseline (paper section 3-A, ChunkTableArray analog): one VA
 * reservation, physical 2 MiB granules appended with cuMemCreate/cuMemMap. */
typedef struct gg_vmm gg_vmm;
int gg_vmm_create(int device, uint64_t va_bytes, gg_vmm **out);
int gg_vmm_ensure(gg_vmm *v, uint64_t bytes);
int gg_vmm_info(gg_vmm *v, uint64_t *h_base, uint64_t *h_mapped, uint64_t *h_granule);
int gg_vmm_destroy(gg_vmm *v);

/* device properties the host layer sizes grids with */
int gg_device_sms(int device, int32_t *h_sms);

#ifdef __cplusplus
}
#endif
#endif /* GGARRAY_H */
