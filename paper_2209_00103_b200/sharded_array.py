"""GGArray drop-in: ``GrowableArray`` with the reference's API
(sharded_array.py:75-288), backed by one ``gg_array`` handle per GPU.

Every operation is a stream-ordered call into the C ABI (include/ggarray.h):
a kernel boundary is the epoch boundary of the reference, so
``commit`` is the device prefix-scan kernel and readers after it see every
earlier write.  ``workers=`` arguments are accepted for compatibility; the
concurrency lives inside the kernels (CTA = actor).
"""

from __future__ import annotations

import contextlib
import ctypes as C
import os
import threading
import weakref
from bisect import bisect_right
from typing import Callable, Sequence

import numpy as np

from . import _lib as L
from .bucket_vector import DEFAULT_FIRST_BUCKET_SIZE, MAX_BUCKETS, ShardVector
from .errors import CapacityError, ShardInsertError, TraversalError
from .insert_index import AtomicReserver

__all__ = ["GrowableArray", "split_batches", "DEFAULT_SHARDS", "RW_MODES"]

DEFAULT_SHARDS = 32
RW_MODES = {"per_shard": L.GG_RW_PER_SHARD, "global": L.GG_RW_GLOBAL, "fused": L.GG_RW_FUSED}

_INT_OF_SIZE = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}
# GG_UNFUSED=1 forces the separate reserve / copy / commit kernels (A/B runs)
_EXTRA_FLAGS = L.GG_F_UNFUSED if os.environ.get("GG_UNFUSED") == "1" else 0


def split_batches(values, shards: int) -> list:
    """ceil(n/S)-element contiguous chunks, chunk c for shard c (sharded_array.py:29-38)."""
    vals = values if hasattr(values, "__len__") and not isinstance(values, list) else np.asarray(values)
    n = len(vals)
    chunk = -(-n // shards) if n else 0
    return [vals[c * chunk:(c + 1) * chunk] for c in range(shards)]


def split_offsets(n: int, shards: int) -> np.ndarray:
    chunk = -(-n // shards) if n else 0
    return np.minimum(np.arange(shards + 1, dtype=np.uint64) * np.uint64(chunk), np.uint64(n))


class _ShardList:
    """``GrowableArray.shards``: a read-only sequence of per-shard views."""

    __slots__ = ("_arr",)

    def __init__(self, arr):
        self._arr = arr

    def __len__(self) -> int:
        return self._arr._S

    def __getitem__(self, s):
        if isinstance(s, slice):
            return [self[i] for i in range(*s.indices(len(self)))]
        s = int(s)
        n = len(self)
        if s < 0:
            s += n
        if not 0 <= s < n:
            raise IndexError(f"shard {s} outside [0, {n})")
        return ShardVector._bind(self._arr, s)

    def __iter__(self):
        return (ShardVector._bind(self._arr, s) for s in range(len(self)))


def _torch_dtype(dt: np.dtype):
    import torch
    return {np.dtype(np.int8): torch.int8, np.dtype(np.uint8): torch.uint8,
            np.dtype(np.int16): torch.int16, np.dtype(np.uint16): torch.uint16,
            np.dtype(np.int32): torch.int32, np.dtype(np.uint32): torch.uint32,
            np.dtype(np.int64): torch.int64, np.dtype(np.uint64): torch.uint64,
            np.dtype(np.float16): torch.float16, np.dtype(np.float32): torch.float32,
            np.dtype(np.float64): torch.float64}[np.dtype(dt)]


class GrowableArray:
    """S LFVectors in per-class device slabs plus the committed prefix directory."""

    def __init__(self, shards: int = DEFAULT_SHARDS,
                 first_bucket_size: int = DEFAULT_FIRST_BUCKET_SIZE, dtype=np.int64,
                 max_buckets: int = MAX_BUCKETS, allocator=None, device=None,
                 arena_va_bytes: int = 0):
        import torch
        if shards < 1:
            raise ValueError(f"shards must be >= 1, got {shards}")
        if not torch.cuda.is_available():
            raise RuntimeError("paper_2209_00103_b200.GrowableArray needs a CUDA device (B200)")
        self.dtype = np.dtype(dtype)
        if self.dtype not in L.DTYPE_CODES:
            raise ValueError(f"unsupported dtype {self.dtype}")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self._torch_dtype = _torch_dtype(self.dtype)
        self._int_np = np.dtype(_INT_OF_SIZE[self.dtype.itemsize])
        # dtype torch can alias through __cuda_array_interface__ (wide uints as ints)
        self._storage_dtype = (self._int_np if self.dtype.kind == "u" and self.dtype.itemsize > 1
                               else self.dtype)
        self._h = None
        h = C.c_void_p()
        with torch.cuda.device(self.device):
            L.check(L.lib.gg_create(self.device.index, shards, first_bucket_size,
                                    L.DTYPE_CODES[self.dtype], max_buckets, int(arena_va_bytes),
                                    C.byref(h)), "create")
        self._h = h
        self._S, self._fb, self._mb = shards, first_bucket_size, max_buckets
        self._hook_exc: dict = {}
        self._hook_fn = None
        self._allocator = allocator
        if allocator is not None:
            me = weakref.ref(self)          # no array <-> hook cycle

            def hook(_ctx, shard, _bucket, elems):
                try:
                    allocator(int(elems))
                    return 0
                except BaseException as exc:  # noqa: BLE001 -- becomes the shard's failure
                    arr = me()
                    if arr is not None:
                        arr._hook_exc[int(shard)] = exc
                    return 1
            self._hook_fn = L.HOOK(hook)
            L.lib.gg_set_alloc_hook(self._h, self._hook_fn, None)
        self._cache = self._tot = None
        self._ptrs = None
        self._summary = np.zeros(3, np.uint64)
        self._status = np.zeros(shards, np.int32)
        self._caps = np.zeros(shards, np.uint64)
        self._shrink_buf = np.zeros(shards, np.uint64)
        self._shrink_p = L.ptr(self._shrink_buf)
        self._status_p = L.ptr(self._status, C.c_int32)     # cached ctypes views (hot paths)
        self._caps_p = L.ptr(self._caps)
        self._failed = C.c_int64(-1)
        self._failed_p = C.byref(self._failed)
        self._dev_index = self.device.index
        # host-side state of concurrent callers (status buffers, hook
        # exceptions, mirror cache) is guarded by _mu; the C handle has its own
        self._mu = threading.RLock()
        self._gen = 0                     # bumped by every mutation (mirror cache validity)
        self._counters: dict = {}

    @property
    def shards(self) -> "_ShardList":
        """Per-shard views (``shards[s]`` -> ShardVector); built on access, so
        the array holds no reference to them (no cycle: a dropped array is
        freed at once, never later by the cyclic collector)."""
        return _ShardList(self)

    def _counter(self, s: int):
        c = self._counters.get(s)
        if c is None:
            from .bucket_vector import _SizeCounter
            c = self._counters.setdefault(s, _SizeCounter(self, s))
        return c

    # ------------------------------------------------------------ plumbing
    def _stream(self):
        return L.stream_handle(self._dev_index)

    def _dirty(self):
        self._gen += 1
        self._cache = self._tot = None
        self._ptrs = None

    def _totals(self):
        # (committed, total size, total capacity) from the host mirrors; cached
        # until the next mutating call (every one goes through _dirty / resets
        # _cache), so per-round `committed_size` reads cost no ctypes call
        tot = self._tot
        if tot is None:
            gen = self._gen
            o = np.zeros(3, np.uint64)
            L.lib.gg_summary(self._h, L.ptr(o))
            tot = (int(o[0]), int(o[1]), int(o[2]))
            if gen == self._gen:          # no mutation raced with the read
                self._tot = tot
        return tot

    def flush(self) -> None:
        """Launch the deferred metadata pass of the last append now (normally it
        rides on the next device-touching call)."""
        L.check(L.lib.gg_flush(self._h), "flush")

    def capture(self, fn, graph=None, stream=None):
        """Capture ``fn()`` (a sequence of operations on this array) into a CUDA
        graph and return it: capture mode with the deferred metadata pass kept
        on, flushed inside the capture before it ends, so the captured appends
        fuse their metadata into the following grows like eager issue does."""
        import torch
        g = graph if graph is not None else torch.cuda.CUDAGraph()
        L.check(L.lib.gg_capture_mode(self._h, 2), "capture_mode")
        try:
            kw = {} if stream is None else {"stream": stream}
            with torch.cuda.graph(g, **kw):
                fn()
                L.check(L.lib.gg_capture_end(self._h, self._stream()), "capture_end")
        finally:
            L.lib.gg_capture_mode(self._h, 0)
        return g

    @contextlib.contextmanager
    def capture_mode(self):
        """Make every operation inside the block legal under CUDA stream capture
        (``torch.cuda.graph``): per-op uploads use graph-owned pinned buffers
        and nothing synchronises.  A captured sequence that starts and ends in
        the same state (e.g. ``shrink(0)`` + inserts) can be replayed."""
        L.check(L.lib.gg_capture_mode(self._h, 1), "capture_mode")
        try:
            yield self
        finally:
            L.lib.gg_capture_mode(self._h, 0)

    def _host(self) -> dict:
        st = self._cache
        if st is None:
            gen = self._gen
            S = self._S
            st = {k: np.zeros(S + (k == "prefix"), np.uint64)
                  for k in ("sizes", "caps", "flags", "prefix", "ops")}
            L.check(L.lib.gg_host_state(self._h, *(L.ptr(st[k]) for k in
                                                   ("sizes", "caps", "flags", "prefix", "ops"))),
                    "host_state")
            if gen == self._gen:          # a mutation in between would make this stale
                self._cache = st
        return st

    def _bucket_ptrs(self) -> np.ndarray:
        if self._ptrs is None:
            p = np.zeros(self._S * self._mb, np.uint64)
            L.check(L.lib.gg_bucket_ptrs(self._h, L.ptr(p), self._stream()), "bucket_ptrs")
            self._ptrs = p.reshape(self._S, self._mb)
        return self._ptrs

    def _device_values(self, values):
        """Values cast like np.asarray(values, dtype) and resident on this device."""
        import torch
        if isinstance(values, torch.Tensor):
            if (values.dtype == self._torch_dtype and values.device == self.device and values.dim() == 1
                    and values.is_contiguous()):
                return values
            t = values.reshape(-1)
            if t.dtype != self._torch_dtype:
                t = t.to(self._torch_dtype)
            return t.to(self.device, non_blocking=True).contiguous()
        a = np.ascontiguousarray(np.asarray(values, dtype=self.dtype).reshape(-1))
        t = torch.from_numpy(a.view(self._int_np))
        return t.to(self.device).view(self._torch_dtype)

    def _to_numpy(self, t) -> np.ndarray:
        import torch
        ti = t.view(getattr(torch, self._int_np.name))
        if ti.numel() <= 65536:
            return ti.cpu().numpy().view(self.dtype)
        # large results land in pinned memory (torch's caching host allocator):
        # one DMA at full PCIe speed instead of a pageable staging copy
        host = torch.empty(ti.numel(), dtype=ti.dtype, pin_memory=True)
        host.copy_(ti, non_blocking=True)
        torch.cuda.current_stream(self.device).synchronize()
        return host.numpy().view(self.dtype)

    def _failure(self, s: int, code: int) -> BaseException:
        if code == L.GG_ECAPACITY:
            return CapacityError(f"shard {s}: range needs a bucket beyond the table of {self._mb}")
        if code == L.GG_ENOMEM:
            return self._hook_exc.pop(s, None) or MemoryError(f"shard {s}: no device memory for a bucket")
        return RuntimeError(f"shard {s}: status {code}")

    def _insert_device(self, vals, offsets: np.ndarray, starts: np.ndarray | None = None,
                       commit: bool = False, want_starts: bool = False):
        """gg_insert_ex2; returns {shard: exception} for failed shards (and, with
        ``want_starts``, each shard's reservation start).  With ``commit`` the
        prefix is rebuilt in the same launch iff nothing failed.  Status and
        hook exceptions are per call (concurrent callers do not share them)."""
        offsets = L.u64_array(offsets)
        status = np.zeros(self._S, np.int32)
        starts = None if starts is None else L.u64_array(starts)
        st = None if starts is None else L.ptr(starts)
        res = np.zeros(self._S, np.uint64) if want_starts else None
        flags = (L.GG_F_COMMIT if commit else 0) | _EXTRA_FLAGS
        with self._mu:
            self._hook_exc = {}
            rc = L.lib.gg_insert_ex2(self._h, C.c_void_p(vals.data_ptr() if vals.numel() else 0),
                                     L.ptr(offsets), st, flags, L.ptr(status, C.c_int32),
                                     None if res is None else L.ptr(res), self._stream())
            self._dirty()
            if rc not in (L.GG_OK, L.GG_EPARTIAL):
                L.check(rc, "insert")
            failures = {} if rc == L.GG_OK else {
                int(s): self._failure(int(s), int(status[s])) for s in np.flatnonzero(status)}
        return (failures, res) if want_starts else failures

    def _write_ranges(self, ranges: dict) -> None:
        """Write values at ranges reserved earlier through size_counter.fetch_add."""
        import torch
        S = self._S
        offsets = np.zeros(S + 1, np.uint64)
        starts = np.zeros(S, np.uint64)
        parts = []
        for s in range(S):
            if s in ranges:
                start, v = ranges[s]
                starts[s] = start
                offsets[s + 1] = offsets[s] + v.numel()
                parts.append(v)
            else:
                offsets[s + 1] = offsets[s]
        vals = torch.cat(parts) if parts else torch.empty(0, dtype=self._torch_dtype, device=self.device)
        failures = self._insert_device(vals, offsets, starts)
        if failures:
            raise next(iter(failures.values()))

    def _pack(self, batches):
        """One device buffer + CSR offsets from per-shard batches."""
        import torch
        if all(isinstance(b, torch.Tensor) and b.is_cuda for b in batches):
            ts = [self._device_values(b) for b in batches]
            counts = [t.numel() for t in ts]
            vals = torch.cat(ts) if ts else torch.empty(0, dtype=self._torch_dtype, device=self.device)
        else:
            dt = self.dtype
            arrs = [b if (type(b) is np.ndarray and b.dtype == dt and b.ndim == 1) else
                    np.asarray(b.cpu() if isinstance(b, torch.Tensor) else b, dtype=dt).reshape(-1)
                    for b in batches]
            counts = [len(a) for a in arrs]
            total = int(sum(counts))
            host = torch.empty(total, dtype=getattr(torch, self._int_np.name), pin_memory=total > 65536)
            if total:
                np.concatenate(arrs, out=host.numpy().view(self.dtype))
            vals = host.to(self.device, non_blocking=True).view(self._torch_dtype)
        offsets = np.zeros(self._S + 1, np.uint64)
        offsets[1:] = np.cumsum(np.asarray(counts, np.uint64))
        return vals, offsets

    def _reserve(self, caps: np.ndarray) -> None:
        if caps is self._caps:
            cp = self._caps_p
        else:
            caps = L.u64_array(caps)
            cp = L.ptr(caps)
        with self._mu:
            failed = self._failed
            failed.value = -1
            if self._hook_exc:
                self._hook_exc = {}
            rc = L.lib.gg_reserve(self._h, cp, self._failed_p, self._stream())
            self._dirty()
            if rc == L.GG_ENOMEM and failed.value in self._hook_exc:
                raise self._hook_exc.pop(failed.value)
            L.check(rc, "grow")

    def _get(self, s: int, i: int):
        if i < 0:
            raise IndexError(f"index {i} outside committed size")
        out = np.zeros(1, self.dtype)
        L.check(L.lib.gg_get(self._h, s, int(i), out.ctypes.data_as(C.c_void_p), self._stream()), "get")
        return out[0]

    def _set(self, s: int, i: int, value) -> None:
        if i < 0:
            raise IndexError(f"index {i} outside committed size")
        v = np.asarray(value).astype(self.dtype).reshape(1)
        L.check(L.lib.gg_set(self._h, s, int(i), v.ctypes.data_as(C.c_void_p), self._stream()), "set")

    # ------------------------------------------------------------ properties
    @property
    def shard_count(self) -> int:
        return self._S

    @property
    def first_bucket_size(self) -> int:
        return self._fb

    @property
    def max_buckets(self) -> int:
        return self._mb

    @property
    def prefix(self) -> list:
        return [int(x) for x in self._host()["prefix"]]

    @property
    def committed_size(self) -> int:
        return int(self._totals()[0])

    @property
    def total_size(self) -> int:
        return int(self._totals()[1])

    @property
    def total_capacity(self) -> int:
        return int(self._totals()[2])

    def __len__(self) -> int:
        return self.committed_size

    def committed_length(self, s: int) -> int:
        p = self._host()["prefix"]
        return int(p[s + 1] - p[s])

    # ------------------------------------------------------------ directory
    def locate_shard(self, g: int) -> tuple:
        n = self.committed_size
        if not 0 <= g < n:
            raise IndexError(f"global index {g} outside committed size {n}")
        p = self.prefix
        s = bisect_right(p, g) - 1
        return s, g - p[s]

    def locate_shard_many(self, indices) -> tuple:
        idx = np.asarray(indices, dtype=np.int64)
        n = self.committed_size
        if idx.size and (idx.min() < 0 or idx.max() >= n):
            raise IndexError(f"indices outside committed size {n}")
        p = self._host()["prefix"].astype(np.int64)
        s = np.searchsorted(p, idx, side="right") - 1
        return s, idx - p[s]

    def get_global(self, g: int):
        s, i = self.locate_shard(g)
        return self._get(s, i)

    def set_global(self, g: int, value) -> None:
        s, i = self.locate_shard(g)
        self._set(s, i, value)

    def get_many(self, indices):
        """Device gather of global indices (rw_g element path); returns a device tensor."""
        import torch
        idx = torch.as_tensor(np.asarray(indices, np.int64) if not isinstance(indices, torch.Tensor)
                              else indices, dtype=torch.int64).to(self.device).contiguous()
        out = torch.empty(idx.numel(), dtype=self._torch_dtype, device=self.device)
        # bounds check fused into the gather kernel (one flag word read back)
        rc = L.lib.gg_gather_checked(self._h, C.c_void_p(idx.data_ptr()), idx.numel(),
                                     C.c_void_p(out.data_ptr()), self._stream())
        if rc == L.GG_EINDEX:
            raise IndexError(f"indices outside committed size {self.committed_size}")
        L.check(rc, "gather")
        return out

    def set_many(self, indices, values) -> None:
        import torch
        idx = torch.as_tensor(np.asarray(indices, np.int64) if not isinstance(indices, torch.Tensor)
                              else indices, dtype=torch.int64).to(self.device).contiguous()
        vals = self._device_values(values)
        if vals.numel() != idx.numel():
            raise ValueError("indices and values differ in length")
        # bounds pass + scatter that writes nothing on a bad index (one flag read back)
        rc = L.lib.gg_scatter_checked(self._h, C.c_void_p(idx.data_ptr()), idx.numel(),
                                      C.c_void_p(vals.data_ptr()), self._stream())
        if rc == L.GG_EINDEX:
            raise IndexError(f"indices outside committed size {self.committed_size}")
        L.check(rc, "scatter")

    # ------------------------------------------------------------ traversal
    def for_each_shard(self, op: Callable, workers: int | None = 1) -> None:
        """Apply ``op`` to writable device views of every committed segment, in
        ascending order within each shard; failures are aggregated.  The views
        are :class:`~paper_2209_00103_b200.views.DeviceView` wrappers of torch
        CUDA tensors aliasing the buckets: numpy ufuncs with ``out=`` (the
        reference's ``np.add(v, 1, out=v)``) and torch methods (``v.add_(1)``)
        both run on the device."""
        from .views import DeviceView
        failures = {}
        for s, sh in enumerate(self.shards):
            n = self.committed_length(s)
            if not n:
                continue
            try:
                for view in sh._segment_tensors(n):
                    op(DeviceView(view))
            except BaseException as exc:  # noqa: BLE001 -- reference aggregates per shard
                failures[s] = exc
        if failures:
            raise TraversalError(failures)

    def rw_add(self, c, passes: int = 1, mode: str = "per_shard") -> None:
        """``passes`` x (every committed element += c) on the device.  ``per_shard``
        walks shard segments (rw_b), ``global`` resolves each global index through
        the directory (rw_g), ``fused`` applies all passes in one sweep."""
        addend = np.asarray(c).astype(self.dtype).reshape(1)
        L.check(L.lib.gg_rw_add(self._h, addend.ctypes.data_as(C.c_void_p), int(passes),
                                RW_MODES[mode], self._stream()), "rw_add")

    # ------------------------------------------------------------ growth
    def insert_parallel(self, per_shard_batches: Sequence, reserver=None,
                        workers: int | None = None) -> None:
        """One batch per shard, appended in argument order, then commit.  On
        failure raises ShardInsertError and withholds the commit."""
        if len(per_shard_batches) != self._S:
            raise ValueError(f"need {self._S} batches, got {len(per_shard_batches)}")
        if reserver is not None and not isinstance(reserver, AtomicReserver):
            failures, ok = self._insert_with_reserver(per_shard_batches, reserver)
        else:
            vals, offsets = self._pack(per_shard_batches)
            failures = self._insert_device(vals, offsets, commit=True)   # commit fused on success
            if not failures:
                self._cache = self._tot = None
                return
            counts = np.diff(offsets.astype(np.int64))
            ok = [s for s in range(self._S) if counts[s] and s not in failures]
        if failures:
            raise ShardInsertError(failures, ok)
        self.commit()

    def _insert_with_reserver(self, batches, reserver):
        failures, ok = {}, []
        lock = threading.Lock()

        def task(s, b):
            try:
                self.shards[s].push_back_batch(b, reserver)
                with lock:
                    ok.append(s)
            except BaseException as exc:  # noqa: BLE001
                with lock:
                    failures[s] = exc
        ths = [threading.Thread(target=task, args=(s, b)) for s, b in enumerate(batches) if len(b)]
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return failures, sorted(ok)

    def insert_csr(self, values, offsets, commit: bool = True) -> None:
        """Fast path: shard s appends values[offsets[s]:offsets[s+1]] (values may be a
        device tensor; no packing copy)."""
        vals = self._device_values(values)
        offsets = L.u64_array(offsets)
        if offsets.shape != (self._S + 1,) or int(offsets[-1]) != vals.numel():
            raise ValueError("offsets must have S+1 entries ending at len(values)")
        failures = self._insert_device(vals, offsets, commit=commit)
        if failures:
            counts = np.diff(offsets.astype(np.int64))
            raise ShardInsertError(failures, [s for s in range(self._S) if counts[s] and s not in failures])

    def insert_lanes(self, values, counts, lane_offsets, values_per_lane: int = 1,
                     commit: bool = True) -> None:
        """Paper Alg. 1: lanes [lane_offsets[s], lane_offsets[s+1]) belong to shard s;
        lane j appends its first counts[j] values values[j*values_per_lane ...]
        (counts above values_per_lane are clamped to it), in lane order.  The
        device reserves each shard's batch with a single atomicAdd on its size
        (insert_index.py:125-143), publishes the buckets and scatters with
        16 B vector stores; the host backs memory for the upper bound
        lanes x values_per_lane and learns the sizes asynchronously (no host
        round trip inside the call).  With an allocator hook, an arena limit
        or a possible capacity overflow the exact two-pass path runs."""
        import torch
        vals = self._device_values(values)
        cnt = torch.as_tensor(np.asarray(counts) if not isinstance(counts, torch.Tensor) else counts)
        cnt = cnt.to(device=self.device, dtype=torch.int32).contiguous()
        lo = L.u64_array(lane_offsets)
        if lo.shape != (self._S + 1,) or int(lo[-1]) != cnt.numel():
            raise ValueError("lane_offsets must have S+1 entries ending at len(counts)")
        if vals.numel() < cnt.numel() * values_per_lane:
            raise ValueError("values must hold values_per_lane slots per lane")
        status = np.zeros(self._S, np.int32)
        with self._mu:
            self._hook_exc = {}
            rc = L.lib.gg_insert_lanes(self._h, C.c_void_p(vals.data_ptr() if vals.numel() else 0),
                                       C.c_void_p(cnt.data_ptr() if cnt.numel() else 0), L.ptr(lo),
                                       int(values_per_lane), L.ptr(status, C.c_int32), self._stream())
            self._dirty()
            if rc not in (L.GG_OK, L.GG_EPARTIAL):
                L.check(rc, "insert_lanes")
            if rc == L.GG_EPARTIAL:
                failures = {int(s): self._failure(int(s), int(status[s])) for s in np.flatnonzero(status)}
                raise ShardInsertError(failures, [])
        if commit:
            self.commit()

    # ------------------------------------------------------------ device-side appends
    def device_view(self, max_sizes=None) -> bytes:
        """Raw ``gg::gg_device_view`` (include/ggarray_device.cuh) for a user kernel
        that appends with ``warp_push_back`` / ``block_push_back``.  The slots of
        every bucket shard s needs to reach ``max_sizes[s]`` elements (scalar or
        per shard; None = no headroom) are backed with memory first.  Call
        :meth:`device_sync` after the kernel."""
        n = int(L.lib.gg_device_view_bytes())
        buf = C.create_string_buffer(n)
        mx = None if max_sizes is None else L.u64_array(np.broadcast_to(np.asarray(max_sizes), (self._S,)))
        L.check(L.lib.gg_device_view_get(self._h, L.ptr(mx) if mx is not None else None, buf, n),
                "device_view")
        return buf.raw

    def device_sync(self) -> None:
        """Refresh the host mirrors after device-side appends; ShardInsertError on
        shards whose appends failed (reservations kept, as in the reference)."""
        status = np.zeros(self._S, np.int32)
        with self._mu:
            rc = L.lib.gg_device_view_sync(self._h, L.ptr(status, C.c_int32), self._stream())
            self._dirty()
        if rc == L.GG_EPARTIAL:
            failures = {int(s): MemoryError(f"shard {s}: no backed bucket slot for a device append")
                        for s in np.flatnonzero(status)}
            raise ShardInsertError(failures, [])
        L.check(rc, "device_sync")

    def push_if(self, values, pred, mode: str = "block", grid: int = 0, commit: bool = True) -> None:
        """Paper Alg. 1 from inside a kernel: block b appends values[i] for the
        i of its slices with pred[i] to shard b % S (block-scan or warp-ballot
        offsets, one atomicAdd per block / warp, on-demand bucket allocation)."""
        import torch
        vals = self._device_values(values)
        p = pred if isinstance(pred, torch.Tensor) else torch.from_numpy(np.asarray(pred))
        p = p.to(device=self.device, dtype=torch.uint8).contiguous()
        if p.numel() != vals.numel():
            raise ValueError("values and pred differ in length")
        status = np.zeros(self._S, np.int32)
        with self._mu:
            rc = L.lib.gg_push_if(self._h, C.c_void_p(vals.data_ptr() if vals.numel() else 0),
                                  C.c_void_p(p.data_ptr() if p.numel() else 0), vals.numel(),
                                  1 if mode == "block" else 0, int(grid), L.ptr(status, C.c_int32),
                                  self._stream())
            self._dirty()
        if rc == L.GG_EPARTIAL:
            failures = {int(s): MemoryError(f"shard {s}: no backed bucket slot for a device append")
                        for s in np.flatnonzero(status)}
            raise ShardInsertError(failures, [])
        L.check(rc, "push_if")
        if commit:
            self.commit()

    def insert_duplicate(self, commit: bool = True) -> None:
        """Every shard appends a copy of its committed contents, read directly from
        its buckets (the bench's _insert_duplicate, bench_cli.py:298-307)."""
        flags = (L.GG_F_COMMIT if commit else 0) | _EXTRA_FLAGS
        with self._mu:
            status = self._status
            if self._hook_exc:
                self._hook_exc = {}
            rc = L.lib.gg_insert_duplicate_ex(self._h, flags, self._status_p, self._stream())
            self._dirty()
            if rc not in (L.GG_OK, L.GG_EPARTIAL):
                L.check(rc, "insert_duplicate")
            if rc == L.GG_EPARTIAL:
                failures = {int(s): self._failure(int(s), int(status[s])) for s in np.flatnonzero(status)}
        if rc == L.GG_EPARTIAL:
            cl = np.diff(self._host()["prefix"].astype(np.int64))
            raise ShardInsertError(failures, [s for s in range(self._S) if cl[s] and s not in failures])

    def commit(self) -> None:
        L.check(L.lib.gg_commit(self._h, self._stream()), "commit")
        self._cache = self._tot = None

    def grow(self, target_total_capacity: int, distribution: Sequence | None = None) -> None:
        if distribution is None:
            per = -(-int(target_total_capacity) // self._S)
            caps = self._caps
            caps.fill(max(per, 0))
        else:
            if len(distribution) != self._S:
                raise ValueError(f"distribution needs {self._S} entries, got {len(distribution)}")
            caps = np.asarray([max(int(x), 0) for x in distribution], np.uint64)
        self._reserve(caps)

    def shrink(self, new_sizes, release=2.0) -> None:
        """Extension (no reference semantics): pop shards to ``new_sizes`` and release
        buckets beyond the minimal prefix; commits.  Slab chunks left without a
        live bucket are unmapped according to ``release``: a number f keeps at
        most f x the needed bytes mapped (default 2.0, the paper's footprint
        bound, unmapping as little as possible -- every unmap/remap costs
        driver time); True unmaps them all; False keeps them all mapped for
        in-place reuse until :meth:`trim`."""
        if isinstance(new_sizes, (int, np.integer)) and new_sizes >= 0:
            ns = self._shrink_buf
            ns.fill(new_sizes)
            total = int(new_sizes) * self._S
        else:
            ns = L.u64_array(np.broadcast_to(np.asarray(new_sizes), (self._S,)))
            total = int(ns.sum())
        if release is True:
            keep = 0
        elif release is False or release is None:
            keep = (1 << 64) - 1
        else:
            keep = int(float(release) * total * self.dtype.itemsize)
        L.check(L.lib.gg_shrink_ex(self._h, self._shrink_p if ns is self._shrink_buf else L.ptr(ns), keep,
                                   self._stream()), "shrink")
        self._dirty()

    def trim(self) -> None:
        """Unmap every cached slab chunk (mapped memory without a live bucket)."""
        L.check(L.lib.gg_trim(self._h), "trim")

    # ------------------------------------------------------------ flattening
    def flatten_device(self, out=None):
        """Committed contents as one contiguous device tensor (K-flatten)."""
        import torch
        n = self.committed_size
        if out is None:
            out = torch.empty(n, dtype=self._torch_dtype, device=self.device)
        elif out.numel() < n or not out.is_contiguous():
            raise ValueError("out must be a contiguous device tensor of committed_size elements")
        L.check(L.lib.gg_flatten(self._h, C.c_void_p(out.data_ptr()), self._stream()), "flatten")
        return out[:n]

    def flatten_to(self, dev_ptr: int) -> int:
        """K-flatten into raw device memory at ``dev_ptr`` (committed_size
        elements) -- any address the GPU can store to, e.g. a peer GPU's
        buffer mapped with CUDA IPC (multigpu.py).  Stream-ordered; returns
        the element count."""
        n = self.committed_size
        L.check(L.lib.gg_flatten(self._h, C.c_void_p(int(dev_ptr)), self._stream()), "flatten")
        return n

    def flatten_range_to(self, lo: int, hi: int, dev_ptr: int) -> int:
        """Committed elements with global index in [lo, hi) to raw device memory
        at ``dev_ptr`` (a slice of flatten(); e.g. into a peer GPU's buffer)."""
        L.check(L.lib.gg_flatten_range(self._h, int(lo), int(hi), C.c_void_p(int(dev_ptr)),
                                       self._stream()), "flatten_range")
        return int(hi) - int(lo)

    def flatten_range(self, lo: int, hi: int):
        """Device tensor of the committed elements with global index in [lo, hi)."""
        import torch
        out = torch.empty(max(0, int(hi) - int(lo)), dtype=self._torch_dtype, device=self.device)
        self.flatten_range_to(lo, hi, out.data_ptr())
        return out

    def flatten(self) -> np.ndarray:
        """Host copy of the committed contents (the reference returns numpy)."""
        return self._to_numpy(self.flatten_device())

    @classmethod
    def from_flat(cls, values, shards: int = DEFAULT_SHARDS,
                  first_bucket_size: int = DEFAULT_FIRST_BUCKET_SIZE, dtype=None,
                  max_buckets: int = MAX_BUCKETS, allocator=None, device=None,
                  arena_va_bytes: int = 0) -> "GrowableArray":
        """Chunk c of ceil(n/S) elements goes to shard c (sharded_array.py:259-282)."""
        import torch
        if isinstance(values, torch.Tensor):
            if dtype is None:
                dtype = values.cpu()[:0].numpy().dtype if values.dtype not in (
                    torch.uint16, torch.uint32, torch.uint64) else {
                    torch.uint16: np.uint16, torch.uint32: np.uint32, torch.uint64: np.uint64}[values.dtype]
            n = values.numel()
        else:
            vals_np = np.asarray(values)
            if dtype is None:
                dtype = vals_np.dtype if (vals_np.size or isinstance(values, np.ndarray)) else np.int64
            values, n = vals_np, vals_np.size
        arr = cls(shards, first_bucket_size, dtype=dtype, max_buckets=max_buckets,
                  allocator=allocator, device=device, arena_va_bytes=arena_va_bytes)
        vals = arr._device_values(values)
        failures = arr._insert_device(vals, split_offsets(n, shards), commit=True)
        if failures:
            raise failures[min(failures)]
        return arr

    # ------------------------------------------------------------ stats / parity
    def memory_stats(self, settle: bool = True) -> dict:
        """Footprint: capacity (the reference's), mapped (physical slab chunks),
        needed bytes.  A shrink unmaps released chunks asynchronously (after
        the work queued before it); ``settle`` waits for that first, so
        ``mapped_bytes`` is the settled footprint (else they are counted in
        ``mapped_bytes`` and reported as ``pending_unmap_bytes``)."""
        if settle:
            L.check(L.lib.gg_settle(self._h), "settle")
        o = np.zeros(7, np.uint64)
        L.check(L.lib.gg_mem_stats(self._h, L.ptr(o), self._stream()), "mem_stats")
        cap, mapped, live, need, allocs, cached, pend = (int(x) for x in o)
        return {"capacity_bytes": cap, "mapped_bytes": mapped, "bucket_bytes": live,
                "needed_bytes": need, "alloc_calls": allocs, "cached_bytes": cached,
                "pending_unmap_bytes": pend,
                "capacity_over_needed": cap / need if need else None,
                "mapped_over_needed": mapped / need if need else None}

    def slab_stats(self) -> dict:
        """Cost of the slab's physical mapping (cumulative counters)."""
        o = np.zeros(11, np.uint64)
        L.check(L.lib.gg_slab_stats(self._h, L.ptr(o)), "slab_stats")
        keys = ("mapped_bytes", "cached_bytes", "chunks_mapped", "chunks_unmapped", "map_ns",
                "unmap_ns", "regions", "va_bytes", "handles_created", "handles_from_pool",
                "pending_unmap_bytes")
        return {k: int(v) for k, v in zip(keys, o)}

    def prefix_device(self, out=None):
        """The committed directory prefix[S+1] as an int64 CUDA tensor (a device
        copy, stream-ordered and capture-safe)."""
        import torch
        if out is None:
            out = torch.empty(self._S + 1, dtype=torch.int64, device=self.device)
        elif out.numel() < self._S + 1 or out.dtype != torch.int64 or not out.is_contiguous():
            raise ValueError("out must be a contiguous int64 device tensor of shards + 1 elements")
        L.check(L.lib.gg_prefix_copy(self._h, C.c_void_p(out.data_ptr()), self._stream()), "prefix_device")
        return out

    def device_state(self) -> dict:
        S = self._S
        st = {k: np.zeros(S + (k == "prefix"), np.uint64) for k in ("sizes", "caps", "flags", "prefix", "ops")}
        L.check(L.lib.gg_device_state(self._h, *(L.ptr(st[k]) for k in
                                                 ("sizes", "caps", "flags", "prefix", "ops")),
                                      self._stream()), "device_state")
        return st

    def _parity_state(self) -> dict:
        """State read back from DEVICE memory; asserts the host mirror agrees."""
        dev = self.device_state()
        host = self._host()
        for k in dev:
            if not np.array_equal(dev[k], host[k]):
                raise AssertionError(f"device/host mirror mismatch in {k}: "
                                     f"{dev[k][:8]} vs {host[k][:8]}")
        return {"sizes": [int(x) for x in dev["sizes"]], "caps": [int(x) for x in dev["caps"]],
                "flags": [int(x) for x in dev["flags"]], "prefix": [int(x) for x in dev["prefix"]],
                "ops": [int(x) for x in dev["ops"]]}

    def synchronize(self) -> None:
        import torch
        torch.cuda.current_stream(self.device).synchronize()

    def close(self) -> None:
        if getattr(self, "_h", None):
            L.lib.gg_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:  # noqa: BLE001 -- interpreter shutdown
            pass

    def __repr__(self) -> str:
        return (f"GrowableArray(shards={self._S}, committed={self.committed_size}, "
                f"capacity={self.total_capacity}, device={self.device})")


def pool_stats(device: int = 0) -> dict:
    """The process-wide cache of physical slab chunks (chunks of destroyed
    arrays and chunks shrinks unmapped), reused by any array before the
    driver is asked for new memory."""
    o = np.zeros(10, np.uint64)
    L.check(L.lib.gg_pool_stats(int(device), L.ptr(o)), "pool_stats")
    return {"cached_bytes": int(o[0]), "chunks": int(o[1]), "hits": int(o[2]), "misses": int(o[3]),
            "cap_bytes": int(o[4]), "graves": int(o[5]), "refused": int(o[6]),
            "slab_cache_bytes": int(o[7]), "slabs_cached": int(o[8]), "slab_cache_hits": int(o[9])}


def pool_trim(device: int = 0) -> None:
    """Wait for destroyed arrays' queued work, then return every cached chunk
    to the driver."""
    L.check(L.lib.gg_pool_trim(int(device)), "pool_trim")


def reclaim(wait: bool = True) -> None:
    """Free what destroyed arrays left behind (their chunks go to the pool);
    destroy itself only records an event behind the array's last work."""
    L.check(L.lib.gg_reclaim(1 if wait else 0), "reclaim")
