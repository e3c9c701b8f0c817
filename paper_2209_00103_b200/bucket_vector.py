"""LFVector (shard) layer of the drop-in API: layout arithmetic and the
``ShardVector`` / ``BucketTable`` views (bucket_vector.py:34-308 in the reference).

Storage lives in the device slabs of a ``gg_array`` handle; a ShardVector is a
(handle, shard) pair.  A standalone ``ShardVector(...)`` owns a one-shard
handle.  Bucket views handed out by ``iter_segments`` / ``table.buckets`` are
device views aliasing the slabs (valid until the array is destroyed or the
bucket is released by a shrink).
"""

from __future__ import annotations

import ctypes as C
import threading
import weakref

import numpy as np

from . import _lib as L
from .errors import CapacityError
from .insert_index import AtomicReserver, ReservedRange

MAX_BUCKETS = 58
DEFAULT_FIRST_BUCKET_SIZE = 32

__all__ = ["MAX_BUCKETS", "DEFAULT_FIRST_BUCKET_SIZE", "locate", "bucket_size", "min_buckets_for",
           "capacity_of", "BucketTable", "ShardVector"]


def _check_fb(fb: int) -> None:
    if fb < 1 or fb & (fb - 1):
        raise ValueError(f"first_bucket_size must be a positive power of two, got {fb}")


def locate(i: int, first_bucket_size: int) -> tuple:
    """(bucket, offset) of local index i: b = hibit(i/fb + 1), off = i - fb(2^b - 1)."""
    if i < 0:
        raise ValueError(f"index must be non-negative, got {i}")
    b = (i // first_bucket_size + 1).bit_length() - 1
    return b, i - first_bucket_size * ((1 << b) - 1)


def bucket_size(b: int, first_bucket_size: int, max_buckets: int = MAX_BUCKETS) -> int:
    if not 0 <= b < max_buckets:
        raise ValueError(f"bucket index {b} outside [0, {max_buckets})")
    return first_bucket_size << b


def capacity_of(bucket_count: int, first_bucket_size: int) -> int:
    return first_bucket_size * ((1 << bucket_count) - 1)


def min_buckets_for(n: int, first_bucket_size: int) -> int:
    return 0 if n <= 0 else (-(-n // first_bucket_size)).bit_length()


class _CudaView:
    """__cuda_array_interface__ shim so torch can alias slab memory."""

    def __init__(self, addr: int, n: int, dtype: np.dtype):
        self.__cuda_array_interface__ = {"shape": (n,), "typestr": dtype.str,
                                         "data": (addr, False), "version": 3, "strides": None}


def _view(arr, addr: int, n: int):
    import torch
    t = torch.as_tensor(_CudaView(addr, n, arr._storage_dtype), device=arr.device)
    return t.view(arr._torch_dtype) if arr._torch_dtype != t.dtype else t


class _SizeCounter:
    """The shard's size as the reference's AtomicCounter (value, op_count,
    fetch_add).  One per (array, shard), cached by the array -- reservers
    compare counters by identity -- and holding the array weakly, so the
    cache forms no reference cycle (arrays are freed when dropped, not by
    the cyclic collector at an arbitrary later point)."""

    def __init__(self, arr, s: int):
        self._ref = weakref.ref(arr)
        self._s = s

    def _arr(self):
        a = self._ref()
        if a is None:
            raise RuntimeError("the GrowableArray of this counter was destroyed")
        return a

    @property
    def value(self) -> int:
        return int(self._arr()._host()["sizes"][self._s])

    @property
    def op_count(self) -> int:
        return int(self._arr()._host()["ops"][self._s])

    def fetch_add(self, amount: int) -> int:
        a = self._arr()
        prev = C.c_uint64(0)
        L.check(L.lib.gg_fetch_add(a._h, self._s, int(amount), C.byref(prev), a._stream()),
                "fetch_add")
        a._dirty()
        return int(prev.value)


class BucketTable:
    """A shard's bucket table (bucket_vector.py:82-101).

    ``BucketTable(first_bucket_size, max_buckets)`` builds an empty standalone
    table like the reference's (no storage, all once-flags clear); the tables
    of device arrays (``ShardVector.table``) are live views of the device
    flags and bucket slots."""

    def __init__(self, first_bucket_size: int, max_buckets: int = MAX_BUCKETS):
        _check_fb(first_bucket_size)
        if max_buckets < 1:
            raise ValueError("max_buckets must be >= 1")
        self._sh = None
        self._fb = first_bucket_size
        self._mb = max_buckets
        self._flags = [False] * max_buckets
        self._lock = threading.Lock()

    @classmethod
    def _bind(cls, shard: "ShardVector") -> "BucketTable":
        t = cls.__new__(cls)
        t._sh = shard
        return t

    @property
    def flag_lock(self):
        """The reference guards its once-flags with this lock
        (bucket_vector.py:94, 189-199); here the flags live on the device and
        are updated by CAS / planned kernels, so the lock only serialises host
        callers of the shard's handle."""
        return self._lock if self._sh is None else self._sh._arr._mu

    @property
    def first_bucket_size(self) -> int:
        return self._fb if self._sh is None else self._sh.first_bucket_size

    @property
    def max_buckets(self) -> int:
        return self._mb if self._sh is None else self._sh.max_buckets

    @property
    def allocated_flags(self) -> list:
        if self._sh is None:
            return list(self._flags)
        m = int(self._sh._arr._host()["flags"][self._sh._s])
        return [bool(m >> b & 1) for b in range(self.max_buckets)]

    def allocated_count(self) -> int:
        return sum(self.allocated_flags)

    @property
    def buckets(self) -> list:
        if self._sh is None:
            return [None] * self._mb
        a, s = self._sh._arr, self._sh._s
        ptrs = a._bucket_ptrs()[s]
        fb = self.first_bucket_size
        from .views import DeviceView
        return [DeviceView(_view(a, int(p), fb << b)) if p else None for b, p in enumerate(ptrs)]


class ShardVector:
    """One LFVector.  ``ShardVector(fb, dtype, max_buckets, allocator)`` builds a
    standalone one-shard array; ``GrowableArray.shards[s]`` returns bound views."""

    def __init__(self, first_bucket_size: int = DEFAULT_FIRST_BUCKET_SIZE, dtype=np.int64,
                 max_buckets: int = MAX_BUCKETS, allocator=None, device=None):
        from .sharded_array import GrowableArray
        _check_fb(first_bucket_size)
        self._arr = GrowableArray(1, first_bucket_size, dtype=dtype, max_buckets=max_buckets,
                                  allocator=allocator, device=device)
        self._s = 0

    @classmethod
    def _bind(cls, arr, s: int) -> "ShardVector":
        sv = cls.__new__(cls)
        sv._arr, sv._s = arr, s
        return sv

    # -- properties
    @property
    def first_bucket_size(self) -> int:
        return self._arr.first_bucket_size

    @property
    def max_buckets(self) -> int:
        return self._arr.max_buckets

    @property
    def dtype(self) -> np.dtype:
        return self._arr.dtype

    @property
    def size(self) -> int:
        return int(self._arr._host()["sizes"][self._s])

    def __len__(self) -> int:
        return self.size

    @property
    def capacity(self) -> int:
        return int(self._arr._host()["caps"][self._s])

    @property
    def size_counter(self) -> _SizeCounter:
        # one counter object per (array, shard): reservers compare counters by identity
        return self._arr._counter(self._s)

    @property
    def table(self) -> BucketTable:
        return BucketTable._bind(self)

    def locate(self, i: int) -> tuple:
        return locate(i, self.first_bucket_size)

    def bucket_size(self, b: int) -> int:
        return bucket_size(b, self.first_bucket_size, self.max_buckets)

    # -- growth
    def new_bucket(self, b: int) -> bool:
        """CAS-once allocation of bucket b on the device (paper Alg. 2)."""
        a = self._arr
        won = C.c_int32(0)
        with a._mu:
            a._hook_exc = {}
            rc = L.lib.gg_new_bucket(a._h, self._s, int(b), C.byref(won), a._stream())
            a._dirty()
            if rc == L.GG_ENOMEM and self._s in a._hook_exc:
                raise a._hook_exc.pop(self._s)
            L.check(rc, "new_bucket")
        return bool(won.value)

    def push_back_batch(self, values, reserver=None) -> ReservedRange:
        """Append ``values`` at a freshly reserved contiguous range, argument
        order; returns the range the library reserved (read under the
        handle's lock, so concurrent callers on one shard get disjoint ranges)."""
        a = self._arr
        vals = a._device_values(values)
        n = int(vals.numel())
        if reserver is not None and not isinstance(reserver, AtomicReserver):
            rng = reserver.reserve(self.size_counter, n)
            if rng.count:
                a._write_ranges({self._s: (rng.start, vals)})
            return rng
        if n == 0:
            return ReservedRange(self.size_counter.fetch_add(0), 0)
        offsets = np.zeros(a.shard_count + 1, np.uint64)
        offsets[self._s + 1:] = n
        failures, starts = a._insert_device(vals, offsets, want_starts=True)
        if failures:
            raise failures[self._s]
        return ReservedRange(int(starts[self._s]), n)

    def reserve(self, min_capacity: int) -> None:
        caps = np.zeros(self._arr.shard_count, np.uint64)
        caps[self._s] = max(int(min_capacity), 0)
        self._arr._reserve(caps)

    # -- element access
    def get(self, i: int):
        return self._arr._get(self._s, i)

    def set(self, i: int, value) -> None:
        self._arr._set(self._s, i, value)

    def iter_segments(self, stop=None, start: int = 0):
        """Writable device views (:class:`~paper_2209_00103_b200.views.DeviceView`,
        numpy-ufunc capable) of local [start, stop), one per touched bucket
        (bucket_vector.py:279-295)."""
        from .views import DeviceView
        for t in self._segment_tensors(stop, start):
            yield DeviceView(t)

    def _segment_tensors(self, stop=None, start: int = 0):
        """Raw torch CUDA tensors aliasing the buckets of local [start, stop)."""
        a = self._arr
        stop = self.size if stop is None else stop
        fb = self.first_bucket_size
        ptrs = a._bucket_ptrs()[self._s] if stop > start else None
        esz = a.dtype.itemsize
        i = start
        while i < stop:
            b, off = locate(i, fb)
            if b >= self.max_buckets or not ptrs[b]:
                raise RuntimeError(f"bucket {b} unpublished while walking [{start}, {stop})")
            n = min((fb << b) - off, stop - i)
            yield _view(a, int(ptrs[b]) + off * esz, n)
            i += n

    def to_numpy(self, stop=None) -> np.ndarray:
        import torch
        segs = list(self._segment_tensors(stop))
        if not segs:
            return np.empty(0, self.dtype)
        return self._arr._to_numpy(torch.cat(segs))

    def __repr__(self) -> str:
        return f"ShardVector(size={self.size}, capacity={self.capacity}, fb={self.first_bucket_size})"
