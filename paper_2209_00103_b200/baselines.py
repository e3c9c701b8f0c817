"""GPU baselines the GGArray is measured against (baselines.py:29-279 in the
reference; paper section 3-A):

* ``StaticArray``   -- one ``cudaMalloc``'d buffer of final capacity; insert
  kernels with one atomic per element / per warp / per CTA (paper 3-B) or a
  single batch reservation (reference ``insert_batch`` semantics).
* ``DoublingArray`` -- semi-static, host-resized: a new stream-ordered
  allocation of initial*2^j elements, a device-to-device copy of the live
  elements, free of the old buffer (``elements_copied`` counts them).
* ``ChunkTableArray`` -- the paper's ``memMap`` baseline: one VA reservation,
  physical 2 MiB granules appended with cuMemCreate/cuMemMap on resize; the
  array stays contiguous and nothing is ever copied.  Capacity keeps the
  reference's chunk semantics (chunks * chunk_size elements).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib as L
from .bucket_vector import _CudaView
from .errors import CapacityError
from .insert_index import ReservedRange

__all__ = ["StaticArray", "DoublingArray", "ChunkTableArray", "DEFAULT_CHUNK_SIZE", "INSERT_ALGOS"]

DEFAULT_CHUNK_SIZE = 64 * 1024
INSERT_ALGOS = {"atomic": L.GG_ALGO_ATOMIC, "warp": L.GG_ALGO_WARP, "block": L.GG_ALGO_BLOCK}


def _zero_bytes(addr: int, nbytes: int, device) -> None:
    import torch
    if nbytes:
        torch.as_tensor(_CudaView(addr, nbytes, np.dtype(np.uint8)), device=device).zero_()


class _Counter:
    """size counter with the reference's AtomicCounter surface; the value lives on
    the device (d_count) and is mirrored on the host."""

    def __init__(self, owner):
        self._o = owner
        self.op_count = 0

    @property
    def value(self) -> int:
        return self._o._count

    def fetch_add(self, n: int) -> int:
        prev = self._o._count
        self._o._count += n
        self._o._d_count.add_(n)
        self.op_count += 1
        return prev


class _FlatArray:
    """Contiguous device storage at ``_base`` with a device size counter."""

    def __init__(self, dtype, device):
        import torch
        from .sharded_array import _INT_OF_SIZE, _torch_dtype
        if not torch.cuda.is_available():
            raise RuntimeError("GPU baselines need a CUDA device")
        self.dtype = np.dtype(dtype)
        if self.dtype not in L.DTYPE_CODES:
            raise ValueError(f"unsupported dtype {self.dtype}")
        self.device = torch.device("cuda", torch.cuda.current_device() if device is None
                                   else torch.device(device).index or 0)
        self._torch_dtype = _torch_dtype(self.dtype)
        self._int_np = np.dtype(_INT_OF_SIZE[self.dtype.itemsize])
        self._count = 0
        self._d_count = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.size_counter = _Counter(self)
        self._base = 0

    # subclass provides: capacity, _base
    def _stream(self):
        import torch
        return torch.cuda.current_stream(self.device).cuda_stream

    def _tensor(self, n: int):
        import torch
        if n == 0:
            return torch.empty(0, dtype=self._torch_dtype, device=self.device)
        sd = self._int_np if self.dtype.kind == "u" and self.dtype.itemsize > 1 else self.dtype
        t = torch.as_tensor(_CudaView(self._base, n, sd), device=self.device)
        return t.view(self._torch_dtype) if t.dtype != self._torch_dtype else t

    @property
    def size(self) -> int:
        return min(self._count, self.capacity)

    def __len__(self) -> int:
        return self.size

    def _vals(self, values):
        import torch
        if isinstance(values, torch.Tensor):
            return values.reshape(-1).to(self._torch_dtype).to(self.device).contiguous()
        a = np.ascontiguousarray(np.asarray(values, dtype=self.dtype).reshape(-1))
        return torch.from_numpy(a.view(self._int_np)).to(self.device).view(self._torch_dtype)

    def insert_batch(self, values, reserver=None, algo: str | None = None) -> ReservedRange:
        """Append ``values``.  Default: one reservation, argument order (the
        reference's insert_batch); ``algo`` in {atomic, warp, block} runs the
        paper's per-element / per-warp / per-CTA reservation kernels (order
        within the batch is then arbitrary)."""
        v = self._vals(values)
        n = v.numel()
        if self._count + n > self.capacity:
            raise CapacityError(f"insert of {n} exceeds capacity {self.capacity}")
        start = self._count
        if algo is None and reserver is not None:
            rng = reserver.reserve(self.size_counter, n)
            self._tensor(rng.end)[rng.start:rng.end].copy_(v)
            return rng
        if algo is None:
            # one reservation of the whole batch (the reference's AtomicReserver:
            # one counter op), then ONE vectorised copy kernel into [start, start+n)
            self._count += n
            self.size_counter.op_count += 1
            L.check(L.lib.gg_flat_append(C.c_void_p(self._base), self.capacity,
                                         C.c_void_p(self._d_count.data_ptr()), start,
                                         C.c_void_p(v.data_ptr()), n, self.dtype.itemsize,
                                         self._stream()), "flat_append")
            return ReservedRange(start, n)
        code = INSERT_ALGOS[algo]
        L.check(L.lib.gg_flat_insert(C.c_void_p(self._base), self.capacity,
                                     C.c_void_p(self._d_count.data_ptr()), C.c_void_p(v.data_ptr()),
                                     n, self.dtype.itemsize, code, self._stream()), "flat_insert")
        self._count += n
        self.size_counter.op_count += {"atomic": n, "warp": -(-n // 32), "block": -(-n // 256)}[algo]
        return ReservedRange(start, n)

    def _check(self, i: int) -> None:
        if not 0 <= i < self.size:
            raise IndexError(f"index {i} outside size {self.size}")

    def get(self, i: int):
        self._check(i)
        return self.to_numpy()[i] if self.size < 4096 else \
            self._tensor(i + 1)[i:i + 1].cpu().numpy().view(self.dtype)[0]

    def set(self, i: int, value) -> None:
        self._check(i)
        self._tensor(i + 1)[i:i + 1].copy_(self._vals([value]))

    def view(self):
        """Writable device view (torch tensor) of the occupied prefix."""
        return self._tensor(self.size)

    def to_numpy(self) -> np.ndarray:
        import torch
        t = self._tensor(self.size).view(getattr(torch, self._int_np.name))
        return t.cpu().numpy().view(self.dtype)

    def rw_add(self, c, passes: int = 1, fused: bool = False) -> None:
        """``passes`` separate +c sweeps over the contiguous array (static r/w)."""
        a = np.asarray(c).astype(self.dtype).reshape(1)
        L.check(L.lib.gg_flat_add(C.c_void_p(self._base), self.size, L.DTYPE_CODES[self.dtype],
                                  a.ctypes.data_as(C.c_void_p), int(passes), int(fused),
                                  self._stream()), "flat_add")


class StaticArray(_FlatArray):
    def __init__(self, capacity: int, dtype=np.int64, device=None):
        if capacity < 0:
            raise ValueError("capacity must be non-negative")
        super().__init__(dtype, device)
        import torch
        self._cap = int(capacity)
        self._store = torch.zeros(max(self._cap, 1) * self.dtype.itemsize, dtype=torch.uint8,
                                  device=self.device)
        self._base = self._store.data_ptr()

    @property
    def capacity(self) -> int:
        return self._cap


class DoublingArray(_FlatArray):
    def __init__(self, initial_capacity: int = 32, dtype=np.int64, device=None):
        if initial_capacity < 1:
            raise ValueError("initial_capacity must be >= 1")
        super().__init__(dtype, device)
        self._initial = int(initial_capacity)
        self._cap = 0
        self.elements_copied = 0
        self._alloc(self._initial, copy=False)

    def _alloc(self, cap: int, copy: bool) -> None:
        import torch
        p = C.c_void_p()
        st = self._stream()
        L.check(L.lib.gg_buf_alloc(cap * self.dtype.itemsize, st, C.byref(p)), "buf_alloc")
        # the reference allocates np.zeros; zero the fresh buffer too
        _zero_bytes(p.value, cap * self.dtype.itemsize, self.device)
        if copy and self.size:
            L.check(L.lib.gg_buf_copy(p, C.c_void_p(self._base), self.size * self.dtype.itemsize, st),
                    "buf_copy")
        if self._base:
            L.check(L.lib.gg_buf_free(C.c_void_p(self._base), st), "buf_free")
        self._base, self._cap = p.value, cap

    @property
    def capacity(self) -> int:
        return self._cap

    def resize(self, min_capacity: int) -> None:
        """Grow to the smallest initial*2^j >= min_capacity, copying every element."""
        if min_capacity <= self._cap:
            return
        cap = self._initial
        while cap < min_capacity:
            cap *= 2
        n = self.size
        self._alloc(cap, copy=True)
        self.elements_copied += n

    def push_back(self, value) -> int:
        n = self._count
        if n + 1 > self._cap:
            self.resize(n + 1)
        self._tensor(n + 1)[n:n + 1].copy_(self._vals([value]))
        self.size_counter.fetch_add(1)
        return n

    def __del__(self):
        try:
            if self._base:
                L.lib.gg_buf_free(C.c_void_p(self._base), None)
        except Exception:  # noqa: BLE001
            pass


class ChunkTableArray(_FlatArray):
    def __init__(self, chunk_size: int = DEFAULT_CHUNK_SIZE, dtype=np.int64, device=None,
                 va_bytes: int = 0):
        if chunk_size < 1:
            raise ValueError("chunk_size must be >= 1")
        super().__init__(dtype, device)
        import torch
        self.chunk_size = int(chunk_size)
        self.elements_copied = 0
        self._chunks = 0
        if not va_bytes:
            va_bytes = torch.cuda.get_device_properties(self.device).total_memory
        h = C.c_void_p()
        L.check(L.lib.gg_vmm_create(self.device.index, int(va_bytes), C.byref(h)), "vmm_create")
        self._vmm = h
        b, m, g = C.c_uint64(), C.c_uint64(), C.c_uint64()
        L.lib.gg_vmm_info(h, C.byref(b), C.byref(m), C.byref(g))
        self._base, self.granule = b.value, g.value

    @property
    def capacity(self) -> int:
        return self._chunks * self.chunk_size

    @property
    def mapped_bytes(self) -> int:
        b, m, g = C.c_uint64(), C.c_uint64(), C.c_uint64()
        L.lib.gg_vmm_info(self._vmm, C.byref(b), C.byref(m), C.byref(g))
        return m.value

    def resize(self, min_capacity: int) -> None:
        """Append chunks (mapping 2 MiB granules) until capacity >= min_capacity."""
        chunks = -(-max(int(min_capacity), 0) // self.chunk_size)
        if chunks <= self._chunks:
            return
        old = self.capacity
        L.check(L.lib.gg_vmm_ensure(self._vmm, chunks * self.chunk_size * self.dtype.itemsize),
                "vmm_ensure")
        self._chunks = chunks
        # new chunks read as zeros, like the reference's np.zeros chunks
        esz = self.dtype.itemsize
        _zero_bytes(self._base + old * esz, (self.capacity - old) * esz, self.device)

    def chunk_views(self, stop=None):
        stop = self.size if stop is None else stop
        t = self._tensor(stop)
        for lo in range(0, stop, self.chunk_size):
            yield t[lo:min(stop, lo + self.chunk_size)]

    def __del__(self):
        try:
            if getattr(self, "_vmm", None):
                L.lib.gg_vmm_destroy(self._vmm)
                self._vmm = None
        except Exception:  # noqa: BLE001
            pass
