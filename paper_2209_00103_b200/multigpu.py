"""GGArray across GPUs: one process per GPU, each owning a
contiguous range of LFVectors in its own device slabs.

Insert / grow / shrink / r/w are purely local (no communication).  The only
exchange steps are
  * the global directory: an all-gather of the per-GPU committed sizes (one
    int64 per rank) whose exclusive scan gives each GPU's global base, so
    global order = GPU-major, then shard-major -- exactly the single-array
    ``flatten()`` order of the concatenated shard list;
  * the global flatten / gather.  ``method="peer"`` (device arrays): the
    root allocates the global buffer (cudaMalloc), publishes its CUDA IPC
    handle, and every rank runs its K-flatten STRAIGHT INTO the root's buffer
    at its global base -- the flatten kernel's 16 B stores cross NVLink /
    NVSwitch, so the gather is fused into the flatten tile by tile, with no
    staging copy and no collective on the data path.  ``all_gather_flat(
    method="peer")`` does the same into every rank's buffer.  ``method=
    "nccl"``: local K-flatten, then point-to-point sends into the root buffer
    (also the CPU/gloo path the tests use with the oracle array).

The class only needs the local array's ``committed_size`` / ``flatten_device``
(or ``flatten``) / ``get_many`` surface, so the host logic is exercised on CPU
with the gloo backend and the oracle array (tests/test_multigpu_gloo.py).
"""

from __future__ import annotations

import ctypes as C

import numpy as np

_TORCH_DT = None


def _torch_dtype(np_dtype):
    import torch
    global _TORCH_DT
    if _TORCH_DT is None:
        _TORCH_DT = {np.dtype(k): v for k, v in [
            (np.int8, torch.int8), (np.uint8, torch.uint8), (np.int16, torch.int16),
            (np.uint16, torch.uint16), (np.int32, torch.int32), (np.uint32, torch.uint32),
            (np.int64, torch.int64), (np.uint64, torch.uint64), (np.float16, torch.float16),
            (np.float32, torch.float32), (np.float64, torch.float64)]}
    return _TORCH_DT[np.dtype(np_dtype)]


class PeerBuffer:
    """A cudaMalloc'd device buffer other processes can map (CUDA IPC).  Exposes
    ``__cuda_array_interface__`` so ``torch.as_tensor(buf, device=...)`` views
    it without a copy; freed when the last reference goes."""

    _TYPESTR = {np.dtype(t): np.dtype(t).str for t in (np.int8, np.uint8, np.int16, np.uint16,
                                                        np.int32, np.uint32, np.int64, np.uint64,
                                                        np.float16, np.float32, np.float64)}

    def __init__(self, n: int, dtype):
        from . import _lib as L
        self.L, self.n, self.dtype = L, int(n), np.dtype(dtype)
        p = C.c_void_p()
        L.check(L.lib.gg_ipc_alloc(max(1, self.n) * self.dtype.itemsize, C.byref(p)), "ipc_alloc")
        self.ptr = int(p.value)

    def handle(self) -> bytes:
        buf = C.create_string_buffer(int(self.L.lib.gg_ipc_handle_bytes()))
        self.L.check(self.L.lib.gg_ipc_get_handle(C.c_void_p(self.ptr), buf), "ipc_get_handle")
        return buf.raw

    @property
    def __cuda_array_interface__(self):
        return {"shape": (self.n,), "typestr": self._TYPESTR[self.dtype], "data": (self.ptr, False),
                "version": 3, "strides": None}

    def tensor(self, device):
        import torch
        t = torch.as_tensor(self, device=device)
        t._peer_buffer_owner = self          # keep the allocation alive with the view
        return t

    def __del__(self):
        if getattr(self, "ptr", 0):
            self.L.lib.gg_ipc_free(C.c_void_p(self.ptr))
            self.ptr = 0


class PeerMapping:
    """A peer's PeerBuffer opened in this process (cudaIpcOpenMemHandle with
    lazy peer access): a device address this GPU's kernels store to over
    NVLink."""

    def __init__(self, handle: bytes):
        from . import _lib as L
        self.L = L
        p = C.c_void_p()
        L.check(L.lib.gg_ipc_open(C.create_string_buffer(handle, len(handle)), C.byref(p)), "ipc_open")
        self.ptr = int(p.value)

    def close(self):
        if self.ptr:
            self.L.lib.gg_ipc_close(C.c_void_p(self.ptr))
            self.ptr = 0

    def __del__(self):
        self.close()


class DistributedGrowableArray:
    def __init__(self, local, group=None, device=None):
        import torch.distributed as dist
        self.local = local
        self.group = group
        self.dist = dist
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        self.device = device

    # ---- directory (the one collective on the data path)
    def global_prefix(self) -> list:
        """[base_0, ..., base_{G-1}, total]: all-gather of committed sizes + scan."""
        import torch
        t = torch.tensor([int(self.local.committed_size)], dtype=torch.int64, device=self.device)
        parts = [torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(parts, t, group=self.group)
        sizes = [int(p.item()) for p in parts]
        out = [0]
        for n in sizes:
            out.append(out[-1] + n)
        return out

    @property
    def global_size(self) -> int:
        return self.global_prefix()[-1]

    def locate_global(self, g: int, prefix=None) -> tuple:
        """Global index -> (rank, local committed index on that rank)."""
        p = prefix or self.global_prefix()
        if not 0 <= g < p[-1]:
            raise IndexError(f"global index {g} outside {p[-1]}")
        r = int(np.searchsorted(np.asarray(p), g, side="right")) - 1
        return r, g - p[r]

    def get_global(self, g: int, prefix=None):
        """Element at global index g (collective: every rank gets the value;
        the owner reads it with its local get_global)."""
        r, loc = self.locate_global(g, prefix)
        box = [self.local.get_global(loc) if self.rank == r else None]
        self.dist.broadcast_object_list(box, src=r, group=self.group)
        return box[0]

    def set_global(self, g: int, value, prefix=None) -> None:
        """Write the element at global index g (collective; only the owner writes)."""
        r, loc = self.locate_global(g, prefix)
        if self.rank == r:
            self.local.set_global(loc, value)
        self.dist.barrier(group=self.group)

    # ---- flatten / gather
    def _local_flat(self):
        import torch
        if hasattr(self.local, "flatten_device"):
            return self.local.flatten_device()
        return torch.from_numpy(np.ascontiguousarray(self.local.flatten()))

    def _peer_ok(self) -> bool:
        return hasattr(self.local, "flatten_to")

    def _sync_local(self):
        import torch
        torch.cuda.current_stream(self.device).synchronize()

    def flatten_global(self, root: int = 0, method: str = "auto"):
        """Gather every rank's committed contents into one array on ``root``
        (global order).  Returns the tensor on root, None elsewhere.
        ``method``: "peer" (fused flatten into the root's buffer over CUDA
        IPC), "nccl" (local flatten + point-to-point), "auto" = peer for
        device arrays."""
        if method == "auto":
            method = "peer" if self._peer_ok() else "nccl"
        if method == "peer":
            return self._flatten_global_peer(root)
        return self._flatten_global_p2p(root)

    def _flatten_global_peer(self, root: int):
        g = PeerGather(self, root)
        g.run()
        g.wait()
        out = g.result()
        g.close()
        return out

    def all_gather_flat_peer(self):
        """Every rank receives the whole flattened array: each rank's K-flatten
        stores its slice into EVERY rank's buffer (one fused flatten per
        destination, over CUDA IPC)."""
        p = self.global_prefix()
        esz = np.dtype(self.local.dtype).itemsize
        buf = PeerBuffer(p[-1], self.local.dtype)
        handles = [None] * self.world
        self.dist.all_gather_object(handles, buf.handle(), group=self.group)
        maps = [None if r == self.rank else PeerMapping(handles[r]) for r in range(self.world)]
        if p[self.rank + 1] > p[self.rank]:
            for r in range(self.world):
                dst = buf.ptr if r == self.rank else maps[r].ptr
                self.local.flatten_to(dst + p[self.rank] * esz)
        self._sync_local()
        self.dist.barrier(group=self.group)
        for m in maps:
            if m is not None:
                m.close()
        return buf.tensor(self.device)

    def rebalance_flat_peer(self):
        """Even flat slices across ranks: rank r ends with global indices
        [r*q, min((r+1)*q, N)), q = ceil(N / G).  Each rank flattens the pieces
        of its committed range straight into the owning ranks' buffers
        (gg_flatten_range into CUDA-IPC mapped peer memory): the rebalance is
        the flatten, with no staging copy and no collective on the data path."""
        p = self.global_prefix()
        n, G, me = p[-1], self.world, self.rank
        q = -(-n // G) if n else 0
        lo = [min(r * q, n) for r in range(G)]
        hi = [min((r + 1) * q, n) for r in range(G)]
        esz = np.dtype(self.local.dtype).itemsize
        buf = PeerBuffer(hi[me] - lo[me], self.local.dtype)
        handles = [None] * G
        self.dist.all_gather_object(handles, buf.handle(), group=self.group)
        maps = [None if r == me else PeerMapping(handles[r]) for r in range(G)]
        for r in range(G):
            a, b = max(lo[r], p[me]), min(hi[r], p[me + 1])
            if a < b:
                dst = buf.ptr if r == me else maps[r].ptr
                self.local.flatten_range_to(a - p[me], b - p[me], dst + (a - lo[r]) * esz)
        self._sync_local()
        self.dist.barrier(group=self.group)
        for m in maps:
            if m is not None:
                m.close()
        return buf.tensor(self.device), (lo[me], hi[me])

    def _flatten_global_p2p(self, root: int):
        import torch
        p = self.global_prefix()
        mine = self._local_flat()
        if self.rank == root:
            out = torch.empty(p[-1], dtype=mine.dtype, device=mine.device)
            out[p[self.rank]:p[self.rank + 1]] = mine
            reqs = []
            for r in range(self.world):
                if r != root and p[r + 1] > p[r]:
                    reqs.append(self.dist.irecv(out[p[r]:p[r + 1]], src=r, group=self.group))
            for q in reqs:
                q.wait()
            return out
        if p[self.rank + 1] > p[self.rank]:
            self.dist.send(mine.contiguous(), dst=root, group=self.group)
        return None

    def allgather_flat(self):
        """Every rank gets the whole flattened array (all-gather of slices)."""
        import torch
        p = self.global_prefix()
        mine = self._local_flat()
        n_max = max(p[r + 1] - p[r] for r in range(self.world))
        buf = torch.zeros(n_max, dtype=mine.dtype, device=mine.device)
        buf[:mine.numel()] = mine
        parts = [torch.empty_like(buf) for _ in range(self.world)]
        self.dist.all_gather(parts, buf, group=self.group)
        return torch.cat([parts[r][:p[r + 1] - p[r]] for r in range(self.world)])


class PeerGather:
    """Reusable fused gather-flatten to ``root`` (collective setup once): the
    root's global buffer is allocated and its IPC handle broadcast; every
    other rank maps it.  ``run()`` launches this rank's K-flatten straight into
    the root buffer at the rank's global base (stream-ordered, no sync);
    ``wait()`` = local stream sync + barrier.  The directory must not change
    between setup and the runs."""

    def __init__(self, d: "DistributedGrowableArray", root: int = 0):
        self.d, self.root = d, root
        self.prefix = d.global_prefix()
        self.esz = np.dtype(d.local.dtype).itemsize
        handle = [None]
        self.buf = self.mapping = None
        if d.rank == root:
            self.buf = PeerBuffer(self.prefix[-1], d.local.dtype)
            handle[0] = self.buf.handle()
        d.dist.broadcast_object_list(handle, src=root, group=d.group)
        if d.rank == root:
            self.dst = self.buf.ptr
        else:
            self.mapping = PeerMapping(handle[0])
            self.dst = self.mapping.ptr

    @property
    def my_bytes(self) -> int:
        r = self.d.rank
        return (self.prefix[r + 1] - self.prefix[r]) * self.esz

    def run(self):
        r = self.d.rank
        if self.prefix[r + 1] > self.prefix[r]:
            self.d.local.flatten_to(self.dst + self.prefix[r] * self.esz)

    def wait(self):
        self.d._sync_local()
        self.d.dist.barrier(group=self.d.group)

    def result(self):
        return self.buf.tensor(self.d.device) if self.buf is not None else None

    def close(self):
        if self.mapping is not None:
            self.mapping.close()
            self.mapping = None
