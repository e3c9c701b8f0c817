"""GGArray across GPUs: one process per GPU, each owning a
contiguous range of LFVectors in its own device arena.

Insert / grow / shrink / r/w are purely local (no communication).  The only
exchange steps are
  * the global directory: an all-gather of the per-GPU committed sizes (one
    int64 per rank) whose exclusive scan gives each GPU's global base, so
    global order = GPU-major, then shard-major -- exactly the single-array
    ``flatten()`` order of the concatenated shard list;
  * the global flatten / gather: every rank flattens locally (K-flatten) and
    ships its slice to the root, which places it at the rank's global base
    (NCCL point-to-point over NVLink/NVSwitch when the backend is nccl).

The class only needs the local array's ``committed_size`` / ``flatten_device``
(or ``flatten``) / ``get_many`` surface, so the host logic is exercised on CPU
with the gloo backend and the oracle array (tests/test_multigpu_gloo.py).
"""

from __future__ import annotations

import numpy as np


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

    # ---- flatten / gather
    def _local_flat(self):
        import torch
        if hasattr(self.local, "flatten_device"):
            return self.local.flatten_device()
        return torch.from_numpy(np.ascontiguousarray(self.local.flatten()))

    def flatten_global(self, root: int = 0):
        """Gather every rank's committed contents into one array on ``root``
        (global order).  Returns the tensor on root, None elsewhere."""
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
