"""Closed-form capacity of the sharded structure (memory_model.py:136-177 in the
reference): the footprint the B200 arena must match byte for byte.  The
reference's section-5 log-normal sizing model (run_model & co.) is analytic,
host-only and outside the hot path; it is not part of this package."""

from __future__ import annotations

import numpy as np

DEFAULT_ELEMENT_SIZE = 4

__all__ = ["sharded_capacity_elements", "ggarray_capacity_for", "DEFAULT_ELEMENT_SIZE"]


def _min_cap(m: np.ndarray, fb: int) -> np.ndarray:
    """fb * (2^k - 1) for the smallest k covering m (0 for m == 0)."""
    t = (m + fb - 1) // fb
    k = np.zeros_like(t)
    nz = t > 0
    k[nz] = np.floor(np.log2(t[nz].astype(np.float64))).astype(np.int64) + 1
    # guard float rounding at exact powers of two
    too_small = fb * ((np.int64(1) << k) - 1) < m
    k[too_small] += 1
    too_big = (k > 0) & (fb * ((np.int64(1) << (k - 1)) - 1) >= m)
    k[too_big] -= 1
    return np.where(m > 0, fb * ((np.int64(1) << k) - 1), 0)


def sharded_capacity_elements(demands, shards: int, first_bucket_size: int) -> np.ndarray:
    """Elements allocated for each total demand split as evenly as possible."""
    d = np.asarray(demands, dtype=np.int64)
    if np.any(d < 0):
        raise ValueError("demand must be non-negative")
    q, r = np.divmod(d, shards)
    return r * _min_cap(q + 1, first_bucket_size) + (shards - r) * _min_cap(q, first_bucket_size)


def ggarray_capacity_for(demand: int, shards: int = 32, first_bucket_size: int = 32,
                         element_size: int = DEFAULT_ELEMENT_SIZE) -> int:
    return int(sharded_capacity_elements([demand], shards, first_bucket_size)[0]) * element_size
