"""Capacity planning under uncertain demand (reference memory_model.py, paper
section 5) with the sharded structure's capacity MEASURED on the device.

The reference's model: a run ends with ``base_size * LogNormal(mu, sigma)``
elements; three sizing policies are compared per sigma -- the realised demand
(optimal, known only afterwards), a static allocation sized to overflow with
probability ``failure_prob``, and the capacity the GGArray allocates on demand
(closed form: demand split evenly, each shard its minimal bucket prefix,
memory_model.py:143-177).  ``run_model`` reproduces the reference's rows for
the same seed (same RNG stream, memory_model.py:184-227).  ``measure_device``
closes the loop the paper leaves open: it builds GGArrays on the B200 for
sampled demands and reports the capacity and the physically mapped bytes the
slab store actually holds next to the closed form (bench_cli ``memory-model
--measure N``).
"""

from __future__ import annotations

import csv
import math
from dataclasses import dataclass, replace
from statistics import NormalDist

import numpy as np

DEFAULT_ELEMENT_SIZE = 4
CSV_COLUMNS = ["sigma", "optimal_mean", "static_p99", "ggarray_mean", "static_ratio", "ggarray_ratio"]
MEASURED_COLUMNS = ["measured_samples", "measured_capacity_mean", "measured_mapped_mean",
                    "measured_mapped_ratio", "measured_mapped_ratio_max"]

__all__ = ["DEFAULT_ELEMENT_SIZE", "CSV_COLUMNS", "MEASURED_COLUMNS", "MemoryModelParams",
           "MemoryReport", "normal_quantile", "static_requirement", "sharded_capacity_elements",
           "ggarray_capacity_for", "run_model", "write_report_csv", "measure_device"]


def normal_quantile(p: float) -> float:
    """Inverse standard-normal CDF (memory_model.py:53-78).  The reference uses
    Acklam's rational approximation refined by one Halley step; the stdlib's
    NormalDist.inv_cdf (Wichura AS241) agrees with it to ~1e-15 relative."""
    if not 0.0 < p < 1.0:
        raise ValueError(f"p must be in (0, 1), got {p}")
    return NormalDist().inv_cdf(p)


@dataclass(frozen=True)
class MemoryModelParams:
    """Inputs of the model (memory_model.py:81-101): same fields, same checks."""
    mu: float = 0.0
    sigma: float = 1.0
    failure_prob: float = 0.01
    base_size: int = 1_000_000
    samples: int = 100_000
    seed: int = 0

    def __post_init__(self):
        if self.sigma < 0:
            raise ValueError(f"sigma must be >= 0, got {self.sigma}")
        if not 0.0 < self.failure_prob < 1.0:
            raise ValueError(f"failure_prob must be in (0, 1), got {self.failure_prob}")
        if self.base_size < 1:
            raise ValueError(f"base_size must be >= 1, got {self.base_size}")
        if self.samples < 1:
            raise ValueError(f"samples must be >= 1, got {self.samples}")


@dataclass(frozen=True)
class MemoryReport:
    """One sigma of the model, in bytes (memory_model.py:104-131)."""
    sigma: float
    element_size: int
    optimal_bytes: float
    static_p_bytes: float
    ggarray_capacity_bytes: float
    ggarray_worst_bytes: float
    static_ratio: float
    ggarray_ratio: float
    ggarray_worst_ratio: float

    @property
    def optimal_elements(self) -> float:
        return self.optimal_bytes / self.element_size

    @property
    def static_p_elements(self) -> float:
        return self.static_p_bytes / self.element_size

    @property
    def ggarray_capacity_elements(self) -> float:
        return self.ggarray_capacity_bytes / self.element_size


def static_requirement(params: MemoryModelParams, element_size: int = DEFAULT_ELEMENT_SIZE) -> float:
    """base_size * exp(mu + sigma * z_{1-p}) * element_size (memory_model.py:134-140)."""
    z = normal_quantile(1.0 - params.failure_prob)
    return params.base_size * math.exp(params.mu + params.sigma * z) * element_size


def _min_cap(m: np.ndarray, fb: int) -> np.ndarray:
    """fb * (2^k - 1) for the smallest k covering m (0 for m == 0): the
    capacity of a shard's minimal bucket prefix (bucket_vector.py:69-79)."""
    m = np.asarray(m, dtype=np.int64)
    t = (m + fb - 1) // fb
    # bit length of t, exact for t < 2^53 via frexp's exponent
    k = np.frexp(np.maximum(t, 1).astype(np.float64))[1].astype(np.int64)
    return np.where(m > 0, fb * ((np.int64(1) << k) - 1), 0)


def sharded_capacity_elements(demands, shards: int, first_bucket_size: int) -> np.ndarray:
    """Elements allocated for each total demand split as evenly as possible
    (memory_model.py:152-166): r shards hold q+1, the others q."""
    d = np.asarray(demands, dtype=np.int64)
    if np.any(d < 0):
        raise ValueError("demand must be non-negative")
    q, r = np.divmod(d, shards)
    return r * _min_cap(q + 1, first_bucket_size) + (shards - r) * _min_cap(q, first_bucket_size)


def ggarray_capacity_for(demand: int, shards: int = 32, first_bucket_size: int = 32,
                         element_size: int = DEFAULT_ELEMENT_SIZE) -> int:
    """Bytes the sharded structure allocates for ``demand`` elements."""
    return int(sharded_capacity_elements([demand], shards, first_bucket_size)[0]) * element_size


def _sigma_grid() -> list:
    return [round(0.1 * i, 1) for i in range(21)]


def run_model(params: MemoryModelParams, shards: int = 32, first_bucket_size: int = 32,
              element_size: int = DEFAULT_ELEMENT_SIZE, sigma_grid=None, out=None,
              header: bool = True) -> list:
    """Sweep sigma (default 0.0..2.0 step 0.1), Monte-Carlo the demand at each
    point, report the three sizing policies (memory_model.py:184-227).  One
    generator for the whole sweep, so rows equal the reference's for a seed."""
    grid = _sigma_grid() if sigma_grid is None else list(sigma_grid)
    rng = np.random.default_rng(params.seed)
    reports = []
    for sigma in grid:
        p = replace(params, sigma=sigma)
        demands = np.rint(p.base_size * rng.lognormal(mean=p.mu, sigma=sigma, size=p.samples))
        demands = np.maximum(demands.astype(np.int64), 1)
        caps = sharded_capacity_elements(demands, shards, first_bucket_size)
        opt = float(demands.mean()) * element_size
        stat = static_requirement(p, element_size)
        gg_mean = float(caps.mean()) * element_size
        reports.append(MemoryReport(
            sigma=sigma, element_size=element_size, optimal_bytes=opt, static_p_bytes=stat,
            ggarray_capacity_bytes=gg_mean, ggarray_worst_bytes=float(caps.max()) * element_size,
            static_ratio=stat / opt, ggarray_ratio=gg_mean / opt,
            ggarray_worst_ratio=float((caps / demands).max())))
    if out is not None:
        write_report_csv(reports, out, header=header)
    return reports


def write_report_csv(reports, out, header: bool = True, measured=None) -> None:
    """The reference's CSV schema (memory_model.py:230-246); ``measured`` rows
    (from :func:`measure_device`) append the device columns."""
    def emit(fh):
        w = csv.writer(fh, lineterminator="\n")
        if header:
            w.writerow(CSV_COLUMNS + (MEASURED_COLUMNS if measured is not None else []))
        for i, r in enumerate(reports):
            row = [r.sigma, r.optimal_bytes, r.static_p_bytes, r.ggarray_capacity_bytes,
                   r.static_ratio, r.ggarray_ratio]
            if measured is not None:
                m = measured[i]
                row += [m["samples"], m["capacity_mean"], m["mapped_mean"], m["mapped_ratio"],
                        m["mapped_ratio_max"]]
            w.writerow(row)

    if hasattr(out, "write"):
        emit(out)
    else:
        with open(out, "w", encoding="utf-8", newline="") as fh:
            emit(fh)


def measure_device(params: MemoryModelParams, per_sigma: int, shards: int = 32,
                   first_bucket_size: int = 32, element_size: int = DEFAULT_ELEMENT_SIZE,
                   sigma_grid=None, device=None) -> list:
    """For each sigma, draw ``per_sigma`` demands (own generator, seed + 1) and
    realise each on the device: a GGArray of ``shards`` LFVectors grown to the
    even split of the demand (``grow(demand)``, the reservation path every
    insert takes).  Asserts the device capacity equals the closed form and
    reports it with the physically mapped slab bytes."""
    from .sharded_array import GrowableArray
    dt = {1: np.int8, 2: np.int16, 4: np.int32, 8: np.int64}[element_size]
    grid = _sigma_grid() if sigma_grid is None else list(sigma_grid)
    rng = np.random.default_rng(params.seed + 1)
    rows = []
    for sigma in grid:
        d = np.rint(params.base_size * rng.lognormal(mean=params.mu, sigma=sigma, size=per_sigma))
        d = np.maximum(d.astype(np.int64), 1)
        caps, mapped = [], []
        for n in d:
            a = GrowableArray(shards, first_bucket_size, dtype=dt, device=device)
            q, r = divmod(int(n), shards)
            a.grow(int(n), distribution=[q + (s < r) for s in range(shards)])
            ms = a.memory_stats()
            want = int(sharded_capacity_elements([n], shards, first_bucket_size)[0]) * element_size
            if ms["capacity_bytes"] != want:
                raise AssertionError(f"device capacity {ms['capacity_bytes']} != closed form {want}")
            caps.append(ms["capacity_bytes"])
            mapped.append(ms["mapped_bytes"])
            a.close()
        ratio = np.asarray(mapped, np.float64) / (d * element_size)
        rows.append({"sigma": sigma, "samples": int(per_sigma),
                     "capacity_mean": float(np.mean(caps)), "mapped_mean": float(np.mean(mapped)),
                     "mapped_ratio": float(np.mean(mapped) / (d.mean() * element_size)),
                     "mapped_ratio_max": float(ratio.max())})
    return rows
