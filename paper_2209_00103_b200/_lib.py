"""ctypes binding of the C ABI in include/ggarray.h (``_ggarray.so``, built in-tree).

There is no fallback: if the library is missing the import fails loudly, and
every GPU entry point fails if no CUDA device is present.
"""

from __future__ import annotations

import ctypes as C
import os

import numpy as np

from .errors import CapacityError

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("GG_LIB_PATH") or os.path.join(_HERE, "_ggarray.so")   # override: A/B builds (tools/)

if not os.path.exists(LIB_PATH):
    raise ImportError(
        f"{LIB_PATH} is missing: build it with `python build_ext.py` or "
        "`python -c 'import __graft_entry__ as g; g.build()'` (nvcc, sm_100a)")

lib = C.CDLL(LIB_PATH)

GG_OK, GG_EVALUE, GG_ECAPACITY, GG_EINDEX, GG_ENOMEM, GG_ECUDA, GG_EUNPUBLISHED, GG_EPARTIAL = range(8)
GG_RW_PER_SHARD, GG_RW_GLOBAL, GG_RW_FUSED = 0, 1, 2
GG_ALGO_ATOMIC, GG_ALGO_WARP, GG_ALGO_BLOCK, GG_ALGO_BATCH = 0, 1, 2, 3
GG_F_COMMIT, GG_F_UNFUSED = 1, 2

# numpy dtype -> GG dtype code (include/ggarray.h)
DTYPE_CODES = {
    np.dtype(np.int8): 0, np.dtype(np.uint8): 1, np.dtype(np.int16): 2, np.dtype(np.uint16): 3,
    np.dtype(np.int32): 4, np.dtype(np.uint32): 5, np.dtype(np.int64): 6, np.dtype(np.uint64): 7,
    np.dtype(np.float16): 8, np.dtype(np.float32): 9, np.dtype(np.float64): 10,
}

HOOK = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint64)

P = C.c_void_p
U32, U64, I32, I64 = C.c_uint32, C.c_uint64, C.c_int32, C.c_int64
PU64, PI32, PI64, PU32 = C.POINTER(U64), C.POINTER(I32), C.POINTER(I64), C.POINTER(U32)

_SIGS = {
    "gg_last_error": ([], C.c_char_p),
    "gg_version": ([], C.c_int),
    "gg_init": ([C.c_int], C.c_int),
    "gg_kernel_launches": ([], U64),
    "gg_device_sms": ([C.c_int, PI32], C.c_int),
    "gg_create": ([C.c_int, U32, U32, U32, U32, U64, C.POINTER(P)], C.c_int),
    "gg_destroy": ([P], C.c_int),
    "gg_set_alloc_hook": ([P, HOOK, P], C.c_int),
    "gg_set_arena_limit": ([P, U64], C.c_int),
    "gg_insert": ([P, P, PU64, PU64, PI32, P], C.c_int),
    "gg_insert_duplicate": ([P, PI32, P], C.c_int),
    "gg_insert_ex": ([P, P, PU64, PU64, U32, PI32, P], C.c_int),
    "gg_insert_ex2": ([P, P, PU64, PU64, U32, PI32, PU64, P], C.c_int),
    "gg_insert_duplicate_ex": ([P, U32, PI32, P], C.c_int),
    "gg_insert_lanes": ([P, P, P, PU64, U64, PI32, P], C.c_int),
    "gg_commit": ([P, P], C.c_int),
    "gg_reserve": ([P, PU64, PI64, P], C.c_int),
    "gg_new_bucket": ([P, U32, U32, PI32, P], C.c_int),
    "gg_fetch_add": ([P, U32, U64, PU64, P], C.c_int),
    "gg_shrink": ([P, PU64, P], C.c_int),
    "gg_shrink_ex": ([P, PU64, U64, P], C.c_int),
    "gg_trim": ([P], C.c_int),
    "gg_rw_add": ([P, P, U32, I32, P], C.c_int),
    "gg_device_view_bytes": ([], U64),
    "gg_device_view_get": ([P, PU64, P, U64], C.c_int),
    "gg_device_view_sync": ([P, PI32, P], C.c_int),
    "gg_push_if": ([P, P, P, U64, I32, U32, PI32, P], C.c_int),
    "gg_flatten": ([P, P, P], C.c_int),
    "gg_flatten_range": ([P, U64, U64, P, P], C.c_int),
    "gg_gather": ([P, P, U64, P, P], C.c_int),
    "gg_gather_checked": ([P, P, U64, P, P], C.c_int),
    "gg_scatter_checked": ([P, P, U64, P, P], C.c_int),
    "gg_scatter": ([P, P, U64, P, P], C.c_int),
    "gg_get": ([P, U32, U64, P, P], C.c_int),
    "gg_set": ([P, U32, U64, P, P], C.c_int),
    "gg_info": ([P, PU32], C.c_int),
    "gg_capture_mode": ([P, I32], C.c_int),
    "gg_flush": ([P], C.c_int),
    "gg_capture_end": ([P, P], C.c_int),
    "gg_set_fuse": ([C.c_int32], C.c_int),
    "gg_set_tuning": ([I32, I32, U32, U32], C.c_int),
    "gg_set_pdl": ([C.c_int32], C.c_int),
    "gg_set_defer": ([C.c_int32], C.c_int),
    "gg_set_batch_backing": ([C.c_int32], C.c_int),
    "gg_capture_release": ([P], C.c_int),
    "gg_summary": ([P, PU64], C.c_int),
    "gg_host_state": ([P, PU64, PU64, PU64, PU64, PU64], C.c_int),
    "gg_device_state": ([P, PU64, PU64, PU64, PU64, PU64, P], C.c_int),
    "gg_bucket_ptrs": ([P, PU64, P], C.c_int),
    "gg_mem_stats": ([P, PU64, P], C.c_int),
    "gg_prefix_copy": ([P, P, P], C.c_int),
    "gg_slab_stats": ([P, PU64], C.c_int),
    "gg_pool_stats": ([C.c_int, PU64], C.c_int),
    "gg_pool_trim": ([C.c_int], C.c_int),
    "gg_reclaim": ([I32], C.c_int),
    "gg_settle": ([P], C.c_int),
    "gg_flat_insert": ([P, U64, P, P, U64, U32, I32, P], C.c_int),
    "gg_flat_add": ([P, U64, U32, P, U32, I32, P], C.c_int),
    "gg_flat_append": ([P, U64, P, U64, P, U64, U32, P], C.c_int),
    "gg_ipc_alloc": ([U64, C.POINTER(C.c_void_p)], C.c_int),
    "gg_ipc_free": ([P], C.c_int),
    "gg_ipc_handle_bytes": ([], C.c_int),
    "gg_ipc_get_handle": ([P, P], C.c_int),
    "gg_ipc_open": ([P, C.POINTER(C.c_void_p)], C.c_int),
    "gg_ipc_close": ([P], C.c_int),
    "gg_buf_alloc": ([U64, P, C.POINTER(P)], C.c_int),
    "gg_buf_free": ([P, P], C.c_int),
    "gg_buf_copy": ([P, P, U64, P], C.c_int),
    "gg_vmm_create": ([C.c_int, U64, C.POINTER(P)], C.c_int),
    "gg_vmm_ensure": ([P, U64], C.c_int),
    "gg_vmm_info": ([P, PU64, PU64, PU64], C.c_int),
    "gg_vmm_destroy": ([P], C.c_int),
}

for _name, (_args, _res) in _SIGS.items():
    _fn = getattr(lib, _name)
    _fn.argtypes = _args
    _fn.restype = _res


def last_error() -> str:
    return (lib.gg_last_error() or b"").decode(errors="replace")


def check(rc: int, what: str = "") -> None:
    """Map a C-ABI return code to the reference's exception types (errors.py)."""
    if rc == GG_OK:
        return
    msg = f"{what}: {last_error()}" if what else last_error()
    if rc == GG_EVALUE:
        raise ValueError(msg)
    if rc == GG_ECAPACITY:
        raise CapacityError(msg)
    if rc == GG_EINDEX:
        raise IndexError(msg)
    if rc == GG_ENOMEM:
        raise MemoryError(msg)
    if rc == GG_EUNPUBLISHED:
        raise RuntimeError(msg)
    raise RuntimeError(f"CUDA failure in {what}: {last_error()}")


def u64_array(a) -> np.ndarray:
    return np.ascontiguousarray(np.asarray(a, dtype=np.uint64))


def ptr(a: np.ndarray, ctype=U64):
    return a.ctypes.data_as(C.POINTER(ctype))


def stream_handle(device_index: int) -> int:
    """Raw cudaStream_t of torch's current stream on ``device_index``."""
    import torch
    try:
        return torch._C._cuda_getCurrentRawStream(device_index)
    except AttributeError:  # older torch
        return torch.cuda.current_stream(device_index).cuda_stream


if os.environ.get("GG_PDL") == "0":        # A/B switch for programmatic dependent launch
    lib.gg_set_pdl(0)
if os.environ.get("GG_DEFER") == "0":      # A/B switch for the deferred metadata pass
    lib.gg_set_defer(0)
if os.environ.get("GG_FUSE_META") == "0":  # A/B switch for the metadata CTA inside the planned walk
    lib.gg_set_fuse(0)
