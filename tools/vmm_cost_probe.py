"""Cost of the CUDA VMM calls the slab store uses (cuMemCreate / cuMemMap /
cuMemSetAccess / cuMemUnmap / cuMemRelease) per chunk size, via ctypes on
libcuda.  Prints one JSON line per size."""
import ctypes as C
import json
import time

import torch

torch.zeros(1, device="cuda")
cu = C.CDLL("libcuda.so.1")


class Loc(C.Structure):
    _fields_ = [("type", C.c_int), ("id", C.c_int)]


class Prop(C.Structure):
    _fields_ = [("type", C.c_int), ("requestedHandleTypes", C.c_int), ("location", Loc),
                ("win32HandleMetaData", C.c_void_p), ("allocFlags", C.c_ubyte * 8)]


class Access(C.Structure):
    _fields_ = [("location", Loc), ("flags", C.c_int)]


prop = Prop()
prop.type = 1            # CU_MEM_ALLOCATION_TYPE_PINNED
prop.location.type = 1   # CU_MEM_LOCATION_TYPE_DEVICE
prop.location.id = 0
acc = Access()
acc.location.type = 1
acc.location.id = 0
acc.flags = 3            # READWRITE


def ck(r, what):
    if r != 0:
        raise RuntimeError(f"{what} -> {r}")


for mib in (2, 8, 64, 256, 1024, 4096):
    size = mib << 20
    reps = 8 if mib <= 1024 else 4
    va = C.c_uint64()
    ck(cu.cuMemAddressReserve(C.byref(va), C.c_size_t(size * reps), C.c_size_t(size), C.c_uint64(0), C.c_uint64(0)), "reserve")
    t = {"create": 0.0, "map": 0.0, "access": 0.0, "unmap": 0.0, "release": 0.0}
    hs = []
    for i in range(reps):
        h = C.c_uint64()
        t0 = time.perf_counter(); ck(cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_uint64(0)), "create")
        t1 = time.perf_counter(); ck(cu.cuMemMap(C.c_uint64(va.value + i * size), C.c_size_t(size), C.c_size_t(0), h, C.c_uint64(0)), "map")
        t2 = time.perf_counter(); ck(cu.cuMemSetAccess(C.c_uint64(va.value + i * size), C.c_size_t(size), C.byref(acc), C.c_size_t(1)), "access")
        t3 = time.perf_counter()
        t["create"] += t1 - t0; t["map"] += t2 - t1; t["access"] += t3 - t2
        hs.append(h)
    torch.cuda.synchronize()
    for i, h in enumerate(hs):
        t0 = time.perf_counter(); ck(cu.cuMemUnmap(C.c_uint64(va.value + i * size), C.c_size_t(size)), "unmap")
        t1 = time.perf_counter(); ck(cu.cuMemRelease(h), "release")
        t2 = time.perf_counter()
        t["unmap"] += t1 - t0; t["release"] += t2 - t1
    # remap cost with a retained handle (map + access only)
    h = C.c_uint64()
    ck(cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_uint64(0)), "create")
    rm = 0.0
    for i in range(reps):
        t0 = time.perf_counter()
        ck(cu.cuMemMap(C.c_uint64(va.value), C.c_size_t(size), C.c_size_t(0), h, C.c_uint64(0)), "map")
        ck(cu.cuMemSetAccess(C.c_uint64(va.value), C.c_size_t(size), C.byref(acc), C.c_size_t(1)), "access")
        ck(cu.cuMemUnmap(C.c_uint64(va.value), C.c_size_t(size)), "unmap")
        rm += time.perf_counter() - t0
    cu.cuMemRelease(h)
    cu.cuMemAddressFree(va, C.c_size_t(size * reps))
    print(json.dumps({"mib": mib, **{k: round(v / reps * 1e6, 1) for k, v in t.items()},
                      "remap_cycle_us": round(rm / reps * 1e6, 1), "unit": "us per call"}))

# one cuMemSetAccess / cuMemUnmap over a run of separately created mappings?
size, n = 64 << 20, 8
va = C.c_uint64()
ck(cu.cuMemAddressReserve(C.byref(va), C.c_size_t(size * n), C.c_size_t(size), C.c_uint64(0), C.c_uint64(0)), "reserve")
hs = []
t0 = time.perf_counter()
for i in range(n):
    h = C.c_uint64()
    ck(cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_uint64(0)), "create")
    ck(cu.cuMemMap(C.c_uint64(va.value + i * size), C.c_size_t(size), C.c_size_t(0), h, C.c_uint64(0)), "map")
    hs.append(h)
t1 = time.perf_counter()
ra = cu.cuMemSetAccess(va, C.c_size_t(size * n), C.byref(acc), C.c_size_t(1))
t2 = time.perf_counter()
x = torch.empty(0)
ru = cu.cuMemUnmap(va, C.c_size_t(size * n))
t3 = time.perf_counter()
for h in hs:
    cu.cuMemRelease(h)
t4 = time.perf_counter()
print(json.dumps({"run_of": n, "mib": 64, "create_map_us": round((t1 - t0) / n * 1e6, 1),
                  "set_access_rc": ra, "set_access_run_us": round((t2 - t1) * 1e6, 1),
                  "unmap_rc": ru, "unmap_run_us": round((t3 - t2) * 1e6, 1),
                  "release_us": round((t4 - t3) / n * 1e6, 1)}))

# partial unmap of one mapping (half of a 1 GiB handle's range)?
size = 1 << 30
va = C.c_uint64()
ck(cu.cuMemAddressReserve(C.byref(va), C.c_size_t(size), C.c_size_t(size), C.c_uint64(0), C.c_uint64(0)), "reserve")
h = C.c_uint64()
ck(cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_uint64(0)), "create")
ck(cu.cuMemMap(va, C.c_size_t(size), C.c_size_t(0), h, C.c_uint64(0)), "map")
ck(cu.cuMemSetAccess(va, C.c_size_t(size), C.byref(acc), C.c_size_t(1)), "access")
r_half = cu.cuMemUnmap(C.c_uint64(va.value + size // 2), C.c_size_t(size // 2))
r_rest = cu.cuMemUnmap(va, C.c_size_t(size // 2 if r_half == 0 else size))
cu.cuMemRelease(h)
cu.cuMemAddressFree(va, C.c_size_t(size))
# one create of 8 GiB vs 8 x 1 GiB vs 2 GiB x 4 (the config-2 footprint), map + access included
for piece_gib, n in ((8, 1), (4, 2), (1, 8)):
    size = piece_gib << 30
    va = C.c_uint64()
    ck(cu.cuMemAddressReserve(C.byref(va), C.c_size_t(size * n), C.c_size_t(1 << 21), C.c_uint64(0), C.c_uint64(0)), "reserve")
    hs = []
    t0 = time.perf_counter()
    for i in range(n):
        h = C.c_uint64()
        ck(cu.cuMemCreate(C.byref(h), C.c_size_t(size), C.byref(prop), C.c_uint64(0)), "create")
        ck(cu.cuMemMap(C.c_uint64(va.value + i * size), C.c_size_t(size), C.c_size_t(0), h, C.c_uint64(0)), "map")
        hs.append(h)
    ck(cu.cuMemSetAccess(va, C.c_size_t(size * n), C.byref(acc), C.c_size_t(1)), "access")
    t1 = time.perf_counter()
    for i, h in enumerate(hs):
        cu.cuMemUnmap(C.c_uint64(va.value + i * size), C.c_size_t(size))
    t2 = time.perf_counter()
    for h in hs:
        cu.cuMemRelease(h)
    t3 = time.perf_counter()
    cu.cuMemAddressFree(va, C.c_size_t(size * n))
    print(json.dumps({"gib_total": piece_gib * n, "pieces": n, "create_map_access_ms": round((t1 - t0) * 1e3, 2),
                      "unmap_ms": round((t2 - t1) * 1e3, 2), "release_ms": round((t3 - t2) * 1e3, 2)}))
print(json.dumps({"partial_unmap_rc": r_half, "rest_unmap_rc": r_rest}))
