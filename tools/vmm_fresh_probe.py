"""Physical allocation cost on a fresh process: create+map+access 8 GiB as
64 MiB / 256 MiB / 1 GiB handles, release, and again (is the first touch
of device memory what costs?)."""
import ctypes as C, json, time
import torch
torch.zeros(1, device="cuda")
cu = C.CDLL("libcuda.so.1")
class Loc(C.Structure): _fields_ = [("type", C.c_int), ("id", C.c_int)]
class Prop(C.Structure): _fields_ = [("type", C.c_int), ("requestedHandleTypes", C.c_int), ("location", Loc), ("win32HandleMetaData", C.c_void_p), ("allocFlags", C.c_ubyte * 8)]
class Acc(C.Structure): _fields_ = [("location", Loc), ("flags", C.c_int)]
prop = Prop(); prop.type = 1; prop.location.type = 1; prop.location.id = 0
acc = Acc(); acc.location.type = 1; acc.location.id = 0; acc.flags = 3
TOT = 8 << 30
va = C.c_uint64()
assert cu.cuMemAddressReserve(C.byref(va), C.c_size_t(TOT), C.c_size_t(1 << 30), C.c_uint64(0), C.c_uint64(0)) == 0
def run(chunk):
    hs = []
    t0 = time.perf_counter(); tc = 0.0
    for i in range(TOT // chunk):
        h = C.c_uint64()
        a = time.perf_counter()
        assert cu.cuMemCreate(C.byref(h), C.c_size_t(chunk), C.byref(prop), C.c_uint64(0)) == 0
        tc += time.perf_counter() - a
        assert cu.cuMemMap(C.c_uint64(va.value + i * chunk), C.c_size_t(chunk), C.c_size_t(0), h, C.c_uint64(0)) == 0
        assert cu.cuMemSetAccess(C.c_uint64(va.value + i * chunk), C.c_size_t(chunk), C.byref(acc), C.c_size_t(1)) == 0
        hs.append(h)
    tm = time.perf_counter() - t0
    t1 = time.perf_counter()
    for i, h in enumerate(hs):
        cu.cuMemUnmap(C.c_uint64(va.value + i * chunk), C.c_size_t(chunk)); cu.cuMemRelease(h)
    tr = time.perf_counter() - t1
    return {"chunk_mib": chunk >> 20, "map_total_ms": round(tm * 1e3, 1), "create_ms": round(tc * 1e3, 1), "release_ms": round(tr * 1e3, 1)}
out = [run(64 << 20), run(64 << 20), run(1 << 30), run(256 << 20), run(64 << 20)]
print(json.dumps(out))
