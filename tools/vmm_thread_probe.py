"""Do cuMemCreate / cuMemMap / cuMemSetAccess overlap across host threads?
64 chunks of 64 MiB mapped by 1, 2, 4, 8 threads (ctypes releases the GIL)."""
import ctypes as C, json, threading, time
import torch
torch.zeros(1, device="cuda")
cu = C.CDLL("libcuda.so.1")
class Loc(C.Structure): _fields_ = [("type", C.c_int), ("id", C.c_int)]
class Prop(C.Structure): _fields_ = [("type", C.c_int), ("requestedHandleTypes", C.c_int), ("location", Loc), ("win32HandleMetaData", C.c_void_p), ("allocFlags", C.c_ubyte * 8)]
class Acc(C.Structure): _fields_ = [("location", Loc), ("flags", C.c_int)]
prop = Prop(); prop.type = 1; prop.location.type = 1; prop.location.id = 0
acc = Acc(); acc.location.type = 1; acc.location.id = 0; acc.flags = 3
ctx = C.c_void_p()
cu.cuCtxGetCurrent(C.byref(ctx))
N, SZ = 64, 64 << 20
va = C.c_uint64()
assert cu.cuMemAddressReserve(C.byref(va), C.c_size_t(N * SZ), C.c_size_t(SZ), C.c_uint64(0), C.c_uint64(0)) == 0


def work(ids, hs):
    cu.cuCtxSetCurrent(ctx)
    for i in ids:
        h = C.c_uint64()
        assert cu.cuMemCreate(C.byref(h), C.c_size_t(SZ), C.byref(prop), C.c_uint64(0)) == 0
        assert cu.cuMemMap(C.c_uint64(va.value + i * SZ), C.c_size_t(SZ), C.c_size_t(0), h, C.c_uint64(0)) == 0
        assert cu.cuMemSetAccess(C.c_uint64(va.value + i * SZ), C.c_size_t(SZ), C.byref(acc), C.c_size_t(1)) == 0
        hs[i] = h


def unwork(ids, hs):
    cu.cuCtxSetCurrent(ctx)
    for i in ids:
        cu.cuMemUnmap(C.c_uint64(va.value + i * SZ), C.c_size_t(SZ))
        cu.cuMemRelease(hs[i])


for order in ((1, 2, 4, 8, 16), (16, 8, 4, 2, 1), (1, 8, 1, 8)):
    for T in order:
        hs = [None] * N
        th = [threading.Thread(target=work, args=(range(t, N, T), hs)) for t in range(T)]
        t0 = time.perf_counter()
        for x in th: x.start()
        for x in th: x.join()
        tm = time.perf_counter() - t0
        th = [threading.Thread(target=unwork, args=(range(t, N, T), hs)) for t in range(T)]
        t0 = time.perf_counter()
        for x in th: x.start()
        for x in th: x.join()
        tu = time.perf_counter() - t0
        print(json.dumps({"threads": T, "map_ms": round(tm * 1e3, 2), "unmap_ms": round(tu * 1e3, 2),
                          "per_chunk_map_us": round(tm / N * 1e6, 1)}), flush=True)
