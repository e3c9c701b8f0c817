"""How much GPU virtual address space can one process reserve (cuMemAddressReserve)?"""
import ctypes as C, json
import torch
torch.cuda.init(); torch.zeros(1, device="cuda")
cu = C.CDLL("libcuda.so.1")
res, got = [], []
for tib in [1, 2, 4, 8, 16, 32, 64, 128]:
    p = C.c_uint64(0)
    r = cu.cuMemAddressReserve(C.byref(p), C.c_size_t(tib << 40), C.c_size_t(2 << 20), C.c_uint64(0), C.c_uint64(0))
    res.append({"tib": tib, "rc": r, "ptr": hex(p.value)})
    if r == 0:
        got.append((p.value, tib << 40))
tot = sum(s for _, s in got) >> 40
for p, s in got:
    cu.cuMemAddressFree(C.c_uint64(p), C.c_size_t(s))
print(json.dumps({"single": res, "cumulative_tib": tot}))
