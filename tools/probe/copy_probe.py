"""Run tools/probe/copy_probe.cu variants on 2^30 int32 (4 GiB -> 4 GiB)."""
import ctypes as C, json, os, subprocess, sys
import torch
here = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(here, "copy_probe.so")
lib = C.CDLL(so)
n = 1 << 32
x = torch.empty(n, dtype=torch.uint8, device="cuda"); y = torch.empty_like(x)
x.random_()


def t(fn, reps=10):
    fn(); torch.cuda.synchronize()
    best = 1e9
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
        e0.record(); fn(); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best


ms = t(lambda: y.copy_(x))
print(json.dumps({"v": "torch copy_", "gbs": round(2 * n / ms / 1e6, 1)}), flush=True)
for v, thr, arg in [(0, 128, 0), (0, 256, 0), (1, 256, 0), (2, 256, 0), (3, 256, 0), (4, 256, 0), (5, 256, 0), (6, 128, 0),
                    (10, 256, 32768), (11, 256, 32768), (11, 256, 65536), (12, 256, 65536), (20, 32, 1), (20, 32, 2), (21, 32, 2), (22, 32, 1), (21, 32, 1)]:
    y.zero_()
    ms = t(lambda: lib.probe_copy(C.c_void_p(y.data_ptr()), C.c_void_p(x.data_ptr()), C.c_uint64(n), v, thr, arg))
    ok = bool(torch.equal(x, y))
    print(json.dumps({"v": v, "threads": thr, "arg": arg, "gbs": round(2 * n / ms / 1e6, 1), "ok": ok}), flush=True)
