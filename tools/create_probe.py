"""Where array construction / destruction time goes (S=512 int32)."""
import ctypes as C, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_2209_00103_b200 as gg
from paper_2209_00103_b200 import _lib as L

torch.zeros(1, device="cuda")
res = {}
def med(f, n=15):
    ts = []
    for _ in range(n):
        t0 = time.perf_counter(); f(); ts.append(time.perf_counter() - t0)
    return round(1e3 * float(np.median(ts[2:])), 3)
hs = []
def c():
    h = C.c_void_p(); L.check(L.lib.gg_create(0, 512, 32, 4, 58, 0, C.byref(h))); hs.append(h)
res["gg_create_ms"] = med(c)
def d():
    L.lib.gg_destroy(hs.pop())
res["gg_destroy_ms"] = med(d)
objs = []
res["GrowableArray_ms"] = med(lambda: objs.append(gg.GrowableArray(512, 32, dtype=np.int32)))
res["close_ms"] = med(lambda: objs.pop().close())
vals = np.arange(1 << 20, dtype=np.int32)
b = gg.split_batches(vals, 512)
a = gg.GrowableArray(512, 32, dtype=np.int32)
res["pack_ms"] = med(lambda: a._pack(b))
print(json.dumps(res))
