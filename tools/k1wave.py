"""Per-CTA K1 phase stamps (profiling level 3) of the first wave of a C2 batch (3 pairs)."""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

L = hap.lib()
L.hap_debug_k1_stamps.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int64]
ctx = hap.Context(0)
P = int(sys.argv[1]) if len(sys.argv) > 1 else 3
Xp, cnx, Yp, cny = HI.varlen_batch([1000] * P, d=768)
X, Y = torch.from_numpy(Xp).cuda(), torch.from_numpy(Yp).cuda()
for _ in range(3):
    ctx.permtest_batch(X, cnx, Y, cny, 10000, HI.PERM_SEED)
hap.hap_profile(ctx.h, 3)
ctx.permtest_batch(X, cnx, Y, cny, 10000, HI.PERM_SEED)
torch.cuda.synchronize()
G = torch.cuda.get_device_properties(0).multi_processor_count
buf = np.zeros(8 + 8 * G, dtype=np.int64)
L.hap_debug_k1_stamps(ctx.h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), buf.size)
st = buf[8:].reshape(G, 8).astype(np.float64)
st = st[st[:, 0] > 0]  # CTAs of this launch (the grid is no larger than the item count)
t0 = st[:, 0].min()
st = (st - t0) / 1e3
names = ["entry", "P1done", "bar1", "P2done", "P3done", "P4coef", "P4done", "exit"]
for k, n in enumerate(names):
    col = st[:, k]
    print(f"{n:7s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
