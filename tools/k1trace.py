"""Per-CTA K1 timeline (profiling level 3 stamps) for a C2 pair."""
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
name = sys.argv[1] if len(sys.argv) > 1 else "C2"
X, Y = HI.config_pair(name)
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
hap.hap_profile(ctx.h, 3)
for _ in range(5):
    hap.hap_align(ctx.h, X, Y, 0, ctx.info)
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
    col = col[col > -1e6]
    print(f"{n:7s} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}  argmax {int(np.argmax(st[:, k]))}")
