"""K3 CTA entry / piece / exit times (exp bit 16 stamps) of the last lane-0 launch of a
C2 batch in the two-lane pipeline: do CTAs start late beside the generator?"""
import ctypes
import os
import sys

os.environ["HAP_K3_EXPERIMENT"] = "16"
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

L = hap.lib()
L.hap_debug_k3_stamps.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int64]
P = int(sys.argv[1]) if len(sys.argv) > 1 else 24
Xp, cnx, Yp, cny = HI.varlen_batch([1000] * P, d=768)
X, Y = torch.from_numpy(Xp).cuda(), torch.from_numpy(Yp).cuda()
ctx = hap.Context(0)
for _ in range(3):
    ctx.permtest_batch(X, cnx, Y, cny, 10000, HI.PERM_SEED)
torch.cuda.synchronize()
buf = np.zeros(148 * 64, dtype=np.int64)
L.hap_debug_k3_stamps(ctx.h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), buf.size)
st = buf.reshape(148, 8, 8).astype(np.float64)
entry = st[:, 7, 0]
t0 = entry[entry > 0].min()
st = np.where(st > 0, (st - t0) / 1e3, np.nan)
entry, exit_ = st[:, 7, 0], st[:, 7, 1]
print(f"entry: min {np.nanmin(entry):.1f} med {np.nanmedian(entry):.1f} p90 {np.nanpercentile(entry, 90):.1f} max {np.nanmax(entry):.1f} us")
print(f"exit : min {np.nanmin(exit_):.1f} med {np.nanmedian(exit_):.1f} max {np.nanmax(exit_):.1f} us")
first_mma = st[::2, 0, 2]
last_mma = np.nanmax(st[::2, :7, 3], axis=1)
print(f"leader first MMA: min {np.nanmin(first_mma):.1f} med {np.nanmedian(first_mma):.1f} max {np.nanmax(first_mma):.1f}")
print(f"leader last MMA issue: min {np.nanmin(last_mma):.1f} med {np.nanmedian(last_mma):.1f} max {np.nanmax(last_mma):.1f}")
