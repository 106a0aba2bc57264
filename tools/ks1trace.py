"""Per-CTA KS1 / KS3 timeline at one streaming shape (development build: -DHAP_EXPERIMENTS;
profiling level 3 stamps).  usage: python tools/ks1trace.py [n] [d]"""
import ctypes
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
L = hap.lib()
L.hap_debug_k1_stamps.argtypes = [ctypes.c_void_p, ctypes.POINTER(ctypes.c_longlong), ctypes.c_int64]
ctx = hap.Context(0)
X, Y = HI.make_pair(HI.PairSpec(n, n, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=5))
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
hap.hap_profile(ctx.h, 3)
G = 4 * torch.cuda.get_device_properties(0).multi_processor_count
buf = np.zeros(8 + 8 * G, dtype=np.int64)
for _ in range(5):
    hap.hap_align(ctx.h, X, Y, 0, ctx.info)
torch.cuda.synchronize()
L.hap_debug_k1_stamps(ctx.h, buf.ctypes.data_as(ctypes.POINTER(ctypes.c_longlong)), buf.size)
st = buf[8:].reshape(G, 8).astype(np.float64)
st = st[st[:, 0] > 0]
t0 = st[:, 0].min()
st = np.where(st > 0, (st - t0) / 1e3, np.nan)
names = ["KS1 entry", "KS1 stage 0", "KS1 loop end", "KS3 loop end", "KS1 exit", "KS3 exit",
         "KS3 P5 done", "KS3 entry"]
print(f"{len(st)} CTAs")
for k, nm in enumerate(names):
    col = st[:, k]
    col = col[~np.isnan(col)]
    if len(col):
        print(f"{nm:12s} n {len(col):4d} min {col.min():7.2f} med {np.median(col):7.2f} max {col.max():7.2f}")
