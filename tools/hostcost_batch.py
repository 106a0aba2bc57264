"""Host-side cost of one hap_permtest_batch call (C2 chunk of 24 tests, inputs in pinned
host memory): the API returns after enqueueing; compare with the device time of the chunk."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

P = 24
Xp, cnx, Yp, cny = HI.varlen_batch([1000] * P, d=768)
Xh, Yh = torch.from_numpy(Xp).pin_memory(), torch.from_numpy(Yp).pin_memory()
ctx = hap.Context(0)
infos = torch.zeros((P, hap.INFO_BYTES), dtype=torch.uint8, device="cuda")
counts = torch.zeros((P, 3), dtype=torch.int64, device="cuda")
cfg = hap.make_cfg(HI.PERM_SEED, 10000)
st = torch.cuda.current_stream()
for _ in range(3):
    hap.hap_permtest_batch(ctx.h, Xh, cnx, Yh, cny, 0, cfg, infos, counts, stream=st)
torch.cuda.synchronize()
host = []
t0 = time.perf_counter()
for _ in range(10):
    a = time.perf_counter()
    hap.hap_permtest_batch(ctx.h, Xh, cnx, Yh, cny, 0, cfg, infos, counts, stream=st)
    host.append(time.perf_counter() - a)
torch.cuda.synchronize()
wall = (time.perf_counter() - t0) / 10
print(f"host per call {1e3*np.median(host):.2f} ms (max {1e3*max(host):.2f}), wall per call {1e3*wall:.2f} ms, "
      f"PCIe-bound estimate {P*6.144e6/55e9*1e3:.2f} ms")
