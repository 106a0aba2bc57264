"""End-to-end legs outside bench.py (so that HAP_LIB_VARIANT may select a library build):
C3 (hap_align from pinned host X, Y + hap_permtest, 4 steps alternating two pairs) and a C2
batch (100 tests from pinned host memory, 3 steps).  Host wall clock, synchronize on both
sides.  usage: python tools/e2e_probe.py"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap
from paper_2605_08048_b200 import parallel

ctx = hap.Context(0)
out = {}
# C3
pool = [HI.config_pair("C3", rep=r) for r in range(2)]
Xh = [torch.from_numpy(X).pin_memory() for X, _ in pool]
Yh = [torch.from_numpy(Y).pin_memory() for _, Y in pool]
B = 100000
infos = torch.zeros((2, hap.INFO_BYTES), dtype=torch.uint8, device="cuda")
cnt = torch.zeros((5, 3), dtype=torch.int64, device="cuda")
parallel.gpu_range_counts(ctx, Xh[0], Yh[0], B, HI.PERM_SEED, 0, 1, cnt[4], infos[0], reduce=False)
torch.cuda.synchronize()
t0 = time.perf_counter()
for k in range(4):
    parallel.gpu_range_counts(ctx, Xh[k % 2], Yh[k % 2], B, HI.PERM_SEED, 0, 1, cnt[k], infos[k % 2],
                              stream_id=k, reduce=False)
torch.cuda.synchronize()
out["c3_e2e_perms_per_s"] = 4 * B / (time.perf_counter() - t0)
t0 = time.perf_counter()
Xd = [x.cuda() for x in Xh]
Yd = [y.cuda() for y in Yh]
torch.cuda.synchronize()
out["c3_h2d_ms_2pairs"] = (time.perf_counter() - t0) * 1e3
out["pinned"] = [bool(x.is_pinned()) for x in Xh + Yh]
# C2 batch: 100 tests (n = 1000 + 1000, d = 768) per call from pinned host memory, 1 warm-up
# call then 5 timed calls enqueued back to back
pairs = [HI.config_pair("C2", rep=r) for r in range(4)]
T = 100
Xp = np.concatenate([pairs[i % 4][0] for i in range(T)])
Yp = np.concatenate([pairs[i % 4][1] for i in range(T)])
cu = np.arange(T + 1, dtype=np.int64) * pairs[0][0].shape[0]
Xh2, Yh2 = torch.from_numpy(Xp).pin_memory(), torch.from_numpy(Yp).pin_memory()
infos2 = torch.zeros((T, hap.INFO_BYTES), dtype=torch.uint8, device="cuda")
cnt2 = torch.zeros((T, 3), dtype=torch.int64, device="cuda")
Bc2 = 10000
for k in range(6):
    if k == 1:
        torch.cuda.synchronize()
        t0 = time.perf_counter()
    cfg = hap.make_cfg(HI.PERM_SEED, Bc2, stream_id=k * T)
    hap.hap_permtest_batch(ctx.h, Xh2, cu, Yh2, cu, 0, cfg, infos2, cnt2)
torch.cuda.synchronize()
out["c2_e2e_perms_per_s"] = 5 * T * Bc2 / (time.perf_counter() - t0)
print(json.dumps(out), flush=True)
