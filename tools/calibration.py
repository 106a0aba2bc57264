"""C5 (BASELINE.json configs[4]): Type-I calibration study on the GPU - R null replicates of
vMF clouds with equal concentration and mean directions theta apart (n = 500/500, d = 768,
B = 10^4), aligned vs naive, through hap_permtest_batch.  Prints one JSON line.
usage: python tools/calibration.py [R] [chunk]"""
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

R = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 100
cfg = HI.CONFIGS["C5"]
n, d, B = cfg["n_x"], cfg["d"], cfg["B"]
theta = float(os.environ.get("HAP_THETA", "30"))
aniso = os.environ.get("HAP_ANISO", "0") == "1"  # SURVEY App. B anisotropic variant
ctx = hap.Context(0)
pv = {0: [], 1: []}
gpu_s = 0.0
gen_s = 0.0
for c0 in range(0, R, chunk):
    m = min(chunk, R - c0)
    t0 = time.perf_counter()
    spec = HI.PairSpec(n, n, d, HI.kappa_for(d), HI.kappa_for(d), theta, seed=1005)
    make = HI.anisotropic_pair if aniso else HI.make_pair
    pairs = [make(spec, rep) for rep in range(c0, c0 + m)]
    X = torch.from_numpy(np.concatenate([p[0] for p in pairs])).cuda()
    Y = torch.from_numpy(np.concatenate([p[1] for p in pairs])).cuda()
    cu = np.arange(m + 1, dtype=np.int64) * n
    torch.cuda.synchronize()
    gen_s += time.perf_counter() - t0
    for mode in (0, 1):
        if c0 == 0:  # warm-up: workspace allocation of the batch lanes
            ctx.permtest_batch(X, cu, Y, cu, B, HI.PERM_SEED, stream_id=c0, mode=mode)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        infos, counts = ctx.permtest_batch(X, cu, Y, cu, B, HI.PERM_SEED, stream_id=c0, mode=mode,
                                           sync=False)
        e1.record()
        e1.synchronize()
        gpu_s += e0.elapsed_time(e1) / 1e3
        pv[mode] += [hap.hap_pvalue(int(c), B) for c in counts[:, 0].cpu().tolist()]
out = {"workload": f"C5: {R} null replicates, n_x = n_y = {n}, d = {d}, B = {B}, "
                   f"kappa(r=0.75) both, mean directions {theta} deg apart"
                   + (", anisotropic noise (SURVEY App. B)" if aniso else ""),
       "tests": 2 * R, "gpu_device_s": gpu_s, "timer": "CUDA events around each batch call", "tests_per_s": 2 * R / gpu_s,
       "perms_per_s": 2 * R * B / gpu_s, "data_gen_s": gen_s}
for a in (0.01, 0.05, 0.10):
    out[f"type1_aligned@{a}"] = float(np.mean(np.array(pv[0]) <= a))
    out[f"type1_naive@{a}"] = float(np.mean(np.array(pv[1]) <= a))
print(json.dumps(out))
