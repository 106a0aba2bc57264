"""NEXT-3 power study on the GPU: R replicates where group X is broader (kappa_X < kappa_Y,
the one-sided alternative of PAPER.md:180) with mean directions theta apart; rejection
rate of the aligned vs the naive test through hap_permtest_batch.  Prints one JSON line.
usage: python tools/power.py [R] [n] [d] [kappa_x] [kappa_y] [theta]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

R = int(sys.argv[1]) if len(sys.argv) > 1 else 200
n = int(sys.argv[2]) if len(sys.argv) > 2 else 500
d = int(sys.argv[3]) if len(sys.argv) > 3 else 768
kx = float(sys.argv[4]) if len(sys.argv) > 4 else 0.97 * HI.kappa_for(d)
ky = float(sys.argv[5]) if len(sys.argv) > 5 else HI.kappa_for(d)
theta = float(sys.argv[6]) if len(sys.argv) > 6 else 30.0
B = 10000
spec = HI.PairSpec(n, n, d, kx, ky, theta, seed=2026)
pairs = [HI.make_pair(spec, rep) for rep in range(R)]
X = torch.from_numpy(np.concatenate([p[0] for p in pairs])).cuda()
Y = torch.from_numpy(np.concatenate([p[1] for p in pairs])).cuda()
cu = np.arange(R + 1, dtype=np.int64) * n
ctx = hap.Context(0)
out = {"workload": f"{R} replicates, n = {n}/{n}, d = {d}, kappa_x = {kx:.2f}, "
                   f"kappa_y = {ky:.2f}, theta = {theta} deg, B = {B}"}
for mode, name in ((0, "aligned"), (1, "naive")):
    res = ctx.permtest_batch(X, cu, Y, cu, B, HI.PERM_SEED, mode=mode)
    p = np.array([r["p_value"] for r in res])
    for a in (0.01, 0.05):
        out[f"power_{name}@{a}"] = float(np.mean(p <= a))
print(json.dumps(out))
