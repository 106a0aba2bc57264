"""K1 at one shape, a few hap_align calls (for ncu launch lists / full captures).
usage: python tools/k1_ncu.py [n] [d] [calls]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

n = int(sys.argv[1]) if len(sys.argv) > 1 else 5000
d = int(sys.argv[2]) if len(sys.argv) > 2 else 4096
calls = int(sys.argv[3]) if len(sys.argv) > 3 else 3
X, Y = HI.make_pair(HI.PairSpec(n, n, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=5))
Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
ctx = hap.Context(0)
for _ in range(calls):
    hap.hap_align(ctx.h, Xd, Yd, 0, ctx.info)
assert hap.hap_sync(ctx.h) == 0
print("ok", hap.decode_info(ctx.info).t_obs)
