"""Device-clock kernel spans of one C3 test (n = 5000/5000, d = 4096, B = 10^5) through
hap_align + hap_permtest: does the generator (K2) of block i+1 overlap the mask-GEMM (K3) of
block i?  usage: python tools/c3_spans.py [B]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

B = int(sys.argv[1]) if len(sys.argv) > 1 else 100000
block = int(sys.argv[2]) if len(sys.argv) > 2 else 0  # permutations per block (0 = library default)
X, Y = HI.config_pair("C3")
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
ctx = hap.Context(0)
for _ in range(2):
    ctx.permtest_pair(X, Y, B, HI.PERM_SEED, stream_id=1, block=block)
hap.hap_profile_spans(ctx.h, 1)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
r = ctx.permtest_pair(X, Y, B, HI.PERM_SEED, stream_id=2, sync=False, block=block)
e1.record()
e1.synchronize()
spans = hap.hap_profile_spans_read(ctx.h)
tot = {}
for ph, a, b in spans:
    print(f"{ph:12s} {a:10.1f} {b:10.1f}  dur {b - a:8.1f}")
    tot[ph] = tot.get(ph, 0.0) + (b - a)
print("sum of spans per phase (us):", {k: round(v, 1) for k, v in tot.items()})
print("block", block, "test (events) ms:", e0.elapsed_time(e1))
