"""Small end-to-end cases for compute-sanitizer (memcheck / racecheck / synccheck): C1 and a
reduced C2 (B = 2000) through hap_permtest with both K3 modes (cta_group::1 and ::2), a
batch of three varlen pairs through hap_permtest_batch, and a streaming-alignment pair.
usage: compute-sanitizer --tool <t> python tools/sanitize_case.py [quick]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

quick = len(sys.argv) > 1 and sys.argv[1] == "quick"
ctx = hap.Context(0)
X, Y = HI.config_pair("C1")
for pm in (1, 2):
    r = ctx.permtest_pair(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), 1000, HI.PERM_SEED,
                          stream_id=1, pair_mode=pm)
    print("C1 pair_mode", pm, r["exceed_ge"], r["p_value"])
if not quick:
    X, Y = HI.config_pair("C2")
    for pm in (1, 2):
        r = ctx.permtest_pair(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), 2000,
                              HI.PERM_SEED, stream_id=2, pair_mode=pm)
        print("C2/B=2000 pair_mode", pm, r["exceed_ge"], r["p_value"])
Xp, cnx, Yp, cny = HI.varlen_batch([70, 300, 41], d=768)
out = ctx.permtest_batch(torch.from_numpy(Xp).cuda(), cnx, torch.from_numpy(Yp).cuda(), cny, 700,
                         HI.PERM_SEED, stream_id=3)
print("batch", [o["exceed_ge"] for o in out])
if not quick:
    X, Y = HI.make_pair(HI.PairSpec(1024, 1024, 4096, HI.kappa_for(4096), HI.kappa_for(4096), 30.0, seed=9))
    r = ctx.permtest_pair(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), 300, HI.PERM_SEED)
    print("stream-aligned pair", r["exceed_ge"], r["p_value"])
assert hap.hap_sync(ctx.h) == 0
ctx.close()
print("sanitize case ok")
