"""Throughput and phase timeline of hap_permtest_batch on P C2-shaped pairs.
usage: python tools/batch.py [P] [reps]"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

P = int(sys.argv[1]) if len(sys.argv) > 1 else 24
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 5
kind = os.environ.get("HAP_SIZES", "c2")
sizes = ([1000] * P if kind == "c2" else [500] * P if kind == "c5" else
         [int(kind[1:])] * P if kind.startswith("n") else HI.c4_sizes(10000)[:P])  # nNNN: n_x = n_y = NNN
shared = os.environ.get("HAP_SHARED", "0") == "1"
Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=768)
X, Y = torch.from_numpy(Xp).cuda(), torch.from_numpy(Yp).cuda()
ctx = hap.Context(0)
B = 10000


# HAP_ORDER=desc|asc: hand the pairs over in size order (pair_sel) - results are the same
order = os.environ.get("HAP_ORDER", "")
sel = None
if order:
    Ns = np.diff(cnx) + np.diff(cny)
    sel = np.argsort(-Ns if order == "desc" else Ns, kind="stable")


def run():
    return ctx.permtest_batch(X, cnx, Y, cny, B, HI.PERM_SEED, sync=False, shared=shared, pair_sel=sel)


for _ in range(3):
    run()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(reps):
    run()
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"batch P={P}: {ms * 1e3 / P:.1f} us/test, {P * B / ms * 1e3:.3e} perms/s, "
      f"{P / ms * 1e3:.0f} tests/s, mean n {np.mean(sizes):.0f}")

for level in (1, 2):
    hap.hap_profile(ctx.h, level)
    run()
    torch.cuda.synchronize()
    tl = hap.hap_profile_timeline(ctx.h)
    hap.hap_profile(ctx.h, 0)
    dur = {}
    for ph, a, b in tl:
        dur.setdefault(ph.split("@")[0], []).append(b - a)
    print(f"level {level}: span {max(b for _, _, b in tl):.1f} us; " +
          ", ".join(f"{k} med {np.median(v):.1f} us x{len(v)}" for k, v in dur.items()))
    if level == 1:
        for ph, a, b in tl[:40]:
            print(f"   {ph:12s} {a:9.1f} {b:9.1f} {b - a:7.1f}")

# device-clock kernel spans in the unperturbed pipeline
hap.hap_profile_spans(ctx.h, 1)
run()
torch.cuda.synchronize()
sp = hap.hap_profile_spans_read(ctx.h)
hap.hap_profile_spans(ctx.h, 0)
dur = {}
for ph, a, b in sp:
    dur.setdefault(ph.split("@")[0], []).append(b - a)
span = max(b for _, _, b in sp)
print(f"spans: total {span:.1f} us = {span / P:.1f} us/test; " +
      ", ".join(f"{k} med {np.median(v):.1f} us" for k, v in dur.items()))
for ph, a, b in sorted(sp, key=lambda r: r[1])[:36]:
    print(f"   {ph:12s} {a:9.1f} {b:9.1f} {b - a:7.1f}")
out = os.environ.get("HAP_SPANS_OUT")
if out:
    import json
    with open(out, "w") as f:
        json.dump(sp, f)
