"""Plane form vs Gram form of the mask-GEMM:
device time per test (hap_align + hap_permtest, CUDA events, median of 5) at N << d shapes,
both forms on the same input, and the form the library picks by itself.
usage: python tools/gram_bench.py [out.json]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

SHAPES = [(64, 64, 768, 10000), (64, 64, 768, 100000), (100, 100, 4096, 10000),
          (100, 100, 4096, 100000), (250, 250, 4096, 100000), (500, 500, 4096, 100000),
          (150, 150, 1536, 100000), (1000, 1000, 4096, 100000)]
ctx = hap.Context(0)
rows = []
for n_x, n_y, d, B in SHAPES:
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=d + n_x))
    X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    row = dict(n_x=n_x, n_y=n_y, d=d, B=B, n_pad=-(-(n_x + n_y) // 64) * 64)
    for name, gram in (("planes", False), ("gram", True), ("auto", None)):
        r = ctx.permtest_pair(X, Y, B, HI.PERM_SEED, stream_id=1, gram=gram)  # warm-up
        ts = []
        for k in range(5):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            ctx.permtest_pair(X, Y, B, HI.PERM_SEED, stream_id=1, gram=gram, sync=False)
            e1.record()
            e1.synchronize()
            ts.append(e0.elapsed_time(e1))
        row[name + "_ms"] = float(np.median(ts))
        row[name + "_exceed_ge"] = r["exceed_ge"]
        row[name + "_flagged"] = r["flagged"]
    row["speedup"] = row["planes_ms"] / row["gram_ms"]
    row["auto_is_gram"] = abs(row["auto_ms"] - row["gram_ms"]) < abs(row["auto_ms"] - row["planes_ms"])
    print(json.dumps(row), flush=True)
    rows.append(row)
if len(sys.argv) > 1:
    with open(sys.argv[1], "w") as f:
        json.dump({"tool": "tools/gram_bench.py", "gpu": torch.cuda.get_device_name(), "rows": rows}, f, indent=1)
