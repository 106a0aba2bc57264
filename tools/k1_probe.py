# time K1 alone (fused vs streaming) at several sizes through hap_align (events)
import sys, os, json
sys.path.insert(0, os.getcwd())
import numpy as np, torch
import hap_inputs as HI
import paper_2605_08048_b200 as hap
ctx = hap.Context(0)
res = []
for (n, d) in [(5000, 4096), (2100, 2048), (1024, 4096), (4000, 1024), (5000, 768), (2600, 1536)]:
    X, Y = HI.make_pair(HI.PairSpec(n, n, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=5))
    Xd, Yd = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
    for _ in range(3):
        hap.hap_align(ctx.h, Xd, Yd, 0, ctx.info)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    K = 20
    e0.record()
    for _ in range(K):
        hap.hap_align(ctx.h, Xd, Yd, 0, ctx.info)
    e1.record(); e1.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / K
    N = 2 * n; npad = -(-N // 64) * 64; dpad = -(-d // 32) * 32
    byt = 4 * N * d + 4 * npad * dpad
    st = hap.hap_sync(ctx.h)
    info = hap.decode_info(ctx.info)
    r = dict(n=n, d=d, us=us, gbs=byt / us / 1e3, stream=bool(hap.lib() and npad * d >= 8 << 20), status=st, r_x=info.r_x)
    print(json.dumps(r), flush=True)
    res.append(r)
json.dump(res, open("gpurun_out/k1s_probe.json", "w"), indent=1)
