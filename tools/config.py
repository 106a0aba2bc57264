"""Single-test throughput of a BASELINE config on one GPU (C1, C2, C3) through
hap_align + hap_permtest: device time per test (CUDA events), perms/s, and the K3
algorithmic TFLOP/s from a serialised profiling pass.  usage: python tools/config.py C3 [B]"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
cfg = HI.CONFIGS[name]
B = int(sys.argv[2]) if len(sys.argv) > 2 else cfg["B"]
block = int(os.environ.get("HAP_BLOCK", "0"))  # permutations per launch (0 = library default)
X, Y = HI.config_pair(name)
X, Y = torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda()
ctx = hap.Context(0)
res = ctx.permtest_pair(X, Y, B, HI.PERM_SEED, block=block)  # warm-up (allocations)
reps = 3
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for k in range(reps):
    ctx.permtest_pair(X, Y, B, HI.PERM_SEED, stream_id=k, sync=False, block=block)
e1.record()
e1.synchronize()
ms = e0.elapsed_time(e1) / reps
hap.hap_profile(ctx.h, 2)
ctx.permtest_pair(X, Y, B, HI.PERM_SEED, block=block)
phase_ms, phase_n = hap.hap_profile_read(ctx.h, reset=True)
hap.hap_profile(ctx.h, 0)
N, d = cfg["n_x"] + cfg["n_y"], cfg["d"]
k3_s = phase_ms["maskgemm"] / 1e3
print(json.dumps({"config": name, "block": block, "n_x": cfg["n_x"], "n_y": cfg["n_y"], "d": d, "B": B,
                  "ms_per_test": ms, "perms_per_s": B / (ms / 1e3),
                  "phase_ms_serialised": phase_ms, "launches": phase_n,
                  "k3_algorithmic_tflops": 2.0 * N * d * B / k3_s / 1e12,
                  "k3_issued_tflops": 4.0 * (-(-N // 64) * 64) * (-(-d // 32) * 32) * B / k3_s / 1e12,
                  "p_value": res["p_value"], "t_obs": res["t_obs"]}))
