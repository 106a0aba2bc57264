"""C5 calibration sweep (BASELINE.json configs[4]) on the
GPU through hap_permtest_batch: R null replicates (equal concentration, E[MRL] = 0.75,
n_x = n_y = 500, d = 768, B = 10^4) for every mean-direction angle theta in {0, 30, 60, 120}
degrees and both cloud families (isotropic vMF; anisotropic = vMF + shared noise x6 on 16
fixed coordinates, hap_inputs.anisotropic_pair), aligned (Householder) vs naive test on
the same permutations.  Reports the rejection rate at alpha in {0.01, 0.05} for the
one-sided "greater" p-value and the two-sided one, with binomial standard errors.

PAPER.md:42-49 (§1, Fig. 1): a mean-direction difference alone should not make the test
reject; the naive test's null distribution is distorted by it.  PAPER.md:445-448 (Limitations):
anisotropy is not captured by a single reflection.

usage: python tools/c5_sweep.py [R] [out.json] [thetas (comma list)] [families (iso,aniso)]
"""
import json
import math
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch

import hap_inputs as HI
import paper_2605_08048_b200 as hap


def run_cell(ctx, R, theta, family, chunk=250):
    cfg = HI.CONFIGS["C5"]
    n, d, B = cfg["n_x"], cfg["d"], cfg["B"]
    spec = HI.PairSpec(n, n, d, HI.kappa_for(d), HI.kappa_for(d), theta, seed=1005)
    make = HI.anisotropic_pair if family == "aniso" else HI.make_pair
    p = {m: {"greater": [], "two_sided": []} for m in ("aligned", "naive")}
    gen_s = gpu_s = 0.0
    for c0 in range(0, R, chunk):
        m = min(chunk, R - c0)
        t0 = time.perf_counter()
        pairs = [make(spec, rep) for rep in range(c0, c0 + m)]
        X = torch.from_numpy(np.concatenate([q[0] for q in pairs])).cuda()
        Y = torch.from_numpy(np.concatenate([q[1] for q in pairs])).cuda()
        cu = np.arange(m + 1, dtype=np.int64) * n
        torch.cuda.synchronize()
        gen_s += time.perf_counter() - t0
        for name, mode in (("aligned", hap.HAP_ALIGN_HOUSEHOLDER), ("naive", hap.HAP_ALIGN_NONE)):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            infos, counts = ctx.permtest_batch(X, cu, Y, cu, B, HI.PERM_SEED, stream_id=c0,
                                               mode=mode, sync=False)
            e1.record()
            e1.synchronize()
            gpu_s += e0.elapsed_time(e1) / 1e3
            assert hap.hap_sync(ctx.h) == 0
            c = counts.cpu().numpy()
            p[name]["greater"] += [hap.hap_pvalue(int(v), B) for v in c[:, 0]]
            p[name]["two_sided"] += [hap.hap_pvalue(int(v), B) for v in c[:, 1]]
    out = {"theta_deg": theta, "family": family, "R": R, "gpu_device_s": gpu_s, "data_gen_s": gen_s}
    for name in ("aligned", "naive"):
        for side in ("greater", "two_sided"):
            arr = np.asarray(p[name][side])
            for a in (0.01, 0.05):
                rate = float(np.mean(arr <= a))
                out[f"{name}/{side}@{a}"] = rate
            out[f"{name}/{side}/mean_p"] = float(arr.mean())
    out["se@0.05"] = math.sqrt(0.05 * 0.95 / R)
    out["se@0.01"] = math.sqrt(0.01 * 0.99 / R)
    return out


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 1000
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    thetas = [float(x) for x in sys.argv[3].split(",")] if len(sys.argv) > 3 else [0, 30, 60, 120]
    fams = sys.argv[4].split(",") if len(sys.argv) > 4 else ["iso", "aniso"]
    ctx = hap.Context(0)
    # warm-up (workspace allocation of the batch lanes)
    X, Y = HI.make_pair(HI.PairSpec(500, 500, 768, HI.kappa_for(768), HI.kappa_for(768), 30.0))
    cu = np.array([0, 500], dtype=np.int64)
    ctx.permtest_batch(torch.from_numpy(X).cuda(), cu, torch.from_numpy(Y).cuda(), cu, 10000,
                       HI.PERM_SEED)
    cells = []
    for fam in fams:
        for th in thetas:
            cell = run_cell(ctx, R, th, fam)
            print(json.dumps(cell), flush=True)
            cells.append(cell)
    out = {"workload": "C5 sweep: R null replicates, n_x=n_y=500, d=768, B=10^4, kappa(r=0.75) "
                       "both groups, mean directions theta apart; aligned vs naive on the same "
                       "permutations; rejection = p <= alpha with p = (1+c)/(B+1)",
           "citation": "PAPER.md:42-49 (Fig. 1 mechanism), :445-448 (anisotropy limitation); "
                       "SURVEY.md App. B", "cells": cells}
    if out_path:
        with open(out_path, "w") as f:
            f.write(json.dumps(out, indent=1) + "\n")


if __name__ == "__main__":
    main()
