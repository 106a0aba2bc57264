"""Same-word split-half sanity check (§3.1 "Fixed-space
permutation after alignment", App. E, Table 6) on the GPU
through hap_permtest_batch.

Each synthetic "word" is one vMF token cloud (d = 768, n tokens with n uniform in
[130, 160] like Table 6's totals, mean resultant length r uniform in [0.6, 0.9]); its
occurrences are split at random into two halves (floor(n/2) | ceil(n/2)) and the baseline
(naive, HAP_ALIGN_NONE) and proposed (Householder, HAP_ALIGN_HOUSEHOLDER) tests are run on
the SAME permutations (generator stream = word id), B = 10^4.  The paper's finding: both
halves share a mean direction, so the two tests give almost identical p-values.  Under
this same-word null the p-values are also uniform, so the rejection rate at alpha is ~alpha.

usage: python tools/split_half.py [words] [out.json]
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

# PAPER.md Table 6: word, total, baseline/greater, proposed/greater,
# baseline/two-sided, proposed/two-sided
TABLE6 = [("ablaze", 160, .2441, .2474, .4895, .4956), ("accolade", 160, .6356, .6345, .7330, .7356),
          ("actuality", 156, .7650, .7644, .4702, .4714), ("acheson", 154, .4623, .4613, .9205, .9191),
          ("adaptability", 153, .5581, .5578, .8827, .8841), ("adenauer", 152, .0369, .0342, .0756, .0709),
          ("additive", 151, .5910, .5918, .8148, .8139), ("absentee", 150, .6509, .6534, .6997, .6950),
          ("abnormally", 149, .3397, .3412, .6888, .6901), ("abstinence", 147, .5419, .5395, .9168, .9186),
          ("aberration", 145, .9040, .9056, .1845, .1815), ("acetate", 145, .6496, .6489, .7017, .7019),
          ("abstracted", 139, .2506, .2562, .5095, .5173), ("abyss", 137, .1744, .1724, .3501, .3466),
          ("abatement", 136, .4426, .4416, .8877, .8860), ("according", 135, .3434, .3443, .6827, .6846),
          ("acrimonious", 135, .9729, .9628, .0519, .0725), ("abstain", 132, .0420, .0363, .0841, .0734),
          ("accomplishment", 130, .4508, .4498, .8928, .8919), ("acne", 130, .7160, .7159, .5633, .5644)]

D = 768
B = 10000
SEED = HI.PERM_SEED


def make_words(W: int, seed: int = 2026):
    rng = np.random.default_rng(seed)
    ns = rng.integers(130, 161, size=W)
    rs = rng.uniform(0.6, 0.9, size=W)
    kap = {}
    X, Y, nx, ny = [], [], [], []
    for w in range(W):
        r = round(float(rs[w]), 2)
        if r not in kap:
            kap[r] = HI.kappa_for_r(D, r)
        wr = np.random.default_rng([seed, w])
        mu = HI.random_unit(wr, D)
        H = HI.raw_cloud(wr, mu, kap[r], int(ns[w]))
        perm = wr.permutation(int(ns[w]))  # random split of the occurrences
        h = int(ns[w]) // 2
        X.append(H[perm[:h]])
        Y.append(H[perm[h:]])
        nx.append(h)
        ny.append(int(ns[w]) - h)
    cnx = np.concatenate([[0], np.cumsum(nx)]).astype(np.int64)
    cny = np.concatenate([[0], np.cumsum(ny)]).astype(np.int64)
    return np.concatenate(X), cnx, np.concatenate(Y), cny, ns, rs


def ks_uniform(p):
    p = np.sort(np.asarray(p))
    n = len(p)
    i = np.arange(1, n + 1)
    return float(max(np.max(i / n - p), np.max(p - (i - 1) / n)))


def main():
    W = int(sys.argv[1]) if len(sys.argv) > 1 else 2000
    out_path = sys.argv[2] if len(sys.argv) > 2 else None
    t0 = time.perf_counter()
    Xp, cnx, Yp, cny, ns, rs = make_words(W)
    gen_s = time.perf_counter() - t0
    ctx = hap.Context(0)
    X, Y = torch.from_numpy(Xp).cuda(), torch.from_numpy(Yp).cuda()
    res = {}
    gpu_s = 0.0
    for name, mode in (("baseline", hap.HAP_ALIGN_NONE), ("proposed", hap.HAP_ALIGN_HOUSEHOLDER)):
        ctx.permtest_batch(X, cnx, Y, cny, B, SEED, stream_id=0, mode=mode)  # warm-up
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        infos, counts = ctx.permtest_batch(X, cnx, Y, cny, B, SEED, stream_id=0, mode=mode,
                                           sync=False)
        e1.record()
        e1.synchronize()
        gpu_s += e0.elapsed_time(e1) / 1e3
        assert hap.hap_sync(ctx.h) == 0
        c = counts.cpu().numpy()
        res[name] = {"greater": np.array([hap.hap_pvalue(int(v), B) for v in c[:, 0]]),
                     "two_sided": np.array([hap.hap_pvalue(int(v), B) for v in c[:, 1]])}
    out = {"workload": f"{W} synthetic words: one vMF cloud each (d={D}, n uniform in [130,160], "
                       "r uniform in [0.6,0.9]), occurrences split at random into halves; "
                       f"baseline (naive) vs proposed (Householder) on the same permutations, B={B}",
           "citation": "PAPER.md:194-199 (fixed-space design), App. E :852-858, Table 6 :734-767",
           "gpu_device_s": gpu_s, "tests": 2 * W, "tests_per_s": 2 * W / gpu_s, "data_gen_s": gen_s}
    for side in ("greater", "two_sided"):
        a, b = res["baseline"][side], res["proposed"][side]
        dp = np.abs(a - b)
        out[side] = {"mean_abs_dp": float(dp.mean()), "median_abs_dp": float(np.median(dp)),
                     "p99_abs_dp": float(np.quantile(dp, 0.99)), "max_abs_dp": float(dp.max()),
                     "pearson_r": float(np.corrcoef(a, b)[0, 1]),
                     "reject@0.05": {"baseline": float(np.mean(a <= 0.05)),
                                     "proposed": float(np.mean(b <= 0.05))},
                     "ks_uniform": {"baseline": ks_uniform(a), "proposed": ks_uniform(b),
                                    "crit_0.01": 1.63 / math.sqrt(W)}}
    t6 = np.array([[r[2], r[3], r[4], r[5]] for r in TABLE6])
    out["paper_table6"] = {"mean_abs_dp_greater": float(np.mean(np.abs(t6[:, 0] - t6[:, 1]))),
                           "max_abs_dp_greater": float(np.max(np.abs(t6[:, 0] - t6[:, 1]))),
                           "mean_abs_dp_two_sided": float(np.mean(np.abs(t6[:, 2] - t6[:, 3]))),
                           "max_abs_dp_two_sided": float(np.max(np.abs(t6[:, 2] - t6[:, 3])))}
    out["table"] = [{"word": f"w{w:04d}", "total": int(ns[w]), "r": round(float(rs[w]), 3),
                     "baseline_greater": float(res["baseline"]["greater"][w]),
                     "proposed_greater": float(res["proposed"]["greater"][w]),
                     "baseline_two_sided": float(res["baseline"]["two_sided"][w]),
                     "proposed_two_sided": float(res["proposed"]["two_sided"][w])}
                    for w in range(min(W, 20))]
    s = json.dumps(out, indent=1)
    print(s)
    if out_path:
        with open(out_path, "w") as f:
            f.write(s + "\n")


if __name__ == "__main__":
    main()
