"""Accuracy of the GPU statistic near r = 1 (narrow clouds, duplicated rows, tiny groups).

For each case: the GPU path (hap_align + hap_permtest with stats) and the fp64 oracle on
the same seeded inputs; prints one JSON line with the largest |dr| of the permuted groups,
the largest |dT| relative to the tie band scale (|L_X| + |L_Y|), the decisions that differ
outside the oracle's tie band, and the largest representation error max_i ||z~_i - z_i||
of the pooled planes (hap_export_pooled vs the oracle's aligned cloud).
Usage (B200): python tests/study_near1.py [--out gpurun_out/near1.jsonl]
(A test-side study: it calls oracle/, which only tests/, smoke() and bench.py's cpu_baseline
may touch, so it lives here rather than in tools/; pytest does not collect it.)
"""
from __future__ import annotations

import argparse
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import hap_inputs as HI  # noqa: E402


def cases():
    out = []
    for d in (48, 768, 4096):
        for r in (0.75, 0.96, 0.99, 0.999, 0.9999):
            k = HI.kappa_for_r(d, r)
            for nx, ny in ((1, 70), (70, 1), (2, 70), (64, 64), (1000, 1000)):
                if d == 4096 and nx == 1000:
                    nx, ny = 500, 500
                out.append(dict(kind="vmf", d=d, r=r, nx=nx, ny=ny,
                                spec=HI.PairSpec(nx, ny, d, k, k, 30.0, seed=int(1e4 * r) + d)))
    for d in (48, 768):
        for nx, ny, ndx, ndy in ((3, 40, 1, 8), (5, 5, 2, 2), (64, 64, 4, 16), (300, 200, 8, 8),
                                 (12, 12, 1, 12)):
            out.append(dict(kind="dup", d=d, r=0.75, nx=nx, ny=ny, ndx=ndx, ndy=ndy,
                            spec=HI.PairSpec(nx, ny, d, HI.kappa_for(d), HI.kappa_for(d), 30.0,
                                             seed=77 + nx)))
    return out


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default=None)
    ap.add_argument("--B", type=int, default=2000)
    args = ap.parse_args()
    import torch

    import oracle
    import paper_2605_08048_b200 as hap
    ctx = hap.Context(0)
    fout = open(args.out, "w") if args.out else None
    for c in cases():
        if c["kind"] == "vmf":
            X, Y = HI.make_pair(c["spec"])
        else:
            X, Y = HI.duplicated_pair(c["spec"], n_distinct_x=c["ndx"], n_distinct_y=c["ndy"], frac=0.7)
        B = args.B
        g = ctx.permtest_pair(torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), B,
                              HI.PERM_SEED, stream_id=5, want_stats=True)
        ref = oracle.run_pair(X, Y, B, HI.PERM_SEED, s=5, want_stats=True)
        gs, rs = g["stats"].cpu().numpy(), ref["stats"]
        Ls = abs(ref["L_x"]) + abs(ref["L_y"])
        tau = ref["tau"]
        out = np.abs(rs[:, 2] - ref["t_obs"]) > tau
        dec = int(np.sum((gs[out, 2] >= g["gemm_t_obs"]) != (rs[out, 2] >= ref["t_obs"])))
        # representation error of the pooled planes
        N, d = X.shape[0] + Y.shape[0], X.shape[1]
        n_pad, d_pad = -(-N // 64) * 64, -(-d // 32) * 32
        zh = torch.empty((d_pad, n_pad), dtype=torch.int16, device="cuda")
        zl = torch.empty_like(zh)
        t = torch.empty(d_pad, dtype=torch.float64, device="cuda")
        m = torch.empty(d_pad, dtype=torch.float64, device="cuda")
        hap.hap_export_pooled(ctx.h, zh, zl, t, m)
        torch.cuda.synchronize()
        zt = (zh.view(torch.bfloat16).double() + zl.view(torch.bfloat16).double()).cpu().numpy().T
        zt = zt[:N, :d] + m.cpu().numpy()[None, :d]
        rep = float(np.max(np.linalg.norm(zt - ref["Z"], axis=1)))
        row = dict(kind=c["kind"], d=d, r=c["r"], nx=c["nx"], ny=c["ny"],
                   r_x=ref["r_x"], r_y=ref["r_y"],
                   gemm_dr_x=g["gemm_r_x"] - ref["r_x"], gemm_dr_y=g["gemm_r_y"] - ref["r_y"],
                   dT_obs=(g["gemm_t_obs"] - ref["t_obs"]) / Ls,
                   max_dr1=float(np.max(np.abs(gs[:, 0] - rs[:, 0]))),
                   max_dr2=float(np.max(np.abs(gs[:, 1] - rs[:, 1]))),
                   max_r1=float(np.max(rs[:, 0])), max_r2=float(np.max(rs[:, 1])),
                   max_dT_rel=float(np.max(np.abs(gs[:, 2] - rs[:, 2]))) / Ls,
                   decisions_differ=dec, flagged=ref["flagged"], gpu_flagged=g["flagged"],
                   dge=g["exceed_ge"] - ref["exceed_ge"], dabs=g["exceed_abs"] - ref["exceed_abs"],
                   rep_err=rep)
        line = json.dumps(row)
        print(line, flush=True)
        if fout:
            fout.write(line + "\n")
    ctx.close()


if __name__ == "__main__":
    main()
