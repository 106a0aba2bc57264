#!/usr/bin/env python
"""bench.py — throughput of the Householder-aligned permutation test hot path on B200.

A "step" is one whole word-pair test of BASELINE.json configs[1] (C2: n_x = n_y = 1000
unit vectors, d = 768, B = 10^4 permutations): S1-S6 (alignment: normalise, means,
Householder reflect, pool/split, T_obs) + S7-S9 (PERM-SPEC v1 masks, tcgen05 mask-GEMM,
statistic, exceedance counts) on inputs resident in HBM, run through the public batch
entry point hap_permtest_batch (independent generator stream per test).
metric = permuted statistics / second (whole job, all ranks).

Multi-GPU (torchrun): word pairs are sharded over ranks (weak scaling: every rank runs
its own tests each step); the per-test integer counts are combined with one NCCL
all_reduce at the end of the timed region.  Timing: CUDA events on the launching
stream, barrier + synchronize on both sides, max over ranks.  L2: each step reads a
different pair from a rotating pool of input pairs larger than the 126 MB L2.

--impl reference runs the fp64 CPU oracle (oracle/, the checker) on the same workload
as the baseline arm (rank 0 only).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import hap_inputs as HI  # noqa: E402

METRIC = "permuted statistics/sec (N=2k, d=768)"
UNIT = "perms/s"
CFG = HI.CONFIGS["C2"]
N_X, N_Y, D, B = CFG["n_x"], CFG["n_y"], CFG["d"], CFG["B"]
WORKLOAD = (f"C2 (BASELINE.json configs[1]): single word-pair test n_x=n_y={N_X}, d={D}, "
            f"B={B} permutations; BERT-base-shaped vMF clouds kappa=1315.34 (r~0.75), "
            f"mean directions 30 deg apart, raw norms LogNormal(ln 20, 0.1)")


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


def make_pool(npairs: int, rank: int):
    pairs = []
    for i in range(npairs):
        spec = HI.PairSpec(N_X, N_Y, D, HI.kappa_for(D), HI.kappa_for(D), 30.0, seed=1002)
        pairs.append(HI.make_pair(spec, rep=1000 * rank + i))
    return pairs


# ----------------------------------------------------------------------------- clocks
class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_id: str | None):
        self.rows = []
        self.proc = None
        self.gpu_id = gpu_id

    def start(self):
        cmd = ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
               "-lms", "100"]
        if self.gpu_id:
            cmd += ["-i", self.gpu_id]
        try:
            self.proc = subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.DEVNULL,
                                         text=True)
        except OSError:
            self.proc = None
            return
        self.t = threading.Thread(target=self._read, daemon=True)
        self.t.start()

    def _read(self):
        for line in self.proc.stdout:
            parts = [p.strip() for p in line.split(",")]
            if len(parts) >= 9:
                self.rows.append((time.time(), parts))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self, t0: float, t1: float):
        rows = [p for (t, p) in self.rows if t0 - 0.25 <= t <= t1 + 0.25] or \
            [p for (_, p) in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(p[1]) for p in rows if p[1].replace(".", "").isdigit()]
        smax = [float(p[2]) for p in rows if p[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in rows for i in range(4) if p[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "samples": len(rows)}


# ----------------------------------------------------------------------------- arms
def run_reference(args):
    """The oracle as it stands, on the host cores, same metric/config; rank 0 only."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    cores = os.cpu_count() or 1
    pool = make_pool(min(args.pool, 4), 0)
    # calibrate so that W + K steps take about `budget` seconds in total
    t0 = time.perf_counter()
    oracle.run_pair(*pool[0], 64, HI.PERM_SEED, nthreads=cores)
    rate = 64 / max(time.perf_counter() - t0, 1e-3)
    budget = float(os.environ.get("HAP_REF_BUDGET_S", "150"))
    per_step = max(0.05, min(10.0, budget / max(1, args.steps + args.warmup)))
    S = int(max(cores, min(B, rate * per_step)))
    total_perms, total_s = 0, 0.0
    for k in range(args.warmup + args.steps):
        X, Y = pool[k % len(pool)]
        t0 = time.perf_counter()
        oracle.run_pair(X, Y, B, HI.PERM_SEED, s=k, b_begin=0, b_end=S, nthreads=cores)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            total_perms += S
            total_s += dt
    value = total_perms / total_s
    sample = (f"each step: oracle align + T_obs + b in [0,{S}) of the B={B} permutations "
              f"(a bounded sample of the C2 test) on {cores} threads")
    out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * total_s / args.steps, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": WORKLOAD, "parallelism": "rank 0 only (host cores)"},
           "cpu_baseline": {"value": value, "unit": UNIT, "cores": cores, "kind": "oracle",
                            "sample": sample},
           "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline(pool):
    """The oracle (untuned) on this box's host cores: whole C2 tests (align + T_obs + all
    B permutations) on successive pool pairs until ~HAP_CPU_BASELINE_S seconds have run."""
    import oracle
    cores = os.cpu_count() or 1
    budget = float(os.environ.get("HAP_CPU_BASELINE_S", "12"))
    done, t0 = 0, time.perf_counter()
    while True:
        X, Y = pool[done % len(pool)]
        oracle.run_pair(X, Y, B, HI.PERM_SEED, s=done, nthreads=cores)
        done += 1
        dt = time.perf_counter() - t0
        if dt >= budget or done >= 200:
            break
    return {"value": done * B / dt, "unit": UNIT, "cores": cores, "kind": "oracle",
            "sample": f"{done} complete C2 tests (B={B} each) on {cores} threads in {dt:.1f} s"}


def run_hap(args):
    import torch
    import torch.distributed as dist

    import paper_2605_08048_b200 as hap

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)

    def barrier():
        if world > 1:
            dist.barrier()

    # a rotating pool of distinct input pairs; the device batch repeats the pool so every
    # test of the run has its own slot (generator stream base + slot: its own permutations)
    # and the whole timed region is ONE hap_permtest_batch call (no drain between calls)
    pool_np = make_pool(args.pool, rank)
    P = len(pool_np)
    K, W = args.steps, args.warmup
    nwave_prof = max(1, min(K, 300) // 3)
    V = W + K + 3 * nwave_prof  # virtual pairs: warm-up, timed, profiling pass
    Xp = np.ascontiguousarray(np.concatenate([X for X, _ in pool_np]))
    Yp = np.ascontiguousarray(np.concatenate([Y for _, Y in pool_np]))
    Xpool, Ypool = torch.from_numpy(Xp).to(dev), torch.from_numpy(Yp).to(dev)
    reps = -(-V // P)
    Xd = Xpool.repeat(reps, 1)[: V * N_X].contiguous()
    Yd = Ypool.repeat(reps, 1)[: V * N_Y].contiguous()
    del Xpool, Ypool
    cu_nx = np.arange(V + 1, dtype=np.int64) * N_X
    cu_ny = np.arange(V + 1, dtype=np.int64) * N_Y
    in_bytes = (Xp.nbytes + Yp.nbytes)
    ctx = hap.Context(local)
    st = torch.cuda.current_stream()
    INFO = hap.INFO_BYTES
    infos = torch.zeros((V, INFO), dtype=torch.uint8, device=dev)
    counts = torch.zeros((max(K, 1), 3), dtype=torch.int64, device=dev)
    vcounts = torch.zeros((V, 3), dtype=torch.int64, device=dev)
    base_sid = (rank * 1_000_003) & 0xFFFFFFFF

    def run_tests(k0, n, out_counts=None, wave=0):
        """tests k0 .. k0+n-1 (virtual pair k = pool pair k % P, generator stream base + k)
        in one hap_permtest_batch call"""
        sel = np.arange(k0, k0 + n, dtype=np.int64)
        cfg = hap.make_cfg(HI.PERM_SEED, B, stream_id=base_sid, wave=wave)
        hap.hap_permtest_batch(ctx.h, Xd, cu_nx, Yd, cu_ny, hap.HAP_ALIGN_HOUSEHOLDER, cfg,
                               infos, vcounts, pair_sel=sel, stream=st)
        if out_counts is not None:
            out_counts[:n].copy_(vcounts[k0:k0 + n])

    gpu_id = None
    try:
        gpu_id = "GPU-" + str(torch.cuda.get_device_properties(local).uuid)
    except Exception:
        pass
    clocks = ClockSampler(gpu_id)
    clocks.start()
    time.sleep(0.3)

    # ---------------- pass 1: the headline number (no instrumentation)
    run_tests(0, W)
    torch.cuda.synchronize()
    vcounts.zero_()
    hap.hap_profile_read(ctx.h, reset=True)
    barrier()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    tw0 = time.time()
    e0.record(st)
    run_tests(W, K, counts)
    if world > 1:
        dist.all_reduce(counts)  # the one combine of the integer counts
    e1.record(st)
    e1.synchronize()
    tw1 = time.time()
    barrier()
    ms = e0.elapsed_time(e1)
    launches = hap.hap_profile_read(ctx.h, reset=True)[1]
    if world > 1:
        t = torch.tensor([ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    total_perms = K * B * world
    value = total_perms / (ms / 1e3)
    ms_per_step = ms / K

    # ---------------- pass 2: per-kernel device time (CUDA events on the launching stream)
    # one wave per call and a sync after it, so no other launch overlaps the timed ones
    wave = 3
    nw = nwave_prof
    hap.hap_profile(ctx.h, 2)
    for i in range(nw):
        run_tests(W + K + i * wave, wave, wave=wave)
        torch.cuda.synchronize()
    phase_ms, phase_n = hap.hap_profile_read(ctx.h, reset=True)
    hap.hap_profile(ctx.h, 0)
    peaks, peak_src = load_peaks()
    Nf = N_X + N_Y
    n_k3 = max(1, phase_n["maskgemm"])
    gemm_flops = 2.0 * Nf * D * B * wave  # algorithmic: the U = S X row per permutation
    gemm_s = phase_ms["maskgemm"] / 1e3 / n_k3  # per launch
    achieved_tflops = gemm_flops / gemm_s / 1e12 if gemm_s > 0 else 0.0
    peak = peaks.get("bf16_tflops_sustained", peaks["bf16_tflops"])
    n_pad = -(-Nf // 64) * 64
    issued_tflops = 4.0 * n_pad * D * B * wave / gemm_s / 1e12 if gemm_s > 0 else 0.0
    traffic = None
    tf = os.path.join(ROOT, "profiles", "k3_traffic.json")
    if os.path.exists(tf):
        with open(tf) as f:
            tj = json.load(f)
        traffic = tj.get("bytes_per_launch")
    roofline = {"bound": "tensor", "achieved": achieved_tflops, "peak": peak, "unit": "TFLOP/s",
                "frac": achieved_tflops / peak, "traffic": traffic,
                "kernel": f"k3_maskgemm (S8+S9), one launch = a wave of {wave} C2 tests",
                "peak_source": f"{peak_src} bf16_tflops_sustained (kernel timed inside the step loop)",
                "achieved_basis": "algorithmic 2*N*d FLOP per permutation (SURVEY.md 8d)",
                "issued_tflops": issued_tflops, "k3_us_per_launch": gemm_s * 1e6,
                "gemm_share_of_step": phase_ms["maskgemm"] / max(1e-9, sum(phase_ms.values()))}
    phases_per_test = {k: v / (nw * wave) for k, v in phase_ms.items()}

    # ---------------- pass 3: end to end through the C ABI with HOST inputs: every chunk
    # of tests passes the packed X, Y in pinned host memory to hap_permtest_batch, which
    # copies each wave's rows on its lane streams (overlapping the other lane's kernels);
    # the counts are read back into pinned host memory; one sync at the end
    Ke = min(K, 480)
    Xh = torch.from_numpy(Xp).pin_memory()
    Yh = torch.from_numpy(Yp).pin_memory()
    host_counts = torch.zeros((Ke, 3), dtype=torch.int64).pin_memory()
    dev_counts = torch.zeros((2, P, 3), dtype=torch.int64, device=dev)

    def e2e_chunk(c, k0, m):
        cfg = hap.make_cfg(HI.PERM_SEED, B, stream_id=(rank * 1_000_003 + k0) & 0xFFFFFFFF)
        dc = dev_counts[c % 2]
        dc.zero_()
        hap.hap_permtest_batch(ctx.h, Xh, cu_nx[: m + 1], Yh, cu_ny[: m + 1],
                               hap.HAP_ALIGN_HOUSEHOLDER, cfg, infos, dc, stream=st)
        host_counts[k0: k0 + m].copy_(dc[:m], non_blocking=True)  # D2H of the results

    e2e_chunk(0, 0, min(P, Ke))
    torch.cuda.synchronize()
    barrier()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    k, c = 0, 0
    while k < Ke:
        m = min(P, Ke - k)
        e2e_chunk(c, k, m)
        k += m
        c += 1
    torch.cuda.synchronize()
    e2e_s = time.perf_counter() - t0
    if world > 1:
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = float(t.item())
    last = int(host_counts[Ke - 1, 0])
    e2e = {"value": Ke * B * world / e2e_s, "unit": UNIT,
           "h2d_bytes_per_step": (N_X + N_Y) * D * 4, "d2h_bytes_per_step": 3 * 8,
           "steps": Ke, "timer": "host wall clock around the loop, synchronize on both sides",
           "api": f"hap_permtest_batch on chunks of {P} tests with X, Y in pinned HOST memory "
                  "(the library copies each wave's rows on its lane streams), counts copied D2H"}

    clocks.stop()
    clk = clocks.summary(tw0, tw1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(pool_np)
    if rank == 0:
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": K,
               "warmup": W, "ms_per_step": ms_per_step, "higher_is_better": True,
               "scaling": "weak", "vs_baseline": None, "dtype": "bf16",
               "data": "synthetic",
               "config": {"workload": WORKLOAD, "global_batch": world, "B": B, "n_x": N_X,
                          "n_y": N_Y, "d": D,
                          "l2": f"rotating pool of {P} distinct input pairs per rank "
                                f"({in_bytes / 1e6:.0f} MB > 126 MB L2), repeated in HBM so "
                                f"each test has its own slot",
                          "parallelism": f"tests sharded over {world} rank(s); each rank runs "
                                         "its own tests; counts combined by one all_reduce",
                          "api": "hap_permtest_batch (2 internal lanes, waves of 3 tests per "
                                 "alignment / generator / mask-GEMM launch)",
                          "arith": "bf16 hi/lo split operands, fp32 TMEM accumulation, "
                                   "fp64 statistic"},
               "roofline": roofline, "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
               "gpu_launches": int(sum(launches.values())),
               "gpu_launches_by_phase": launches, "phase_ms_per_test": phases_per_test,
               "last_test": {"exceed_ge": last, "p_value": hap.hap_pvalue(last, B)}}
        print(json.dumps(out), flush=True)
    ctx.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=2000)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="hap", choices=["hap", "reference"])
    ap.add_argument("--pool", type=int, default=24, help="distinct input pairs per rank")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_hap(args)


if __name__ == "__main__":
    main()
