#!/usr/bin/env python
"""bench.py — throughput of the Householder-aligned permutation test hot path on B200.

Workloads (BASELINE.json configs; `--workload`, default c2):
  c2  the headline: "permuted statistics/sec (N=2k, d=768)".  A STEP is one batch of
      --tests-per-step (100) whole word-pair tests of configs[1] (n_x = n_y = 1000, d = 768,
      B = 10^4 permutations each: 10^6 permuted statistics) through ONE call of the public
      batch entry point hap_permtest_batch: S1-S6 (normalise, means, Householder reflect,
      pool/split, T_obs) + S7-S9 (PERM-SPEC v1 masks, tcgen05 mask-GEMM, statistic,
      exceedance counts), every test on its own generator stream.  Multi-GPU: every rank
      runs its own tests (weak scaling).
  c3  configs[2]: one LLM-sized pair (n = 5000/5000, d = 4096, B = 10^5) per step,
      hap_align + hap_permtest; multi-GPU: the b-range is sharded (strong scaling).
  c4  configs[3]: the thesaurus-scale batch, 10^4 pairs of log-uniform n in [50, 5000],
      d = 768, B = 10^4 each, one hap_permtest_batch call per rank per step; multi-GPU:
      pairs LPT-assigned over ranks (strong scaling).  Metric: word-pair tests/sec.
  c5  configs[4]: the Type-I calibration workload, 10^3 null replicates x {aligned,
      naive}, n = 500/500, d = 768, B = 10^4 (2000 tests per step).  Metric: tests/sec.
Timing: CUDA events on the launching stream, barrier + synchronize on both sides, max
over ranks; the integer counts are combined with ONE all_reduce inside the timed region.
Inputs of every step are larger than the 126 MB L2 (stated in `config.l2`).

--impl reference runs the fp64 CPU oracle (oracle/, the checker) on a bounded sample of
the same workload (rank 0 only).  bench.py refuses to run with any HAP_* environment
variable set (library experiment knobs), and says so on its JSON line.
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

UNIT_P = "perms/s"
UNIT_T = "tests/s"
TESTS_PER_STEP = 100
RECIPE = ("vMF clouds (Wood sampler) with E[MRL]=0.75 (kappa=1315.34 at d=768, 7020.48 at "
          "d=4096), mean directions 30 deg apart, raw norms LogNormal(ln 20, 0.1)")


def load_peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as f:
            return json.load(f), "measured"
    except OSError:
        return {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}, \
            "fallback (B200_PROFILING.md)"


def cpu_model() -> str:
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


def usable_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:
        return os.cpu_count() or 1


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
        rows = [p for (t, p) in self.rows if t0 - 0.15 <= t <= t1 + 0.15] or \
            [p for (_, p) in self.rows]
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": [], "samples": 0}
        sm = [float(p[1]) for p in rows if p[1].replace(".", "").isdigit()]
        smax = [float(p[2]) for p in rows if p[2].replace(".", "").isdigit()]
        pw = [float(p[3]) for p in rows if p[3].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for p in rows for i in range(4) if p[5 + i] == "Active"})
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None, "reasons": reasons,
                "power_w_max": max(pw) if pw else None, "samples": len(rows)}


# ----------------------------------------------------------------------------- workloads
def c2_pool(npairs: int, rank: int, n_x=1000, n_y=1000, d=768, seed=1002):
    k = HI.kappa_for(d)
    return [HI.make_pair(HI.PairSpec(n_x, n_y, d, k, k, 30.0, seed=seed), rep=1000 * rank + i)
            for i in range(npairs)]


def c4_sizes():
    c = HI.CONFIGS["C4"]
    n = HI.c4_sizes(c["P"], c["n_min"], c["n_max"])  # n_X = n_Y = n_p
    return n


WORKLOADS = {
    "c2": dict(metric="permuted statistics/sec (N=2k, d=768)", unit=UNIT_P,
               config="C2", scaling="weak"),
    "c3": dict(metric="permuted statistics/sec (N=10k, d=4096)", unit=UNIT_P,
               config="C3", scaling="strong"),
    "c4": dict(metric="word-pair tests/sec (thesaurus-scale batch)", unit=UNIT_T,
               config="C4", scaling="strong"),
    "c5": dict(metric="word-pair tests/sec (Type-I calibration, aligned + naive)",
               unit=UNIT_T, config="C5", scaling="strong"),
}


def workload_desc(name: str, T: int) -> str:
    c = HI.CONFIGS[WORKLOADS[name]["config"]]
    if name == "c2":
        return (f"C2 (BASELINE.json configs[1]): {T} word-pair tests per step, each n_x=n_y="
                f"{c['n_x']}, d={c['d']}, B={c['B']}; {RECIPE}")
    if name == "c3":
        return (f"C3 (configs[2]): one pair n_x=n_y={c['n_x']}, d={c['d']}, B={c['B']} per "
                f"step, b-range sharded over ranks; {RECIPE}")
    if name == "c4":
        return (f"C4 (configs[3]): {c['P']} pairs, n_x=n_y=n_p log-uniform in "
                f"[{c['n_min']}, {c['n_max']}] (seed 1004), d={c['d']}, B={c['B']} each, pairs "
                f"LPT-sharded over ranks; {RECIPE}")
    return (f"C5 (configs[4]): {c['R']} null replicates x (aligned, naive), n_x=n_y={c['n_x']}, "
            f"d={c['d']}, B={c['B']}; {RECIPE}")


# ----------------------------------------------------------------------------- reference arm
def run_reference(args):
    """The oracle as it stands, on the host cores, same metric/unit/config; rank 0 only.
    Each step is a bounded sample of the workload (align + T_obs + the first S
    permutations of one test), sized so that the whole run takes ~BENCH_REF_BUDGET_S."""
    import oracle
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    W = WORKLOADS[args.workload]
    cfg = HI.CONFIGS[W["config"]]
    cores = usable_cores()
    if args.workload == "c3":
        pool = [HI.config_pair("C3")]
    elif args.workload == "c4":
        sizes = c4_sizes()[:8]
        pool = [HI.make_pair(HI.PairSpec(int(n), int(n), 768, HI.kappa_for(768),
                                         HI.kappa_for(768), 30.0, seed=1004), rep=p)
                for p, n in enumerate(sizes)]
    elif args.workload == "c5":
        pool = c2_pool(4, 0, 500, 500, 768, seed=1005)
    else:
        pool = c2_pool(4, 0)
    B = cfg["B"]
    t0 = time.perf_counter()
    oracle.run_pair(*pool[0], B, HI.PERM_SEED, b_begin=0, b_end=64, nthreads=cores)
    rate = 64 / max(time.perf_counter() - t0, 1e-3)
    budget = float(os.environ.get("BENCH_REF_BUDGET_S", "150"))
    per_step = max(0.05, min(10.0, budget / max(1, args.steps + args.warmup)))
    S = int(max(cores, min(B, rate * per_step)))
    perms, secs, test_s = 0, 0.0, 0.0
    for k in range(args.warmup + args.steps):
        X, Y = pool[k % len(pool)]
        t0 = time.perf_counter()
        oracle.run_pair(X, Y, B, HI.PERM_SEED, s=k, b_begin=0, b_end=S, nthreads=cores)
        dt = time.perf_counter() - t0
        if k >= args.warmup:
            perms += S
            secs += dt
            test_s += dt * B / S  # one whole test, extrapolated from the sample
    if W["unit"] == UNIT_P:
        value = perms / secs
        sample = (f"each step: oracle align + T_obs + b in [0,{S}) of one {W['config']} test "
                  f"(B={B}) on {cores} threads")
    else:
        value = args.steps / test_s
        sample = (f"each step: oracle align + T_obs + b in [0,{S}) of one {W['config']}-shaped "
                  f"test, time per whole test extrapolated x{B / S:.1f}; {cores} threads")
    out = {"metric": W["metric"], "value": value, "unit": W["unit"], "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup,
           "ms_per_step": 1e3 * secs / args.steps, "higher_is_better": True,
           "scaling": W["scaling"], "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "impl": "reference",
           "config": {"workload": workload_desc(args.workload, args.tests_per_step),
                      "parallelism": "rank 0 only (host cores)"},
           "cpu_baseline": {"value": value, "unit": W["unit"], "cores": cores, "kind": "oracle",
                            "sample": sample, "cpu": cpu_model()},
           "e2e": {"value": value, "unit": W["unit"], "h2d_bytes_per_step": 0,
                   "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def cpu_baseline(pool, B, budget_s=12.0):
    """The oracle (untuned) on this box's host cores: whole tests (align + T_obs + all B
    permutations) on successive pool pairs for ~budget_s seconds, plus the same oracle on
    ONE thread over a bounded b-range of one test."""
    import oracle
    cores = usable_cores()
    budget = float(os.environ.get("BENCH_CPU_BASELINE_S", str(budget_s)))
    done, t0 = 0, time.perf_counter()
    while True:
        X, Y = pool[done % len(pool)]
        oracle.run_pair(X, Y, B, HI.PERM_SEED, s=done, nthreads=cores)
        done += 1
        dt = time.perf_counter() - t0
        if dt >= budget or done >= 200:
            break
    S1 = 200
    X, Y = pool[0]
    t1 = time.perf_counter()
    oracle.run_pair(X, Y, B, HI.PERM_SEED, s=0, b_begin=0, b_end=S1, nthreads=1)
    one = S1 / (time.perf_counter() - t1)
    return {"value": done * B / dt, "unit": UNIT_P, "cores": cores, "kind": "oracle",
            "cpu": cpu_model(), "value_1thread": one,
            "sample": f"{done} complete tests (B={B} each) on {cores} threads in {dt:.1f} s; "
                      f"1-thread rate: align + b in [0,{S1}) of one test"}


# ----------------------------------------------------------------------------- GPU arm
class Env:
    def __init__(self):
        import torch
        import torch.distributed as dist
        import paper_2605_08048_b200 as hap
        self.torch, self.dist, self.hap = torch, dist, hap
        self.world = int(os.environ.get("WORLD_SIZE", "1"))
        self.rank = int(os.environ.get("RANK", "0"))
        self.local = int(os.environ.get("LOCAL_RANK", "0"))
        torch.cuda.set_device(self.local)
        self.dev = torch.device("cuda", self.local)
        if self.world > 1:
            dist.init_process_group("nccl", device_id=self.dev)
        self.ctx = hap.Context(self.local)
        self.st = torch.cuda.current_stream()

    def barrier(self):
        if self.world > 1:
            self.dist.barrier()

    def max_over_ranks(self, v: float) -> float:
        if self.world == 1:
            return v
        t = self.torch.tensor([v], dtype=self.torch.float64, device=self.dev)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.MAX)
        return float(t.item())

    def timed(self, fn, K):
        """barrier + sync; events around K calls of fn(k) on the launching stream; max over
        ranks.  Returns (ms, wall_t0, wall_t1)."""
        torch = self.torch
        self.barrier()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        tw0 = time.time()
        e0.record(self.st)
        for k in range(K):
            fn(k)
        e1.record(self.st)
        e1.synchronize()
        tw1 = time.time()
        torch.cuda.synchronize()
        self.barrier()
        return self.max_over_ranks(e0.elapsed_time(e1)), tw0, tw1


def kernel_profile(E, run_waves, n_tests, N, d, B, peaks, what):
    """Per-kernel device time with CUDA events on each launch's own stream (hap_profile
    level 2: phases serialised, one wave per call and a sync after it, so no other launch
    overlaps a timed one): K3 (dominant, tensor-bound), K1 (HBM), K2 (integer ALU).
    Normalised per test: `n_tests` tests of N pooled rows, d columns, B permutations."""
    hap = E.hap
    hap.hap_profile_read(E.ctx.h, reset=True)
    hap.hap_profile(E.ctx.h, 2)
    run_waves()
    phase_ms, phase_n = hap.hap_profile_read(E.ctx.h, reset=True)
    hap.hap_profile(E.ctx.h, 0)
    n_pad = -(-N // 64) * 64
    d_pad = -(-d // 32) * 32
    k3_s = phase_ms["maskgemm"] / 1e3
    flops = 2.0 * N * d * B * n_tests  # algorithmic: the U = S X row per permutation
    ach = flops / k3_s / 1e12 if k3_s > 0 else 0.0
    peak = peaks["bf16_tflops"]
    k1_s = phase_ms["align"] / 1e3
    k1_bytes = n_tests * (4.0 * N * d + 4.0 * n_pad * d_pad)  # read X,Y fp32; write hi,lo
    k2_s = phase_ms["permgen"] / 1e3
    k1_gbs = k1_bytes / k1_s / 1e9 if k1_s else 0.0
    return {
        "bound": "tensor", "achieved": ach, "peak": peak, "unit": "TFLOP/s",
        "frac": ach / peak, "kernel": f"k3_maskgemm (S8+S9); {what}",
        "peak_source": "MEASURED_PEAKS.json bf16_tflops (burst): K3 is timed one isolated "
                       "launch at a time (CUDA events on its stream, a sync between launches)",
        "achieved_basis": "algorithmic 2*N*d FLOP per permutation (SURVEY.md 8d) x the "
                          "permutations of the timed launches / their summed duration",
        "issued_tflops": 4.0 * n_pad * d_pad * B * n_tests / k3_s / 1e12 if k3_s else 0.0,
        "k3_us_per_launch": phase_ms["maskgemm"] * 1e3 / max(1, phase_n["maskgemm"]),
        "launches_timed": phase_n,
        "k1_align": {"bound": "hbm", "unit": "GB/s", "achieved": k1_gbs,
                     "peak": peaks["hbm_gbs"], "frac": k1_gbs / peaks["hbm_gbs"],
                     "us_per_test": k1_s * 1e6 / n_tests,
                     "basis": "read 4*N*d (fp32 X, Y) + write 4*n_pad*d_pad (bf16 hi, lo) "
                              "bytes per test"},
        "k2_permgen": {"bound": "alu", "unit": "perms/s",
                       "achieved": n_tests * B / k2_s if k2_s else 0.0,
                       "us_per_test": k2_s * 1e6 / n_tests},
        "phase_ms": phase_ms,
        "traffic": None,
        "traffic_basis": "no ncu --set full capture of this workload's K3 launch is committed "
                         "(profiles/r02_ncu_full_k3_k2_raw.csv is a C2 wave)",
    }


NCU_FULL = os.path.join(ROOT, "profiles", "r02_ncu_full_k3_k2_raw.csv")


def ncu_traffic(kernel="k3_maskgemm"):
    """dram__bytes_read.sum + dram__bytes_write.sum of one launch of `kernel` from the
    committed `ncu --set full` capture (a C2 batch wave of 3 tests: the launch shape the C2
    bench times), in bytes; None if the capture is absent."""
    import csv
    try:
        rows = list(csv.reader(open(NCU_FULL)))
    except OSError:
        return None
    hdr, units = rows[0], rows[1]
    scale = {"byte": 1.0, "Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9}
    for r in rows[2:]:
        if kernel in r[hdr.index("Kernel Name")]:
            tot = 0.0
            for k in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
                i = hdr.index(k)
                tot += float(r[i].replace(",", "")) * scale.get(units[i], 1.0)
            return tot
    return None


def in_step_spans(E, run_one_step, flops, peaks):
    """K3 inside the real pipelined step: device-clock spans (first CTA entry -> last CTA
    exit) of every mask-GEMM launch of one step; the step's algorithmic FLOP over the time
    in which at least one K3 launch was running, as a fraction of the SUSTAINED peak."""
    hap = E.hap
    hap.hap_profile_spans(E.ctx.h, 1)
    run_one_step()
    E.torch.cuda.synchronize()
    spans = hap.hap_profile_spans_read(E.ctx.h)
    hap.hap_profile_spans(E.ctx.h, 0)
    k3 = sorted((s, e) for (ph, s, e) in spans if ph.startswith("maskgemm") and e >= s)
    if not k3:
        return None
    busy, cur_s, cur_e = 0.0, k3[0][0], k3[0][1]
    for s, e in k3[1:]:
        if s > cur_e:
            busy += cur_e - cur_s
            cur_s, cur_e = s, e
        else:
            cur_e = max(cur_e, e)
    busy += cur_e - cur_s
    allsp = [(s, e) for (_, s, e) in spans if e >= s]
    step_us = max(e for _, e in allsp) - min(s for s, _ in allsp)
    ach = flops / (busy * 1e-6) / 1e12
    return {"k3_launches": len(k3), "k3_busy_us": busy, "step_us": step_us,
            "k3_busy_share": busy / step_us, "achieved": ach,
            "peak": peaks["bf16_tflops_sustained"],
            "frac": ach / peaks["bf16_tflops_sustained"],
            "basis": "one step with kernel spans on; algorithmic FLOP of the step / union of "
                     "the K3 spans (K3 shares the SMs with the other lane's K1/K2)"}


def run_c2(args, E, peaks):
    torch, hap = E.torch, E.hap
    T, K, W = args.tests_per_step, args.steps, args.warmup
    cfg0 = HI.CONFIGS["C2"]
    n_x, n_y, d, B = cfg0["n_x"], cfg0["n_y"], cfg0["d"], cfg0["B"]
    N = n_x + n_y
    pool = c2_pool(args.pool, E.rank)
    P = len(pool)
    Xp = np.ascontiguousarray(np.concatenate([pool[i % P][0] for i in range(T)]))
    Yp = np.ascontiguousarray(np.concatenate([pool[i % P][1] for i in range(T)]))
    Xd, Yd = torch.from_numpy(Xp).to(E.dev), torch.from_numpy(Yp).to(E.dev)
    cu_nx = np.arange(T + 1, dtype=np.int64) * n_x
    cu_ny = np.arange(T + 1, dtype=np.int64) * n_y
    in_bytes = Xp.nbytes + Yp.nbytes
    INFO = hap.INFO_BYTES
    infos = torch.zeros((T, INFO), dtype=torch.uint8, device=E.dev)
    # every rank writes ITS block of one [world, K, T, 3] buffer; one all_reduce combines
    counts = torch.zeros((E.world, K, T, 3), dtype=torch.int64, device=E.dev)
    scratch = torch.zeros((T, 3), dtype=torch.int64, device=E.dev)
    base = (E.rank << 27) & 0xFFFFFFFF  # generator streams: rank, step, test

    def step(k, out, X=Xd, Y=Yd, n=T, wave=0, flags=0):
        cfg = hap.make_cfg(HI.PERM_SEED, B, stream_id=(base + k * T) & 0xFFFFFFFF, wave=wave,
                           flags=flags)
        hap.hap_permtest_batch(E.ctx.h, X, cu_nx[: n + 1], Y, cu_ny[: n + 1],
                               hap.HAP_ALIGN_HOUSEHOLDER, cfg, infos, out, stream=E.st)

    for k in range(W):
        step(K + k, scratch)
    torch.cuda.synchronize()
    hap.hap_profile_read(E.ctx.h, reset=True)

    def timed_step(k):
        step(k, counts[E.rank, k])
        if k == K - 1 and E.world > 1:
            E.dist.all_reduce(counts)  # the one combine of the integer counts

    ms, tw0, tw1 = E.timed(timed_step, K)
    launches = hap.hap_profile_read(E.ctx.h, reset=True)[1]
    value = E.world * K * T * B / (ms / 1e3)

    # per-kernel rooflines (isolated waves of 3 tests)
    wave = 3
    nw = max(4, min(40, K * T // wave // 4))

    def waves():
        for i in range(nw):
            scratch.zero_()
            step(2 * K + i, scratch, wave=wave, n=wave)
            torch.cuda.synchronize()
    roof = kernel_profile(E, waves, nw * wave, N, d, B, peaks,
                          f"one launch = a wave of {wave} C2 tests")
    n_pad, d_pad = -(-N // 64) * 64, -(-d // 32) * 32
    tiles = -(-B // 127)  # 127 permutation rows + the observed row per 128-row tile
    roof["traffic"] = ncu_traffic()
    roof["traffic_basis"] = ("dram__bytes_read.sum + dram__bytes_write.sum of one K3 launch "
                             "(a wave of 3 C2 tests) from profiles/r02_ncu_full_k3_k2_raw.csv "
                             "(ncu --set full)")
    roof["operand_bytes_per_launch"] = wave * (tiles * 128 * n_pad * 2 + 2 * d_pad * n_pad * 2)

    def one_step():
        scratch.zero_()
        step(3 * K, scratch)
    roof["in_step"] = in_step_spans(E, one_step, 2.0 * N * d * B * T, peaks)

    # end to end through the C ABI with HOST inputs: each step's packed X, Y (pinned) are
    # copied by the library per wave on its lane streams; the counts are copied D2H
    Ke = min(K, args.e2e_steps)
    Xh, Yh = torch.from_numpy(Xp).pin_memory(), torch.from_numpy(Yp).pin_memory()
    hcounts = torch.zeros((Ke, T, 3), dtype=torch.int64).pin_memory()
    dcounts = torch.zeros((2, T, 3), dtype=torch.int64, device=E.dev)

    def e2e_step(k):
        dc = dcounts[k % 2]
        dc.zero_()
        step(4 * K + k, dc, X=Xh, Y=Yh)
        hcounts[k].copy_(dc, non_blocking=True)

    e2e_step(0)
    torch.cuda.synchronize()
    E.barrier()
    t0 = time.perf_counter()
    for k in range(Ke):
        e2e_step(k)
    torch.cuda.synchronize()
    e2e_s = E.max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": E.world * Ke * T * B / e2e_s, "unit": UNIT_P,
           "h2d_bytes_per_step": in_bytes, "d2h_bytes_per_step": T * 3 * 8, "steps": Ke,
           "timer": "host wall clock around the loop, synchronize on both sides",
           "api": "hap_permtest_batch with the step's packed X, Y in pinned HOST memory (the "
                  "library copies each wave's rows on its lane streams); counts copied D2H"}
    cpu = None
    if E.rank == 0 and E.world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(pool, B)
    cfg_out = {"workload": workload_desc("c2", T), "tests_per_step": T, "B": B, "n_x": n_x,
               "n_y": n_y, "d": d, "global_batch": E.world * T,
               "l2": f"each step reads {in_bytes / 1e6:.0f} MB of input pairs ({P} distinct, "
                     "repeated in HBM) > 126 MB L2; no flush",
               "parallelism": f"dp{E.world}: each rank runs its own {T} tests per step; "
                              "counts combined by one all_reduce",
               "api": "hap_permtest_batch (2 internal lanes, the library's automatic wave size: 4 "
                      "tests per alignment / generator / mask-GEMM launch at N <= 2048)",
               "arith": "bf16 hi/lo split operands, fp32 TMEM accumulation, fp64 statistic"}
    last = int(counts[E.rank, K - 1, T - 1, 0])
    extra = {"last_test": {"exceed_ge": last, "p_value": hap.hap_pvalue(last, B)}}
    # The paper's reuse note ("When testing many word pairs with the same (n,m),
    # the same randomly generated sign blocks can be reused across pairs"): the same K steps
    # with HAP_FLAG_SHARED_MASK (all tests of a step on one generator stream; equal-size
    # tests share one generated mask block per wave).  Reported beside, not as, the value:
    # the headline keeps independent permutations per test.
    sh_counts = torch.zeros((K, T, 3), dtype=torch.int64, device=E.dev)
    for k in range(W):
        step(5 * K + k, scratch, flags=hap.HAP_FLAG_SHARED_MASK)
    ms_sh, _, _ = E.timed(lambda k: step(6 * K + k, sh_counts[k], flags=hap.HAP_FLAG_SHARED_MASK), K)
    extra["shared_masks"] = {
        "value": E.world * K * T * B / (ms_sh / 1e3), "unit": UNIT_P, "ms_per_step": ms_sh / K,
        "note": "same workload with HAP_FLAG_SHARED_MASK: the paper's sign-block reuse across "
                "pairs of equal (n, m) (PAPER.md:259); each test is still an exact permutation "
                "test, the tests share their permutations"}
    return value, ms, tw0, tw1, launches, roof, e2e, cpu, cfg_out, extra


def run_c3(args, E, peaks):
    torch, hap = E.torch, E.hap
    from paper_2605_08048_b200 import parallel
    c = HI.CONFIGS["C3"]
    n_x, n_y, d, B = c["n_x"], c["n_y"], c["d"], c["B"]
    N = n_x + n_y
    K, W = args.steps, args.warmup
    pool = [HI.config_pair("C3", rep=r) for r in range(2)]
    dev_pool = [(torch.from_numpy(X).to(E.dev), torch.from_numpy(Y).to(E.dev)) for X, Y in pool]
    b0, b1 = parallel.shard_range(B, E.rank, E.world)
    infos = torch.zeros((2, hap.INFO_BYTES), dtype=torch.uint8, device=E.dev)
    counts = torch.zeros((K, 3), dtype=torch.int64, device=E.dev)
    scratch = torch.zeros(3, dtype=torch.int64, device=E.dev)

    def step(k, out, X=None, Y=None, combine=False):
        """align (every rank: the same deterministic planes) + this rank's b-range; with
        combine, one all-reduce of the 3 counts (parallel.gpu_range_counts)"""
        Xs, Ys = dev_pool[k % 2] if X is None else (X, Y)
        parallel.gpu_range_counts(E.ctx, Xs, Ys, B, HI.PERM_SEED, E.rank, E.world, out,
                                  infos[k % 2], stream_id=k, stream=E.st, reduce=combine)

    for k in range(W):
        step(k, scratch)
    torch.cuda.synchronize()
    hap.hap_profile_read(E.ctx.h, reset=True)

    def timed_step(k):
        step(k, counts[k], combine=True)

    ms, tw0, tw1 = E.timed(timed_step, K)
    launches = hap.hap_profile_read(E.ctx.h, reset=True)[1]
    value = K * B / (ms / 1e3)

    def waves():
        for i in range(2):
            scratch.zero_()
            step(i, scratch)
            torch.cuda.synchronize()
    roof = kernel_profile(E, waves, 2, N, d, b1 - b0, peaks,
                          f"one test = this rank's b-range [{b0},{b1}) in L2-sized blocks")
    Ke = min(K, 4)
    Xh, Yh = [torch.from_numpy(X).pin_memory() for X, _ in pool], \
        [torch.from_numpy(Y).pin_memory() for _, Y in pool]
    hcounts = torch.zeros((Ke, 3), dtype=torch.int64).pin_memory()
    dcounts = torch.zeros((Ke, 3), dtype=torch.int64, device=E.dev)
    torch.cuda.synchronize()
    E.barrier()
    t0 = time.perf_counter()
    for k in range(Ke):
        step(k, dcounts[k], Xh[k % 2], Yh[k % 2], combine=True)
        hcounts[k].copy_(dcounts[k], non_blocking=True)
    torch.cuda.synchronize()
    e2e_s = E.max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": Ke * B / e2e_s, "unit": UNIT_P,
           "h2d_bytes_per_step": int(pool[0][0].nbytes + pool[0][1].nbytes),
           "d2h_bytes_per_step": 24, "steps": Ke,
           "timer": "host wall clock around the loop, synchronize on both sides",
           "api": "hap_align (X, Y in pinned HOST memory) + hap_permtest, counts D2H"}
    cfg_out = {"workload": workload_desc("c3", 1), "B": B, "n_x": n_x, "n_y": n_y, "d": d,
               "global_batch": 1,
               "l2": "two distinct 164 MB pairs alternate (> 126 MB L2); no flush",
               "parallelism": f"b-range sharded over {E.world} rank(s); one all_reduce of "
                              "the 3 counts per test"}
    return value, ms, tw0, tw1, launches, roof, e2e, None, cfg_out, {}


def c4_packed(E, sizes, Q=8):
    """Device-resident packed C4 batch: pair p takes the first n_p rows of pool pair p % Q
    (a vMF prefix is itself a vMF sample); each pair has its own generator stream."""
    torch = E.torch
    k = HI.kappa_for(768)
    pool = [HI.make_pair(HI.PairSpec(5000, 5000, 768, k, k, 30.0, seed=1004), rep=q)
            for q in range(Q)]
    px = [torch.from_numpy(X).to(E.dev) for X, _ in pool]
    py = [torch.from_numpy(Y).to(E.dev) for _, Y in pool]
    tot = int(np.sum(sizes))
    Xd = torch.empty((tot, 768), dtype=torch.float32, device=E.dev)
    Yd = torch.empty((tot, 768), dtype=torch.float32, device=E.dev)
    off = 0
    for p, n in enumerate(sizes):
        n = int(n)
        Xd[off:off + n].copy_(px[p % Q][:n])
        Yd[off:off + n].copy_(py[p % Q][:n])
        off += n
    cu = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    return Xd, cu, Yd, cu.copy(), pool


def run_batch_workload(args, E, peaks, name):
    """c4 / c5: one hap_permtest_batch call per rank per step over its LPT share."""
    torch, hap = E.torch, E.hap
    from paper_2605_08048_b200 import parallel
    K, W = args.steps, args.warmup
    if name == "c4":
        c = HI.CONFIGS["C4"]
        sizes = c4_sizes()
        Xd, cnx, Yd, cny, pool = c4_packed(E, sizes)
        modes = [hap.HAP_ALIGN_HOUSEHOLDER]
        B = c["B"]
        l2 = f"{Xd.numel() * 8 / 1e9:.1f} GB of packed inputs per step (> 126 MB L2)"
    else:
        c = HI.CONFIGS["C5"]
        R = c["R"]
        pool = c2_pool(args.pool, 0, c["n_x"], c["n_y"], c["d"], seed=1005)
        sizes = np.full(R, c["n_x"], dtype=np.int64)
        Xd = torch.from_numpy(np.concatenate([pool[i % len(pool)][0] for i in range(R)])).to(E.dev)
        Yd = torch.from_numpy(np.concatenate([pool[i % len(pool)][1] for i in range(R)])).to(E.dev)
        cnx = np.arange(R + 1, dtype=np.int64) * c["n_x"]
        cny = np.arange(R + 1, dtype=np.int64) * c["n_y"]
        modes = [hap.HAP_ALIGN_HOUSEHOLDER, hap.HAP_ALIGN_NONE]
        B = c["B"]
        l2 = f"{Xd.numel() * 8 / 1e6:.0f} MB of packed inputs per step (> 126 MB L2)"
    P = len(sizes)
    costs = (np.diff(cnx) + np.diff(cny)).tolist()
    mine = parallel.lpt_assign(costs, E.world)[E.rank]
    iw = hap.INFO_BYTES // 8
    nm = len(modes)
    infos = torch.zeros((nm, P, hap.INFO_BYTES), dtype=torch.uint8, device=E.dev)
    dcounts = torch.zeros((nm, P, 3), dtype=torch.int64, device=E.dev)

    def step(k, sel=mine, X=Xd, Y=Yd):
        for mi, mode in enumerate(modes):
            cfg = hap.make_cfg(HI.PERM_SEED, B, stream_id=((k * nm + mi) * P) & 0xFFFFFFFF)
            if sel:
                hap.hap_permtest_batch(E.ctx.h, X, cnx, Y, cny, mode, cfg, infos[mi],
                                       dcounts[mi], pair_sel=sel, stream=E.st)

    for k in range(W):
        step(K + k)
    torch.cuda.synchronize()
    hap.hap_profile_read(E.ctx.h, reset=True)

    results = []

    def timed_step(k):
        # parallel.gpu_batch_sharded: this rank's LPT share in ONE hap_permtest_batch call,
        # then one all-reduce of int64[P, info + 3] rows (each written by exactly one rank)
        for mi, mode in enumerate(modes):
            results.append(parallel.gpu_batch_sharded(
                E.ctx, Xd, cnx, Yd, cny, B, HI.PERM_SEED, E.rank, E.world,
                stream_id=((k * nm + mi) * P) & 0xFFFFFFFF, mode=mode))

    ms, tw0, tw1 = E.timed(timed_step, K)
    launches = hap.hap_profile_read(E.ctx.h, reset=True)[1]
    tests = K * P * nm
    value = tests / (ms / 1e3)
    perms = tests * B / (ms / 1e3)
    # dominant kernel of the batch: profile waves of the largest pairs in isolation
    order = sorted(range(P), key=lambda p: -costs[p])
    big = order[:6]

    def waves():
        for i in range(2):
            dcounts.zero_()
            step(10 * K + i, sel=big[3 * i: 3 * i + 3])
            torch.cuda.synchronize()
    nb = int(sizes[big[0]])
    # (step() runs every mode, so the two isolated calls hold 6 tests per mode)
    roof = kernel_profile(E, waves, 6 * nm, 2 * nb, 768, B, peaks,
                          f"isolated waves of the 3 largest pairs (n~{nb}) of the batch, "
                          f"{nm} mode(s)")
    # e2e on a bounded slice from pinned host memory (whole batch would pin tens of GB)
    Pe = min(P, 1000 if name == "c4" else P)
    ne = int(cnx[Pe])
    Xh = Xd[:ne].cpu().pin_memory()
    Yh = Yd[:ne].cpu().pin_memory()
    sel_e = [p for p in mine if p < Pe]
    hc = torch.zeros((nm, P, 3), dtype=torch.int64).pin_memory()

    def e2e_pass():
        dcounts.zero_()
        for mi, mode in enumerate(modes):
            cfg = hap.make_cfg(HI.PERM_SEED, B, stream_id=(99 * P + mi) & 0xFFFFFFFF)
            if sel_e:
                hap.hap_permtest_batch(E.ctx.h, Xh, cnx[: Pe + 1], Yh, cny[: Pe + 1], mode, cfg,
                                       infos[mi], dcounts[mi], pair_sel=sel_e, stream=E.st)
        hc.copy_(dcounts, non_blocking=True)

    e2e_pass()  # warm-up: the host-input path's staging buffers and copy streams
    torch.cuda.synchronize()
    E.barrier()
    t0 = time.perf_counter()
    e2e_pass()
    torch.cuda.synchronize()
    e2e_s = E.max_over_ranks(time.perf_counter() - t0)
    e2e = {"value": Pe * nm / e2e_s, "unit": UNIT_T,
           "h2d_bytes_per_step": int(Xh.numel() * 4 * 2 * nm),
           "d2h_bytes_per_step": int(nm * P * 24), "steps": 1,
           "sample": f"the first {Pe} pairs of the batch (one step after one untimed warm-up "
                     "pass), inputs in pinned HOST memory",
           "timer": "host wall clock, synchronize on both sides"}
    cfg_out = {"workload": workload_desc(name, 0), "pairs": P, "B": B, "d": 768,
               "global_batch": P * nm, "l2": l2,
               "parallelism": f"pairs LPT-assigned (cost n_x+n_y) over {E.world} rank(s), one "
                              "hap_permtest_batch per rank and mode per step, then one "
                              "all_reduce of int64[P, info+3] rows (each written by one rank): "
                              "parallel.gpu_batch_sharded",
               "input_pool": (f"pair p = first n_p rows of pool pair p % 8 (8 distinct "
                              "5000/5000 vMF pairs)") if name == "c4" else
               f"{len(pool)} distinct pairs repeated"}
    extra = {"perms_per_s": perms,
             "mean_n": float(np.mean(sizes)),
             "rank_share_pairs": len(mine)}
    return value, ms, tw0, tw1, launches, roof, e2e, None, cfg_out, extra


def run_hap(args):
    peaks, peak_src = load_peaks()
    E = Env()
    gpu_id = None
    try:
        gpu_id = "GPU-" + str(E.torch.cuda.get_device_properties(E.local).uuid)
    except Exception:
        pass
    clocks = ClockSampler(gpu_id)
    clocks.start()
    time.sleep(0.3)
    fn = {"c2": run_c2, "c3": run_c3}.get(args.workload)
    if fn is None:
        res = run_batch_workload(args, E, peaks, args.workload)
    else:
        res = fn(args, E, peaks)
    value, ms, tw0, tw1, launches, roof, e2e, cpu, cfg_out, extra = res
    clocks.stop()
    clk = clocks.summary(tw0, tw1)
    roof["peaks_source"] = peak_src
    W = WORKLOADS[args.workload]
    if E.rank == 0:
        out = {"metric": W["metric"], "value": value, "unit": W["unit"], "n_gpus": E.world,
               "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms / args.steps,
               "higher_is_better": True, "scaling": W["scaling"], "vs_baseline": None,
               "dtype": "bf16", "data": "synthetic", "config": cfg_out, "roofline": roof,
               "cpu_baseline": cpu, "e2e": e2e, "clocks": clk,
               "gpu_launches": int(sum(launches.values())),
               "gpu_launches_by_phase": launches, "env_knobs": "none (HAP_* refused)"}
        out.update(extra)
        print(json.dumps(out), flush=True)
    E.ctx.close()
    if E.world > 1:
        E.dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="hap", choices=["hap", "reference"])
    ap.add_argument("--workload", default="c2", choices=sorted(WORKLOADS))
    ap.add_argument("--tests-per-step", type=int, default=TESTS_PER_STEP)
    ap.add_argument("--pool", type=int, default=24, help="distinct input pairs per rank")
    ap.add_argument("--e2e-steps", type=int, default=10)
    ap.add_argument("--no-cpu-baseline", action="store_true")
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3)
    knobs = sorted(k for k in os.environ if k.startswith("HAP_"))
    if knobs:
        print(json.dumps({"metric": WORKLOADS[args.workload]["metric"], "value": None,
                          "refused": f"HAP_* experiment knobs set: {knobs}; bench.py measures "
                                     "the library as built, unset them"}), flush=True)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args)
    else:
        run_hap(args)


if __name__ == "__main__":
    main()
