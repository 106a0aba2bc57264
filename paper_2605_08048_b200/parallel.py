"""Multi-GPU sharding of the permutation test (one process per GPU, torch.distributed).

Permutations are independent given the aligned pool and PERM-SPEC v1 is addressable by
`b` (R6), and word pairs are independent tests, so the path shards without any
data-path collective: each rank runs its share and the integer exceedance counts are
combined with ONE all_reduce(SUM) (NCCL over NVLink on B200; gloo in the CPU tests).
Counts are therefore identical for every world size.

The per-rank work is a callable, so the same host logic drives the CUDA library (the
product) and, in the CPU tests, any other counter of the same contract.
"""
from __future__ import annotations

from typing import Callable, Sequence

import numpy as np


def shard_range(B: int, rank: int, world: int) -> tuple[int, int]:
    """Rank r handles b in [floor(rB/W), floor((r+1)B/W))."""
    return (B * rank) // world, (B * (rank + 1)) // world


def lpt_assign(costs: Sequence[float], world: int) -> list[list[int]]:
    """Longest-processing-time-first assignment of items (pairs) to ranks; deterministic
    (ties broken by item index, then by rank index)."""
    order = sorted(range(len(costs)), key=lambda i: (-float(costs[i]), i))
    load = [0.0] * world
    out: list[list[int]] = [[] for _ in range(world)]
    for i in order:
        r = min(range(world), key=lambda k: (load[k], k))
        out[r].append(i)
        load[r] += float(costs[i])
    for lst in out:
        lst.sort()
    return out


def _allreduce_sum(vec: np.ndarray, group=None, device=None) -> np.ndarray:
    import torch
    import torch.distributed as dist
    t = torch.from_numpy(np.ascontiguousarray(vec, dtype=np.int64))
    if device is not None:
        t = t.to(device)
    dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
    return t.cpu().numpy()


def permtest_sharded(run_range: Callable[[int, int], np.ndarray], B: int, rank: int, world: int,
                     group=None, device=None) -> np.ndarray:
    """One pair, b-range sharding (config C3): every rank aligns the same pair (a
    deterministic replica) and counts its b-range; one all_reduce of int64[3]."""
    b0, b1 = shard_range(B, rank, world)
    local = np.asarray(run_range(b0, b1), dtype=np.int64).reshape(3)
    if world == 1:
        return local
    return _allreduce_sum(local, group, device)


def batch_sharded(run_pair: Callable[[int], np.ndarray], sizes: Sequence[int], rank: int,
                  world: int, group=None, device=None) -> np.ndarray:
    """Many pairs (configs C4/C5): LPT over the pair costs N_p, each rank fills its pairs'
    rows of a zero int64[P, 3] buffer, one all_reduce combines them."""
    P = len(sizes)
    mine = lpt_assign(sizes, world)[rank]
    buf = np.zeros((P, 3), dtype=np.int64)
    for p in mine:
        buf[p] = np.asarray(run_pair(p), dtype=np.int64).reshape(3)
    if world == 1:
        return buf
    return _allreduce_sum(buf, group, device).reshape(P, 3)


def allreduce_device(t, group=None) -> None:
    """In-place SUM all-reduce of a device tensor: NCCL reduces on the device; other
    backends (gloo in the multi-process tests) go through a host copy."""
    import torch.distributed as dist
    if dist.get_backend(group) == "nccl":
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        return
    h = t.cpu()
    dist.all_reduce(h, op=dist.ReduceOp.SUM, group=group)
    t.copy_(h)


def gpu_range_counts(ctx, X, Y, B: int, seed: int, rank: int, world: int, counts, info,
                     stream_id: int = 0, mode: int = 0, group=None, stream=None,
                     reduce: bool = True) -> None:
    """Config C3 on the CUDA library, asynchronous: every rank aligns the same pair (the
    K1 arithmetic is deterministic, so every rank builds bit-identical planes), counts its
    b-range shard into `counts` (device int64[3], added into) and ONE all-reduce combines
    the ranks.  Nothing synchronises the host."""
    import paper_2605_08048_b200 as hap
    b0, b1 = shard_range(B, rank, world)
    hap.hap_align(ctx.h, X, Y, mode, info, stream=stream)
    if b1 > b0:
        cfg = hap.make_cfg(seed, B, b0, b1, stream_id)
        hap.hap_permtest(ctx.h, info, cfg, counts, None, stream=stream)
    if world > 1 and reduce:
        allreduce_device(counts, group)


def gpu_range_runner(ctx, X, Y, B: int, seed: int, stream_id: int = 0, mode: int = 0):
    """run_range for the CUDA library: align once, then count any b-range."""
    import paper_2605_08048_b200 as hap
    import torch

    def run(b0: int, b1: int) -> np.ndarray:
        ctx.counts.zero_()
        hap.hap_align(ctx.h, X, Y, mode, ctx.info)
        cfg = hap.make_cfg(seed, B, b0, b1, stream_id)
        hap.hap_permtest(ctx.h, ctx.info, cfg, ctx.counts, None)
        st = hap.hap_sync(ctx.h)
        if st != hap.HAP_OK:
            raise hap.HapError(st, hap.hap_last_error(ctx.h))
        return ctx.counts.cpu().numpy()
    del torch
    return run


def gpu_batch_sharded(ctx, X_packed, cu_nx, Y_packed, cu_ny, B: int, seed: int, rank: int,
                      world: int, stream_id: int = 0, mode: int = 0, group=None,
                      reduce: bool = True):
    """Configs C4/C5 on the CUDA library: the pairs are LPT-assigned by cost N_p, each rank
    runs its share with ONE hap_permtest_batch call (pair_sel), and one all_reduce(SUM) on
    the device combines int64[P, INFO_WORDS + 3] = the bit-cast hap_align_info rows plus
    the counts (every row is written by exactly one rank, the rest are zero, so the sum
    reproduces the bits).  Returns (infos uint8[P, INFO_BYTES], counts int64[P, 3]) on the
    device, identical on every rank and for every world size."""
    import paper_2605_08048_b200 as hap
    import torch

    P = len(cu_nx) - 1
    assert hap.INFO_BYTES % 8 == 0
    iw = hap.INFO_BYTES // 8
    cnx = np.asarray(cu_nx, dtype=np.int64)
    cny = np.asarray(cu_ny, dtype=np.int64)
    costs = (cnx[1:] - cnx[:-1]) + (cny[1:] - cny[:-1])
    mine = lpt_assign(costs.tolist(), world)[rank]
    buf = torch.zeros((P, iw + 3), dtype=torch.int64, device=ctx.device)
    infos = buf[:, :iw]
    counts = buf[:, iw:]
    cfg = hap.make_cfg(seed, B, 0, B, stream_id)
    if mine:
        # infos / counts are row-strided views: the C ABI takes dense arrays, so stage them
        inf_d = torch.zeros((P, hap.INFO_BYTES), dtype=torch.uint8, device=ctx.device)
        cnt_d = torch.zeros((P, 3), dtype=torch.int64, device=ctx.device)
        hap.hap_permtest_batch(ctx.h, X_packed, cnx, Y_packed, cny, mode, cfg, inf_d, cnt_d,
                               pair_sel=mine, stream=torch.cuda.current_stream(ctx.device))
        infos.copy_(inf_d.view(torch.int64))
        counts.copy_(cnt_d)
    if world > 1 and reduce:
        allreduce_device(buf, group)
    return buf[:, :iw].contiguous().view(torch.uint8), buf[:, iw:].contiguous()
