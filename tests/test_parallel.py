"""Multi-process sharding logic on CPU (gloo, world size 2): combined counts equal the
single-process counts.  The per-rank counter here is the oracle (test infrastructure);
on a GPU box the same functions drive the CUDA library (tests/test_gpu_parity.py and
bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import hap_inputs as HI
from paper_2605_08048_b200 import parallel as par


def test_shard_range_covers_exactly():
    for B in (1, 7, 1000, 100000):
        for W in (1, 2, 3, 8):
            rs = [par.shard_range(B, r, W) for r in range(W)]
            assert rs[0][0] == 0 and rs[-1][1] == B
            assert all(rs[i][1] == rs[i + 1][0] for i in range(W - 1))


def test_lpt_is_deterministic_and_balanced():
    sizes = HI.c4_sizes(1000)
    a = par.lpt_assign(sizes, 8)
    b = par.lpt_assign(sizes, 8)
    assert a == b
    assert sorted(i for lst in a for i in lst) == list(range(1000))
    loads = [sum(sizes[i] for i in lst) for lst in a]
    assert max(loads) - min(loads) <= max(sizes)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, out_q):
    import torch.distributed as dist

    import oracle
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        X, Y = HI.make_pair(HI.PairSpec(40, 50, 24, 20.0, 20.0, 45.0, seed=3))
        a = oracle.align(X, Y, 0)
        ob = oracle.observed(a.Z, 40)
        tau = oracle.tie_tau(ob["L1"], ob["L2"])
        run = lambda b0, b1: oracle.permtest(a.Z, 40, HI.PERM_SEED, 5, b0, b1, ob["T"], tau, 1)
        tot = par.permtest_sharded(run, 900, rank, world)
        sizes = [30, 55, 41, 70, 38]
        pairs = [HI.make_pair(HI.PairSpec(n, n + 3, 16, 15.0, 15.0, 40.0, seed=n)) for n in sizes]

        def run_pair(p):
            Xp, Yp = pairs[p]
            r = oracle.run_pair(Xp, Yp, 200, HI.PERM_SEED, s=p, nthreads=1)
            return [r["exceed_ge"], r["exceed_abs"], r["flagged"]]
        batch = par.batch_sharded(run_pair, [2 * n + 3 for n in sizes], rank, world)
        out_q.put((rank, tot.tolist(), batch.tolist()))
    finally:
        dist.destroy_process_group()


def test_gloo_world2_matches_single_process(orc):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    # single-process references
    X, Y = HI.make_pair(HI.PairSpec(40, 50, 24, 20.0, 20.0, 45.0, seed=3))
    ref = orc.run_pair(X, Y, 900, HI.PERM_SEED, s=5, nthreads=2)
    want = [ref["exceed_ge"], ref["exceed_abs"], ref["flagged"]]
    sizes = [30, 55, 41, 70, 38]
    want_b = []
    for p, n in enumerate(sizes):
        Xp, Yp = HI.make_pair(HI.PairSpec(n, n + 3, 16, 15.0, 15.0, 40.0, seed=n))
        r = orc.run_pair(Xp, Yp, 200, HI.PERM_SEED, s=p, nthreads=1)
        want_b.append([r["exceed_ge"], r["exceed_abs"], r["flagged"]])
    for rank, tot, batch in res:
        assert tot == want, (rank, tot, want)
        assert batch == want_b
