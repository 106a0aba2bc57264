"""The multi-GPU host path with the CUDA library on every rank: two processes (gloo process
group; both ranks on cuda:0 of the one-GPU test box — their kernels never wait on each
other, only the host-side all-reduce joins them) run config C3's b-range sharding
(parallel.gpu_range_counts) and config C4's LPT pair sharding (parallel.gpu_batch_sharded)
through libhap; the combined counts and infos must equal the world-1 run bit for bit, and
the counts must match the fp64 oracle within the tie-flagged permutations."""
import os
import socket

import numpy as np
import pytest
import torch.multiprocessing as mp

import hap_inputs as HI

pytestmark = pytest.mark.gpu

B_RANGE = 3000
B_BATCH = 1500
SIZES = [(300, 280), (50, 61), (1000, 990), (7, 9), (420, 400), (123, 150), (64, 64)]


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _inputs():
    X, Y = HI.make_pair(HI.PairSpec(700, 650, 768, HI.kappa_for(768), HI.kappa_for(768), 30.0,
                                    seed=21))
    xs, ys = [], []
    for p, (nx, ny) in enumerate(SIZES):
        a, b = HI.make_pair(HI.PairSpec(nx, ny, 768, 200.0, 200.0, 30.0, seed=300 + p))
        xs.append(a)
        ys.append(b)
    cnx = np.concatenate([[0], np.cumsum([n for n, _ in SIZES])]).astype(np.int64)
    cny = np.concatenate([[0], np.cumsum([n for _, n in SIZES])]).astype(np.int64)
    return X, Y, np.concatenate(xs), cnx, np.concatenate(ys), cny


def _run(rank, world, port, out_q):
    import torch
    import torch.distributed as dist

    import paper_2605_08048_b200 as hap
    from paper_2605_08048_b200 import parallel as par
    if world > 1:
        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        X, Y, Xp, cnx, Yp, cny = _inputs()
        ctx = hap.Context(0)
        counts = torch.zeros(3, dtype=torch.int64, device="cuda")
        info = torch.zeros(hap.INFO_BYTES, dtype=torch.uint8, device="cuda")
        par.gpu_range_counts(ctx, torch.from_numpy(X).cuda(), torch.from_numpy(Y).cuda(), B_RANGE,
                             HI.PERM_SEED, rank, world, counts, info, stream_id=9)
        infos, bc = par.gpu_batch_sharded(ctx, torch.from_numpy(Xp).cuda(), cnx,
                                          torch.from_numpy(Yp).cuda(), cny, B_BATCH, HI.PERM_SEED,
                                          rank, world, stream_id=40)
        st = hap.hap_sync(ctx.h)
        out_q.put((rank, st, counts.cpu().tolist(), bytes(infos.cpu().numpy().tobytes()),
                   bc.cpu().tolist()))
        ctx.close()
    finally:
        if world > 1:
            dist.destroy_process_group()


def _spawn(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_run, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=600) for _ in procs])
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    return res


def test_world2_cuda_equals_world1_and_oracle(orc):
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    one = _spawn(1)[0]
    two = _spawn(2)
    assert one[1] == 0 and all(r[1] == 0 for r in two)
    for rank, st, counts, infos, bc in two:
        assert counts == one[2], (rank, counts, one[2])
        assert infos == one[3]
        assert bc == one[4]
    # the combined counts against the fp64 oracle (decisions outside the tie band agree)
    X, Y, Xp, cnx, Yp, cny = _inputs()
    ref = orc.run_pair(X, Y, B_RANGE, HI.PERM_SEED, s=9)
    for k, key in enumerate(("exceed_ge", "exceed_abs")):
        assert abs(one[2][k] - ref[key]) <= ref["flagged"]
    for p in range(len(SIZES)):
        r = orc.run_pair(Xp[cnx[p]:cnx[p + 1]], Yp[cny[p]:cny[p + 1]], B_BATCH, HI.PERM_SEED,
                         s=40 + p)
        assert abs(one[4][p][0] - r["exceed_ge"]) <= r["flagged"], p
        assert abs(one[4][p][1] - r["exceed_abs"]) <= r["flagged"], p
