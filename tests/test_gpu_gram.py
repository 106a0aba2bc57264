"""GPU parity of the Gram form of the mask-GEMM (DESIGN.md
"Gram form", include/hap.h HAP_FLAG_GRAM): the same bars as the plane form against the fp64
oracle (tests/test_gpu_parity.py check_pair), over ragged shapes, singleton groups, narrow
clouds, both K3 CTA modes, b-range shards, waves, shared masks and the automatic choice."""
import numpy as np
import pytest

import hap_inputs as HI
from test_gpu_parity import SEED, _cuda, check_pair

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def hap():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("no GPU")
    from paper_2605_08048_b200 import build
    build.build()
    import paper_2605_08048_b200 as h
    return h


@pytest.fixture(scope="module")
def ctx(hap):
    c = hap.Context(0)
    yield c
    c.close()


@pytest.mark.parametrize("pair_mode", [1, 2])
def test_gram_config1(ctx, orc, pair_mode):
    """C1 (n_x = n_y = 64, d = 768, B = 1000) through the Gram form, every permutation."""
    X, Y = HI.config_pair("C1")
    check_pair(ctx, orc, X, Y, 1000, s=1, pair_mode=pair_mode, gram=True)


@pytest.mark.parametrize("n_x,n_y,d,B", [(37, 50, 100, 300), (5, 3, 3, 200), (1, 70, 768, 257),
                                         (70, 1, 40, 129), (200, 150, 4096, 700),
                                         (300, 200, 1024, 600), (129, 127, 2048, 1100),
                                         (1000, 1000, 768, 300)])
def test_gram_shapes(ctx, orc, n_x, n_y, d, B):
    """Ragged N (Gram tiles of 32 rows, N_pad a multiple of 64), N_pad above and below d,
    several K3 tiles with a ragged tail, groups of one, N_pad up to 2048."""
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, 30.0 + d / 10, 60.0 + d / 10, 40.0, seed=n_x * 3 + d))
    check_pair(ctx, orc, X, Y, B, s=7, gram=True)


@pytest.mark.parametrize("r", [0.96, 0.99])
def test_gram_narrow_clouds(ctx, orc, r):
    """Narrow clouds (MRL ~ r): the quadratic form of a cloud near r = 1."""
    d = 768
    k = HI.kappa_for_r(d, r)
    X, Y = HI.make_pair(HI.PairSpec(150, 170, d, k, k, 5.0, seed=31))
    check_pair(ctx, orc, X, Y, 800, s=2, gram=True)


def test_gram_shards_and_naive_mode(ctx, orc):
    """A b-range shard and the naive (unaligned) pooling through the Gram form."""
    X, Y = HI.make_pair(HI.PairSpec(90, 110, 1536, HI.kappa_for(1536), HI.kappa_for(1536), 60.0, seed=5))
    check_pair(ctx, orc, X, Y, 3000, s=4, b_begin=700, b_end=1900, gram=True)
    check_pair(ctx, orc, X, Y, 600, s=4, mode=1, gram=True)


def test_gram_choice_is_automatic_and_consistent(hap, ctx, orc):
    """For N << d and a large B the library takes the Gram form by itself (one more
    alignment-phase launch: the Gram kernel; one more generator-phase launch per block: the
    bit packing) and then gives bitwise the forced-Gram result; the plane form agrees with
    the oracle on the same input."""
    d = 4096
    X, Y = HI.make_pair(HI.PairSpec(100, 100, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=8))
    B = 200000
    hap.hap_profile_read(ctx.h, reset=True)
    auto = ctx.permtest_pair(_cuda(X), _cuda(Y), B, SEED, stream_id=3)
    la = hap.hap_profile_read(ctx.h, reset=True)[1]
    forced = ctx.permtest_pair(_cuda(X), _cuda(Y), B, SEED, stream_id=3, gram=True)
    planes = ctx.permtest_pair(_cuda(X), _cuda(Y), B, SEED, stream_id=3, gram=False)
    lp = hap.hap_profile_read(ctx.h, reset=True)[1]
    for k in ("gemm_t_obs", "exceed_ge", "exceed_abs", "flagged"):
        assert auto[k] == forced[k], k
    assert la["align"] >= 4  # K1s (3 kernels) + the Gram kernel
    assert la["permgen"] > la["maskgemm"] - 1  # a bit-packing launch per generator launch
    ref = orc.run_pair(X, Y, 4000, SEED, s=3)  # oracle on the first 4000 permutations
    g4 = ctx.permtest_pair(_cuda(X), _cuda(Y), 4000, SEED, stream_id=3, gram=True)
    p4 = ctx.permtest_pair(_cuda(X), _cuda(Y), 4000, SEED, stream_id=3, gram=False)
    for res in (g4, p4):
        for k in ("exceed_ge", "exceed_abs"):
            assert abs(res[k] - ref[k]) <= ref["flagged"], k
    assert abs(planes["exceed_ge"] - auto["exceed_ge"]) <= auto["flagged"] + planes["flagged"]


@pytest.mark.parametrize("shared", [False, True])
def test_gram_batch_matches_single_pairs(ctx, orc, shared):
    """A varlen batch through the Gram form (waves of up to 4 tests, each with its own Gram
    planes and mask bits; shared=True: equal-size pairs share one mask block and its bits)
    gives bitwise the single-pair results, and matches the oracle."""
    sizes = [120, 120, 120, 64, 64, 200, 120, 33] if not shared else [120] * 6 + [64] * 3
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=1024)
    X, Y = _cuda(Xp), _cuda(Yp)
    B, s0 = 1300, 40
    res = ctx.permtest_batch(X, cnx, Y, cny, B, SEED, stream_id=s0, shared=shared, gram=True)
    for p in range(len(sizes)):
        Xq, Yq = Xp[cnx[p]:cnx[p + 1]], Yp[cny[p]:cny[p + 1]]
        s = s0 if shared else s0 + p
        one = ctx.permtest_pair(_cuda(Xq), _cuda(Yq), B, SEED, stream_id=s, gram=True)
        for k in ("gemm_t_obs", "exceed_ge", "exceed_abs", "flagged"):
            assert one[k] == res[p][k], (p, k)
        if p % 3 == 0:
            ref = orc.run_pair(Xq, Yq, B, SEED, s=s)
            for k in ("exceed_ge", "exceed_abs"):
                assert abs(res[p][k] - ref[k]) <= ref["flagged"], (p, k)


def test_gram_mixed_wave(ctx, orc):
    """One wave holding Gram-form and plane-form tests (the forced flag applies to pairs
    with N_pad <= 4096 only; a 4100-row pair stays in the plane form) in one K3 launch."""
    sizes = [2100, 60, 2050, 70]
    ny = [2000, 50, 2050, 90]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=768, ny_sizes=ny)
    X, Y = _cuda(Xp), _cuda(Yp)
    res = ctx.permtest_batch(X, cnx, Y, cny, 700, SEED, stream_id=9, gram=True, wave=4)
    for p in range(len(sizes)):
        Xq, Yq = Xp[cnx[p]:cnx[p + 1]], Yp[cny[p]:cny[p + 1]]
        ref = orc.run_pair(Xq, Yq, 700, SEED, s=9 + p)
        Ls = abs(ref["L_x"]) + abs(ref["L_y"])
        assert abs(res[p]["gemm_t_obs"] - ref["t_obs"]) <= 1e-5 * Ls
        for k in ("exceed_ge", "exceed_abs"):
            assert abs(res[p][k] - ref[k]) <= ref["flagged"], (p, k)
