"""GPU parity: the CUDA path (through the C ABI) vs the fp64 oracle, element by element
on the same seeded inputs.  Bars:
  * permutation index sets: bit-exact;
  * r1, r2 (and r_X, r_Y): relative 1e-5; L: relative 1e-5;
  * T: |dT| <= 1e-5 (|L1| + |L2|)  (T is a near-zero difference, D6);
  * counts: every permutation outside the tie band tau decides identically, so
    |c_gpu - c_oracle| <= flagged (tie band tau = 1e-6 (|L_X| + |L_Y|), R8).
"""
import math
import os

import numpy as np
import pytest

import hap_inputs as HI

pytestmark = pytest.mark.gpu

SEED = HI.PERM_SEED


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


def _cuda(a):
    import torch
    return torch.from_numpy(np.ascontiguousarray(a)).cuda()


def check_pair(ctx, orc, X, Y, B, s=0, mode=0, block=0, b_begin=0, b_end=None, pair_mode=0, gram=None):
    """Run both sides with stats; assert the parity bars; return (gpu, ref).  gram: K3 form
    (None = the library's choice, True = Gram form, False = plane form)."""
    b_end = B if b_end is None else b_end
    g = ctx.permtest_pair(_cuda(X), _cuda(Y), B, SEED, stream_id=s, mode=mode, block=block,
                          b_begin=b_begin, b_end=b_end, want_stats=True, pair_mode=pair_mode,
                          gram=gram)
    ref = orc.run_pair(X, Y, B, SEED, s=s, mode=mode, b_begin=b_begin, b_end=b_end,
                       want_stats=True)
    Ls = abs(ref["L_x"]) + abs(ref["L_y"])
    # observed statistic: fp64 on both sides (K1 means vs oracle direct sums)
    assert math.isclose(g["r_x"], ref["r_x"], rel_tol=1e-10)
    assert math.isclose(g["r_y"], ref["r_y"], rel_tol=1e-10)
    assert math.isclose(g["logk_x"], ref["L_x"], rel_tol=1e-10, abs_tol=1e-12)
    assert math.isclose(g["logk_y"], ref["L_y"], rel_tol=1e-10, abs_tol=1e-12)
    assert abs(g["t_obs"] - ref["t_obs"]) <= 1e-10 * Ls
    # the same-path observed value the permutations were compared against
    assert math.isclose(g["gemm_r_x"], ref["r_x"], rel_tol=1e-5)
    assert math.isclose(g["gemm_r_y"], ref["r_y"], rel_tol=1e-5)
    assert abs(g["gemm_t_obs"] - ref["t_obs"]) <= 1e-5 * Ls
    gs = g["stats"].cpu().numpy()
    rs = ref["stats"]
    assert np.allclose(gs[:, 0], rs[:, 0], rtol=1e-5, atol=0)
    assert np.allclose(gs[:, 1], rs[:, 1], rtol=1e-5, atol=0)
    assert np.all(np.abs(gs[:, 2] - rs[:, 2]) <= 1e-5 * Ls)
    # decisions identical outside the tie bands (GPU compares against its same-path T_obs)
    tau = ref["tau"]
    tg = g["gemm_t_obs"]
    out = np.abs(rs[:, 2] - ref["t_obs"]) > tau
    assert np.array_equal(gs[out, 2] >= tg, rs[out, 2] >= ref["t_obs"])
    out2 = np.abs(np.abs(rs[:, 2]) - abs(ref["t_obs"])) > tau
    assert np.array_equal(np.abs(gs[out2, 2]) >= abs(tg), np.abs(rs[out2, 2]) >= abs(ref["t_obs"]))
    for k in ("exceed_ge", "exceed_abs"):
        assert abs(g[k] - ref[k]) <= ref["flagged"], (k, g[k], ref[k], ref["flagged"])
    return g, ref


# ------------------------------------------------------------------ K2 (index sets)
@pytest.mark.parametrize("N,n_x", [(2, 1), (10, 4), (8, 4), (128, 64), (100, 37), (2000, 1000),
                                   (2000, 1), (2000, 1999), (4097, 2500), (65535, 32767)])
def test_perm_sets_bit_exact(hap, ctx, orc, N, n_x):
    import torch
    count = 64 if N < 10000 else 6
    for s, b0 in [(0, 0), (5, 123456), (0xFFFFFFFF, 2**32 - count)]:
        out = torch.empty((count, N), dtype=torch.uint8, device="cuda")
        hap.hap_perm_sets(ctx.h, SEED, s, b0, count, N, n_x, out)
        got = out.cpu().numpy()
        for i in range(count):
            want = orc.perm_set(SEED, s, b0 + i, N, n_x)
            assert np.array_equal(got[i], want), (N, n_x, s, b0 + i)


def test_perm_sets_golden(hap, ctx):
    """The product generator reproduces the SURVEY golden sets directly."""
    import torch
    from conftest import read_golden
    for row in read_golden("permspec_v1.txt"):
        lhs, rhs = row.split(":")
        seed, s, b, N, n = lhs.split()
        out = torch.empty((1, int(N)), dtype=torch.uint8, device="cuda")
        hap.hap_perm_sets(ctx.h, int(seed, 16), int(s), int(b), 1, int(N), int(n), out)
        assert np.nonzero(out.cpu().numpy()[0])[0].tolist() == [int(x) for x in rhs.split()]


def test_perm_sets_side_stream_golden(hap, ctx):
    """The product generator on the Lemire-rejection golden sets (independent pure-Python
    generator, tests/golden/gen_permspec_rejections.py) at the pooled sizes it supports."""
    import hashlib
    import torch
    from test_oracle import _rejection_rows
    rows = [r for r in _rejection_rows() if r[3] <= 65535]
    assert len(rows) >= 6
    for seed, s, b, N, n, rej, kind, want in rows:
        out = torch.empty((1, N), dtype=torch.uint8, device="cuda")
        hap.hap_perm_sets(ctx.h, seed, s, b, 1, N, n, out)
        members = np.nonzero(out.cpu().numpy()[0])[0].tolist()
        if kind == "sha":
            assert hashlib.sha256(" ".join(map(str, members)).encode()).hexdigest() == want, (s, b)
        else:
            assert members == [int(x) for x in want.split()], (s, b, N, n)


# ------------------------------------------------------------------ K1 (pooled planes)
@pytest.mark.parametrize("n_x,n_y,d,mode", [(64, 64, 768, 0), (37, 50, 100, 0), (1000, 1000, 768, 0),
                                            (300, 200, 64, 1), (5, 3, 3, 0),
                                            # fused cooperative K1 (d % 4 != 0), lean K1s with
                                            # d > 1024 (block variant), warp variant at d = 1024
                                            (40, 50, 770, 0), (300, 200, 766, 1), (100, 120, 1028, 0),
                                            (2000, 1000, 2048, 0), (129, 3, 1024, 0),
                                            # streaming K1s path (n_pad d >= 8 Mi): R = 4 / 8
                                            # row items, an item straddling X | Y, naive mode
                                            (1024, 1024, 4096, 0), (3001, 1500, 2048, 0),
                                            (2731, 10, 3072, 1)])
def test_pooled_planes(hap, ctx, orc, n_x, n_y, d, mode):
    import torch
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, 40.0, 40.0, 50.0, seed=d + n_x))
    ctx.permtest_pair(_cuda(X), _cuda(Y), 128, SEED, mode=mode)
    n_pad = -(-(n_x + n_y) // 64) * 64
    d_pad = -(-d // 32) * 32
    zh = torch.empty((d_pad, n_pad), dtype=torch.int16, device="cuda")
    zl = torch.empty_like(zh)
    t = torch.empty(d_pad, dtype=torch.float64, device="cuda")
    m = torch.empty(d_pad, dtype=torch.float64, device="cuda")
    hap.hap_export_pooled(ctx.h, zh, zl, t, m)
    torch.cuda.synchronize()
    hi = zh.view(torch.bfloat16).float().double().cpu().numpy().T
    lo = zl.view(torch.bfloat16).float().double().cpu().numpy().T
    mm = m.cpu().numpy()
    ref = orc.align(X, Y, mode)
    N = n_x + n_y
    # the planes hold the centred cloud z - m (m a multiple of 2^-12, ~ t/N)
    assert np.all(mm * 4096 == np.round(mm * 4096)) and np.all(mm[d:] == 0)
    assert np.allclose(mm[:d], ref.Z.sum(0) / N, atol=2.0 ** -13 + 1e-9)
    zc = hi[:N, :d] + lo[:N, :d]
    want = ref.Z - mm[None, :d]
    # bf16 hi+lo keeps 16 mantissa bits of z - m, computed in fp32 (abs. error < 2^-22)
    assert np.all(np.abs(zc - want) <= 2.0 ** -16 * np.abs(want) + 2.0 ** -22)
    assert np.all(hi[N:] == 0) and np.all(lo[N:] == 0)
    assert np.all(hi[:, d:] == 0) and np.all(lo[:, d:] == 0)
    tt = t.cpu().numpy()
    assert np.allclose(tt[:d], zc.sum(0) + N * mm[:d], rtol=1e-12, atol=1e-12)
    # t against the oracle's exact column sums: the per-element bound above, summed
    bound = (2.0 ** -16 * np.abs(want) + 2.0 ** -22).sum(0) + 1e-9
    assert np.all(np.abs(tt[:d] - ref.Z.sum(0)) <= bound)


# ------------------------------------------------------------------ K3 + end to end
@pytest.mark.parametrize("pair_mode", [1, 2])
def test_config1_full(ctx, orc, pair_mode):
    """C1: n_x=n_y=64, d=768, B=1000, every permutation compared; both K3 modes
    (cta_group::1, M=128 and cta_group::2, M=256)."""
    X, Y = HI.config_pair("C1")
    check_pair(ctx, orc, X, Y, 1000, s=1, pair_mode=pair_mode)


@pytest.mark.parametrize("pair_mode", [1, 2])
@pytest.mark.parametrize("n_x,n_y,d,B,block", [(37, 50, 100, 300, 128), (2, 70, 48, 257, 0),
                                               (70, 2, 40, 129, 0), (1, 70, 48, 257, 0),
                                               (70, 1, 40, 129, 0), (200, 300, 300, 1000, 256),
                                               (5, 3, 3, 200, 0), (64, 64, 544, 700, 300)])
def test_ragged_shapes(ctx, orc, n_x, n_y, d, B, block, pair_mode):
    """Ragged N (not a multiple of 64), d not a multiple of 32 (last d-chunk narrower than
    256), several tiles with a ragged tail, multi-launch blocks, two-row groups."""
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, 30.0, 60.0, 40.0, seed=n_x * 7 + d))
    check_pair(ctx, orc, X, Y, B, s=3, block=block, pair_mode=pair_mode)


@pytest.mark.parametrize("d", [4096, 9000, 16384])
def test_wide_dimension(ctx, orc, d):
    """K1 item geometry for wide rows: fewer rows per smem tile (8 / 4 / 2), per-column
    axis/centre computed on the fly and t' partials straight to the accumulators."""
    X, Y = HI.make_pair(HI.PairSpec(37, 41, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=9))
    check_pair(ctx, orc, X, Y, 300, s=3)


@pytest.mark.parametrize("n_x,n_y,d", [(1, 70, 48), (70, 1, 768), (1, 1, 8), (1, 300, 4096)])
def test_singleton_group(ctx, orc, n_x, n_y, d):
    """A group of one unit vector has MRL exactly 1 (Eq. 8), so its L sits at the clamp
    r = 1 - 1e-9 (R4) for every split: full parity bars, and the single side's r is exactly 1
    in every permutation (n_x = n_y = 1: T = 0 for every split, all ties, all counted)."""
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, 30.0 + d, 60.0 + d, 40.0, seed=11 + d))
    g, ref = check_pair(ctx, orc, X, Y, 300)
    gs = g["stats"].cpu().numpy()
    if n_x == 1:
        assert np.all(gs[:, 0] == 1.0)
    if n_y == 1:
        assert np.all(gs[:, 1] == 1.0)
    if n_x == n_y == 1:
        assert np.all(gs[:, 2] == 0.0) and g["exceed_ge"] == 300 == ref["exceed_ge"]


def _eps_rep(hap, ctx, d):
    """The test's representation-error scale as K1 forms it (R14), from the
    exported centre m: 2^-17 sqrt(1 - ||m||^2) + 2^-23."""
    import torch
    d_pad = -(-d // 32) * 32
    n_pad = int(hap.decode_info(ctx.info).n_pad)
    zh = torch.empty((d_pad, n_pad), dtype=torch.int16, device="cuda")
    t = torch.empty(d_pad, dtype=torch.float64, device="cuda")
    m = torch.empty(d_pad, dtype=torch.float64, device="cuda")
    hap.hap_export_pooled(ctx.h, zh, torch.empty_like(zh), t, m)
    mm = m.cpu().numpy()
    return 2.0 ** -17 * math.sqrt(max(1.0 - float(mm @ mm), 0.0)) + 2.0 ** -23


def _l_width(r, n, eps, d, n_mask=None, gram=False):
    """DESIGN.md R14 (mirror of k_maskgemm.cu row_stat / l_width): half-width of the interval
    holding L(r) given the GPU's r and |dr| <= 8 eps / sqrt(n d) (+ R14b: the accumulation
    over the masked group's n_mask rows, or the Gram form's dS of n_mask^2 entries)."""
    r = np.asarray(r, dtype=np.float64)
    if n == 1:
        return np.zeros_like(r)
    n_mask = n if n_mask is None else n_mask
    delta = 8.0 * eps / math.sqrt(n * d)
    if gram:
        dS = 8.0 * 4.0 * math.sqrt(1.0 + n_mask / d) * (2.0 ** -17 * math.sqrt(n_mask) + 2.0 ** -22 * n_mask)
        delta = delta + dS / (2.0 * n * n * np.maximum(r, 1e-6))
    else:
        delta = delta + 2.0 ** -22 * n_mask / (math.sqrt(d) * n)

    def q(x):
        x = np.minimum(x, 1 - 1e-9)
        return x * (d - x * x) / (1 - x * x)
    with np.errstate(divide="ignore", invalid="ignore"):
        near = r + 2 * delta >= 1 - 1e-9
        w = np.where(near, np.log(q(np.ones_like(r)) / q(np.maximum(r - 2 * delta, 1e-300))),
                     2 * delta * (1 / r + 2 * r / (1 - r * r)))
    return np.where(r <= 2 * delta, np.inf, w)


def check_certified(hap, ctx, orc, X, Y, B, s=0, mode=0, block=0, pair_mode=0, gram=None):
    """R14 at any r: the GPU's error bound e_T covers its actual error on every permutation
    (and on T_obs); every decision outside the widened band matches the oracle; the GPU
    flags a superset of the oracle's near-ties, and the counts differ by at most those."""
    g = ctx.permtest_pair(_cuda(X), _cuda(Y), B, SEED, stream_id=s, want_stats=True, mode=mode,
                          block=block, pair_mode=pair_mode, gram=gram)
    ref = orc.run_pair(X, Y, B, SEED, s=s, want_stats=True, mode=mode)
    d, n_x, n_y = X.shape[1], X.shape[0], Y.shape[0]
    eps = _eps_rep(hap, ctx, d)
    gs, rs = g["stats"].cpu().numpy(), ref["stats"]
    gf = hap.hap_debug_last_form(ctx.h) == 1
    e = _l_width(gs[:, 0], n_x, eps, d, n_x, gf) + _l_width(gs[:, 1], n_y, eps, d, n_x, gf)
    e_obs = float(_l_width(np.array([g["gemm_r_x"]]), n_x, eps, d, n_x, gf)[0] +
                  _l_width(np.array([g["gemm_r_y"]]), n_y, eps, d, n_x, gf)[0])
    assert abs(g["gemm_t_obs"] - ref["t_obs"]) <= e_obs + 1e-6 * (abs(ref["L_x"]) + abs(ref["L_y"]))
    assert np.all(np.abs(gs[:, 2] - rs[:, 2]) <= e + 1e-7 * (abs(ref["L_x"]) + abs(ref["L_y"])))
    band = ref["tau"] + e + e_obs
    tg = g["gemm_t_obs"]
    out = np.abs(gs[:, 2] - tg) > band
    assert np.array_equal(gs[out, 2] >= tg, rs[out, 2] >= ref["t_obs"])
    out2 = np.abs(np.abs(gs[:, 2]) - abs(tg)) > band
    assert np.array_equal(np.abs(gs[out2, 2]) >= abs(tg), np.abs(rs[out2, 2]) >= abs(ref["t_obs"]))
    assert g["flagged"] >= ref["flagged"]
    for k in ("exceed_ge", "exceed_abs"):
        assert abs(g[k] - ref[k]) <= g["flagged"], (k, g[k], ref[k], g["flagged"])
    return g, ref


@pytest.mark.parametrize("d", [768, 4096])
@pytest.mark.parametrize("r", [0.96, 0.99, 0.999])
@pytest.mark.parametrize("n_x,n_y", [(2, 70), (64, 64), (500, 500)])
def test_narrow_clouds(ctx, orc, d, r, n_x, n_y):
    """Narrow words (r ~ 0.96, Table 4 colitis) up to r = 0.999, where L is
    ill-conditioned (dL/dr ~ 1/(1 - r), "drift near r ~ 1"): the full parity bars
    (1e-5 Ls on T, decisions outside tau, counts within the oracle's flagged)."""
    if d == 4096 and n_x == 500:
        n_x = n_y = 300
    k = HI.kappa_for_r(d, r)
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, k, k, 30.0, seed=int(r * 1e4) + d + n_x))
    check_pair(ctx, orc, X, Y, 1500, s=6)


@pytest.mark.parametrize("d,r,n_x,n_y", [(48, 0.9999, 2, 70), (768, 0.9999, 64, 64),
                                         (768, 0.9999, 1000, 1000), (4096, 0.9999, 300, 300),
                                         (768, 0.75, 1000, 1000), (48, 0.999, 2, 70)])
def test_certified_band_near_unit_mrl(hap, ctx, orc, d, r, n_x, n_y):
    """Beyond r = 0.999 the two-term bf16 path's T error exceeds the plain tie band; the
    kernel's error bound (R14) widens the band so that every decision it does not flag is
    still the oracle's (and the bound holds at ordinary r too)."""
    k = HI.kappa_for_r(d, r)
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, k, k, 30.0, seed=int(r * 1e4) + d + n_x))
    check_certified(hap, ctx, orc, X, Y, 2000, s=5)


@pytest.mark.parametrize("d", [48, 768])
@pytest.mark.parametrize("n_x,n_y,ndx,ndy", [(3, 40, 1, 8), (5, 5, 2, 2), (64, 64, 4, 16),
                                             (300, 200, 8, 8), (12, 12, 1, 12)])
def test_duplicated_rows(hap, ctx, orc, d, n_x, n_y, ndx, ndy):
    """Clouds with duplicated rows (identical contexts give identical embeddings): 70 % of
    each cloud's rows are copies of a few distinct ones, so some permuted groups - and with
    n_distinct = 1 the observed X itself - consist of identical vectors (r = 1 exactly)."""
    X, Y = HI.duplicated_pair(HI.PairSpec(n_x, n_y, d, HI.kappa_for(d), HI.kappa_for(d), 30.0,
                                          seed=77 + n_x), n_distinct_x=ndx, n_distinct_y=ndy, frac=0.7)
    check_certified(hap, ctx, orc, X, Y, 1500, s=4)


def test_naive_mode(ctx, orc):
    X, Y = HI.make_pair(HI.PairSpec(120, 90, 256, 100.0, 100.0, 90.0, seed=4))
    g, ref = check_pair(ctx, orc, X, Y, 500, mode=1)
    assert g["is_identity"]


def test_config2_full(ctx, orc):
    """C2 (the metric's configuration): n_x=n_y=1000, d=768, B=10^4, all b compared."""
    X, Y = HI.config_pair("C2")
    check_pair(ctx, orc, X, Y, 10000, s=2)


def test_config3_sampled(ctx, orc):
    """C3 shape (n_x=n_y=5000, d=4096): a b-range shard far from 0, every b of it
    compared (full B=10^5 runs in test_sharding / bench)."""
    X, Y = HI.config_pair("C3")
    check_pair(ctx, orc, X, Y, 100000, s=3, b_begin=77000, b_end=77300)


def test_worked_example_counts_exact(ctx, orc):
    """SURVEY worked example (d=3): T values are >= 0.0155 apart from T_obs, so the
    one-sided count must be identical, and the MC p approaches the exhaustive 12/70.
    (With n_x = n_y the complement split has T = -T_obs exactly: a true two-sided tie,
    which the tie band flags, so the two-sided count is only checked within `flagged`.)"""
    from conftest import read_golden
    rows = read_golden("worked_example.txt")
    X = np.array([[float(v) for v in r.split()[1:]] for r in rows if r.startswith("X ")], np.float32)
    Y = np.array([[float(v) for v in r.split()[1:]] for r in rows if r.startswith("Y ")], np.float32)
    g, ref = check_pair(ctx, orc, X, Y, 20000)
    assert g["exceed_ge"] == ref["exceed_ge"]
    assert abs(g["exceed_ge"] / 20000 - 12 / 70) < 4 * math.sqrt(12 / 70 * 58 / 70 / 20000)


def test_dyadic_exact(ctx, orc):
    """Dyadic unit rows in naive mode: every sum is exact on both sides, so r1, r2 are
    bit-identical to the oracle."""
    rng = np.random.default_rng(0)
    X, Y = HI.dyadic_pair(rng, 7, 9, 64)
    g, ref = check_pair(ctx, orc, X, Y, 512, mode=1)
    gs = g["stats"].cpu().numpy()
    assert np.array_equal(gs[:, 0], ref["stats"][:, 0])
    assert np.array_equal(gs[:, 1], ref["stats"][:, 1])


def test_duplicate_sets_tie_bit_exactly(ctx, orc):
    """N=4, n=2: only 6 distinct splits, so many b repeat the observed split; those T
    must equal T_obs bit-exactly (same GEMM + epilogue path, D7) and count as >=."""
    X = np.array([[1, 0.2, 0], [0.3, 1, 0]], np.float32)
    Y = np.array([[0, 0.1, 1], [1, 1, 1]], np.float32)
    g, ref = check_pair(ctx, orc, X, Y, 600)
    gs = g["stats"].cpu().numpy()
    sets = [tuple(np.nonzero(orc.perm_set(SEED, 0, b, 4, 2))[0]) for b in range(600)]
    obs = [i for i, s in enumerate(sets) if s == (0, 1)]
    assert len(obs) > 50
    assert np.all(gs[obs, 2] == g["gemm_t_obs"])
    assert g["exceed_ge"] == ref["exceed_ge"]


def _export_planes(hap, ctx, n_pad, d_pad):
    import torch
    zh = torch.empty((d_pad, n_pad), dtype=torch.int16, device="cuda")
    zl = torch.empty_like(zh)
    t = torch.empty(d_pad, dtype=torch.float64, device="cuda")
    m = torch.empty(d_pad, dtype=torch.float64, device="cuda")
    hap.hap_export_pooled(ctx.h, zh, zl, t, m)
    torch.cuda.synchronize()
    return [a.cpu().numpy() for a in (zh, zl, t, m)]


def test_stream_align_path(hap, ctx, orc):
    """Large pairs take the streaming alignment K1s (3 kernels, counted in the profile);
    two runs give bitwise identical planes, t and observed statistic; the batch entry
    point (a streaming pair in a wave of its own) reproduces the single-pair bits; full
    count parity with the oracle on a b-range."""
    import torch
    n_x, n_y, d = 2200, 1900, 2048  # n_pad d = 4160 * 2048 >= 8 Mi
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=77))
    hap.hap_profile_read(ctx.h, reset=True)
    g1, ref = check_pair(ctx, orc, X, Y, 3000, s=5, b_begin=1000, b_end=1600)
    launches = hap.hap_profile_read(ctx.h, reset=True)[1]
    assert launches["align"] == 3, launches
    n_pad, d_pad = -(-(n_x + n_y) // 64) * 64, -(-d // 32) * 32
    a = _export_planes(hap, ctx, n_pad, d_pad)
    ctx.permtest_pair(_cuda(X), _cuda(Y), 10, SEED)
    b = _export_planes(hap, ctx, n_pad, d_pad)
    for u, v in zip(a, b):
        assert np.array_equal(u, v)
    info2 = hap.decode_info(ctx.info)
    assert info2.t_obs == g1["t_obs"] and info2.r_x == g1["r_x"]
    # batch: one streaming pair next to two small (fused-path) pairs
    X2, Y2 = HI.make_pair(HI.PairSpec(100, 90, d, 40.0, 40.0, 30.0, seed=78))
    Xp = np.concatenate([X2, X, X2])
    Yp = np.concatenate([Y2, Y, Y2])
    cnx = np.array([0, 100, 100 + n_x, 200 + n_x])
    cny = np.array([0, 90, 90 + n_y, 180 + n_y])
    out = ctx.permtest_batch(_cuda(Xp), cnx, _cuda(Yp), cny, 3000, SEED, stream_id=4)
    assert out[1]["t_obs"] == g1["t_obs"] and out[1]["r_x"] == g1["r_x"]
    single = ctx.permtest_pair(_cuda(X), _cuda(Y), 3000, SEED, stream_id=5)
    assert out[1]["exceed_ge"] == single["exceed_ge"] and out[1]["gemm_t_obs"] == single["gemm_t_obs"]
    del torch


def test_stream_align_zero_vector(hap, ctx):
    """ZeroVector is reported by the streaming path with the first bad pooled row."""
    d = 4096
    X, Y = HI.make_pair(HI.PairSpec(1100, 1000, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=79))
    Y[517] = 0
    Y[900] = 0
    with pytest.raises(hap.HapError) as e:
        ctx.permtest_pair(_cuda(X), _cuda(Y), 100, SEED)
    assert e.value.status == 3
    assert hap.decode_info(ctx.info).bad_row == 1100 + 517


def test_errors_are_reported(hap, ctx):
    import torch
    X = np.ones((4, 8), np.float32)
    Y = np.ones((4, 8), np.float32)
    X[2] = 0
    with pytest.raises(hap.HapError) as e:
        ctx.permtest_pair(_cuda(X), _cuda(Y), 100, SEED)
    assert e.value.status == 3
    assert hap.decode_info(ctx.info).bad_row == 2
    X = np.array([[1, 0], [-1, 0]], np.float32)
    with pytest.raises(hap.HapError) as e:
        ctx.permtest_pair(_cuda(X), _cuda(np.array([[0, 1.0]], np.float32)), 100, SEED)
    assert e.value.status == 4
    # identity: coincident mean directions
    X, Y = HI.make_pair(HI.PairSpec(50, 50, 32, 20.0, 20.0, 0.0, seed=1))
    g = ctx.permtest_pair(_cuda(X), _cuda(X), 100, SEED)
    assert g["is_identity"]
    with pytest.raises(hap.HapError):
        ctx.permtest_pair(_cuda(X), _cuda(Y[:, :16].copy()), 100, SEED)


def test_sharding_is_additive_and_deterministic(ctx):
    """Counts over [0,B) equal the sum over shards; two runs are bitwise identical."""
    X, Y = HI.config_pair("C2")
    full = ctx.permtest_pair(_cuda(X), _cuda(Y), 10000, SEED, want_stats=True)
    again = ctx.permtest_pair(_cuda(X), _cuda(Y), 10000, SEED, want_stats=True)
    assert np.array_equal(full["stats"].cpu().numpy(), again["stats"].cpu().numpy())
    tot = np.zeros(3, np.int64)
    for b0, b1 in [(0, 1234), (1234, 5000), (5000, 10000)]:
        r = ctx.permtest_pair(_cuda(X), _cuda(Y), 10000, SEED, b_begin=b0, b_end=b1)
        tot += [r["exceed_ge"], r["exceed_abs"], r["flagged"]]
    assert tot.tolist() == [full["exceed_ge"], full["exceed_abs"], full["flagged"]]


def test_host_inputs_match_device_inputs(ctx):
    """hap_align accepts host buffers (copied in on the stream): same result."""
    import torch
    X, Y = HI.config_pair("C1")
    a = ctx.permtest_pair(_cuda(X), _cuda(Y), 1000, SEED, want_stats=True)
    b = ctx.permtest_pair(torch.from_numpy(X).pin_memory(), torch.from_numpy(Y), 1000, SEED,
                          want_stats=True)
    assert np.array_equal(a["stats"].cpu().numpy(), b["stats"].cpu().numpy())
    assert a["exceed_ge"] == b["exceed_ge"]


# ------------------------------------------------------------------ varlen batch
def _batch_vs_oracle(orc, res, Xp, cnx, Yp, cny, B, s0, sel):
    for p in sel:
        X = Xp[cnx[p]:cnx[p + 1]]
        Y = Yp[cny[p]:cny[p + 1]]
        ref = orc.run_pair(X, Y, B, SEED, s=s0 + p)
        g = res[p]
        assert g["status"] == 0
        Ls = abs(ref["L_x"]) + abs(ref["L_y"])
        assert abs(g["t_obs"] - ref["t_obs"]) <= 1e-10 * Ls
        assert math.isclose(g["r_x"], ref["r_x"], rel_tol=1e-10)
        assert abs(g["gemm_t_obs"] - ref["t_obs"]) <= 1e-5 * Ls
        for k in ("exceed_ge", "exceed_abs"):
            assert abs(g[k] - ref[k]) <= ref["flagged"], (p, k, g[k], ref[k])


def test_batch_varlen_matches_oracle(ctx, orc):
    """hap_permtest_batch over a ragged batch (C4 recipe, small B): every pair agrees
    with the oracle run on generator stream stream_id + p, and is bitwise identical to
    the same pair run alone through hap_permtest."""
    sizes = [50, 300, 7, 129, 1000, 64, 2]
    ny = [60, 250, 9, 128, 1000, 64, 3]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=96, ny_sizes=ny)
    B, s0 = 700, 11
    res = ctx.permtest_batch(_cuda(Xp), cnx, _cuda(Yp), cny, B, SEED, stream_id=s0)
    _batch_vs_oracle(orc, res, Xp, cnx, Yp, cny, B, s0, range(len(sizes)))
    for p in (1, 4):
        one = ctx.permtest_pair(_cuda(Xp[cnx[p]:cnx[p + 1]]), _cuda(Yp[cny[p]:cny[p + 1]]), B,
                                SEED, stream_id=s0 + p)
        for k in ("t_obs", "gemm_t_obs", "exceed_ge", "exceed_abs", "flagged"):
            assert one[k] == res[p][k], (p, k)


def test_batch_config4_slice(ctx, orc):
    """A slice of C4 at full size (d=768, B=10^4, log-uniform n): counts vs oracle."""
    sizes = HI.c4_sizes(10000)[:4]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=768)
    res = ctx.permtest_batch(_cuda(Xp), cnx, _cuda(Yp), cny, 10000, SEED, stream_id=0)
    _batch_vs_oracle(orc, res, Xp, cnx, Yp, cny, 10000, 0, range(len(sizes)))


def test_batch_pair_sel_and_data_errors(hap, ctx, orc):
    """pair_sel runs only the selected pairs (others untouched); a pair with a zero row
    reports its own status and the batch continues; shape errors are synchronous."""
    import torch
    sizes = [40, 33, 80, 20, 55]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=64)
    Xp[cnx[2] + 5] = 0.0                       # pair 2: ZeroVector
    sel = [4, 2, 0]
    res = ctx.permtest_batch(_cuda(Xp), cnx, _cuda(Yp), cny, 300, SEED, stream_id=3,
                             pair_sel=sel)
    assert res[1] is None and res[3] is None
    assert res[2]["status"] == 3 and res[2]["exceed_ge"] == 0 and res[2]["p_value"] is None
    _batch_vs_oracle(orc, res, Xp, cnx, Yp, cny, 300, 3, [4, 0])
    infos, counts = ctx.permtest_batch(_cuda(Xp), cnx, _cuda(Yp), cny, 300, SEED,
                                       pair_sel=sel, sync=False)
    hap.hap_sync(ctx.h)
    assert counts[1].abs().sum().item() == 0 and counts[3].abs().sum().item() == 0
    assert int(infos[1].to(torch.int64).sum()) == 0
    bad = cnx.copy()
    bad[3] = bad[2]                            # pair 2 gets n_x = 0
    with pytest.raises(hap.HapError):
        ctx.permtest_batch(_cuda(Xp), bad, _cuda(Yp), cny, 300, SEED)


def test_gpu_batch_sharded_world_invariant(ctx):
    """gpu_batch_sharded: the per-rank shares of a 3-way split (combined here by hand,
    as the all_reduce would) equal the world-1 result bit for bit."""
    import torch
    from paper_2605_08048_b200 import parallel
    sizes = [30, 200, 75, 12, 90, 140]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=128)
    X, Y = _cuda(Xp), _cuda(Yp)
    i1, c1 = parallel.gpu_batch_sharded(ctx, X, cnx, Y, cny, 500, SEED, 0, 1, stream_id=5)
    acc_i = torch.zeros((len(sizes), i1.shape[1] // 8), dtype=torch.int64, device=X.device)
    acc_c = torch.zeros_like(c1)
    for r in range(3):
        ir, cr = parallel.gpu_batch_sharded(ctx, X, cnx, Y, cny, 500, SEED, r, 3, stream_id=5,
                                            reduce=False)
        acc_i += ir.view(torch.int64)
        acc_c += cr
    torch.cuda.synchronize()
    assert torch.equal(acc_c, c1)
    assert torch.equal(acc_i.view(torch.uint8), i1)


@pytest.mark.parametrize("wave", [2, 3, 4])
def test_batch_waves_are_bitwise_invariant(ctx, wave):
    """Several tests per generator/GEMM launch (cfg.wave) give bitwise the same statistics
    and counts as one test per launch (ragged sizes, several waves and a short last one)."""
    sizes = [50, 300, 7, 129, 1000, 64, 2, 333, 90]
    ny = [60, 250, 9, 128, 1000, 64, 3, 300, 91]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=96, ny_sizes=ny)
    X, Y = _cuda(Xp), _cuda(Yp)
    ref = ctx.permtest_batch(X, cnx, Y, cny, 900, SEED, stream_id=4, wave=1)
    got = ctx.permtest_batch(X, cnx, Y, cny, 900, SEED, stream_id=4, wave=wave)
    for p in range(len(sizes)):
        for k in ("t_obs", "gemm_t_obs", "exceed_ge", "exceed_abs", "flagged"):
            assert got[p][k] == ref[p][k], (wave, p, k)


def test_batch_shared_mask(ctx, orc):
    """HAP_FLAG_SHARED_MASK: every pair uses generator stream cfg.stream_id; equal-size pairs
    share one generated block per wave; results equal the oracle (and the single-pair path)
    run with that stream."""
    sizes = [120, 120, 120, 120, 120, 64, 64, 120]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=128)
    X, Y = _cuda(Xp), _cuda(Yp)
    B, s0 = 1500, 21
    res = ctx.permtest_batch(X, cnx, Y, cny, B, SEED, stream_id=s0, shared=True)
    for p in range(len(sizes)):
        Xq, Yq = Xp[cnx[p]:cnx[p + 1]], Yp[cny[p]:cny[p + 1]]
        ref = orc.run_pair(Xq, Yq, B, SEED, s=s0)
        Ls = abs(ref["L_x"]) + abs(ref["L_y"])
        assert abs(res[p]["t_obs"] - ref["t_obs"]) <= 1e-10 * Ls
        for k in ("exceed_ge", "exceed_abs"):
            assert abs(res[p][k] - ref[k]) <= ref["flagged"], (p, k)
        one = ctx.permtest_pair(_cuda(Xq), _cuda(Yq), B, SEED, stream_id=s0)
        for k in ("gemm_t_obs", "exceed_ge", "exceed_abs", "flagged"):
            assert one[k] == res[p][k], (p, k)


def test_batch_multiblock_and_errors_in_waves(hap, ctx, orc):
    """A batch whose B needs several generator/GEMM blocks per test (cfg.block) and a data
    error inside a wave: every good pair matches the oracle, the bad one only reports."""
    import torch
    sizes = [40, 33, 80, 20, 55, 61]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=64)
    Xp[cnx[4] + 3] = 0.0                     # pair 4 (second of the second wave): ZeroVector
    B, s0 = 700, 8
    X, Y = _cuda(Xp), _cuda(Yp)
    infos = torch.zeros((len(sizes), hap.INFO_BYTES), dtype=torch.uint8, device=X.device)
    counts = torch.zeros((len(sizes), 3), dtype=torch.int64, device=X.device)
    cfg = hap.make_cfg(SEED, B, 0, B, s0, block=200, wave=3)
    hap.hap_permtest_batch(ctx.h, X, cnx, Y, cny, 0, cfg, infos, counts)
    hap.hap_sync(ctx.h)
    cts = counts.cpu().tolist()
    raw = infos.cpu().numpy()
    for p in range(len(sizes)):
        info = hap.hap_align_info.from_buffer_copy(bytes(raw[p].tobytes()))
        if p == 4:
            assert info.status == 3 and cts[p] == [0, 0, 0]
            continue
        assert info.status == 0
        ref = orc.run_pair(Xp[cnx[p]:cnx[p + 1]], Yp[cny[p]:cny[p + 1]], B, SEED, s=s0 + p)
        for k, c in zip(("exceed_ge", "exceed_abs"), cts[p][:2]):
            assert abs(c - ref[k]) <= ref["flagged"], (p, k)


# ------------------------------------------------------------------ exhaustive (exact p)
def _colex_unrank(r, N, k):
    """Independent colex unranking (combinatorial number system), plain Python."""
    out = []
    c = N - 1
    for i in range(k, 0, -1):
        while math.comb(c, i) > r:
            c -= 1
        r -= math.comb(c, i)
        out.append(c)
        c -= 1
    return sorted(out)


@pytest.mark.parametrize("N,n_x", [(6, 3), (10, 4), (12, 9), (16, 1), (20, 10)])
def test_comb_sets_enumerate_all_splits(hap, ctx, N, n_x):
    """HAP_FLAG_EXHAUSTIVE generator: rank b -> b-th combination in colex order (the
    complement of the n_y-subset when n_x > n_y): every split exactly once."""
    import itertools
    import torch
    total = math.comb(N, n_x)
    assert hap.hap_n_choose_k(N, n_x) == total
    out = torch.zeros((total, N), dtype=torch.uint8, device="cuda")
    hap.hap_comb_sets(ctx.h, 0, total, N, n_x, out)
    got = out.cpu().numpy()
    assert np.all(got.sum(1) == n_x)
    seen = {tuple(np.flatnonzero(r)) for r in got}
    assert seen == set(itertools.combinations(range(N), n_x))
    k = min(n_x, N - n_x)
    for b in range(0, total, max(1, total // 50)):
        sub = _colex_unrank(b, N, k)
        want = sub if k == n_x else sorted(set(range(N)) - set(sub))
        assert list(np.flatnonzero(got[b])) == want, b


def test_comb_sets_large_sampled(hap, ctx):
    """C(34, 17) = 2.3e9 splits: sampled ranks near both ends and the middle."""
    import torch
    N, n_x = 34, 17
    total = math.comb(N, n_x)
    for b0 in (0, total // 2 - 3, total - 7):
        out = torch.zeros((7, N), dtype=torch.uint8, device="cuda")
        hap.hap_comb_sets(ctx.h, b0, 7, N, n_x, out)
        for r, row in enumerate(out.cpu().numpy()):
            assert list(np.flatnonzero(row)) == _colex_unrank(b0 + r, N, n_x)
    with pytest.raises(hap.HapError):
        hap.hap_comb_sets(ctx.h, total - 3, 7, N, n_x, torch.zeros((7, N), dtype=torch.uint8,
                                                                   device="cuda"))


def test_exhaustive_worked_example_exact(ctx):
    """SURVEY worked example: the exact permutation distribution gives 12 of 70 splits with
    T >= T_obs (tests/golden/worked_example.txt, computed independently) - the GPU path
    must reproduce the integer exactly; two-sided 24 within the flagged true ties."""
    from conftest import read_golden
    rows = read_golden("worked_example.txt")
    X = np.array([[float(v) for v in r.split()[1:]] for r in rows if r.startswith("X ")], np.float32)
    Y = np.array([[float(v) for v in r.split()[1:]] for r in rows if r.startswith("Y ")], np.float32)
    vals = {r.split()[0]: r.split()[1:] for r in rows}
    total = int(vals["exhaustive_total"][0])
    g = ctx.permtest_pair(_cuda(X), _cuda(Y), total, SEED, exhaustive=True)
    assert g["exceed_ge"] == int(vals["exhaustive_ge"][0])
    assert abs(g["exceed_abs"] - int(vals["exhaustive_abs"][0])) <= g["flagged"]
    assert g["p_exact"] == 12 / 70


def test_exhaustive_flagged_exact_ties(ctx, orc):
    """The flagged counter on the tie-structured pool of tests/tiecase.py: over all C(10, 5)
    splits exactly prod C(m_k, c_k) + prod C(m_k, m_k - c_k) = 72 are near-ties (pinned by
    combinatorics in test_oracle.py::test_flagged_counter_exact_ties); the GPU flags the same
    72 and its counts agree with the oracle's up to them."""
    import tiecase
    X, Y, order = tiecase.pool()
    want = tiecase.expected_flagged(order)[0]
    total = math.comb(10, 5)
    g = ctx.permtest_pair(_cuda(X), _cuda(Y), total, SEED, mode=1, exhaustive=True)
    assert g["flagged"] == want
    ref = orc.run_pair(X, Y, 10, SEED, mode=1)
    counts, _ = orc.exhaustive(ref["Z"], 5, ref["t_obs"], ref["tau"])
    assert int(counts[2]) == want
    for k, c in (("exceed_ge", counts[0]), ("exceed_abs", counts[1])):
        assert abs(g[k] - int(c)) <= want


@pytest.mark.parametrize("n_x,n_y,d", [(5, 6, 32), (9, 9, 100), (3, 12, 768)])
def test_exhaustive_matches_oracle(ctx, orc, n_x, n_y, d):
    """Exhaustive GPU counts vs the oracle's brute-force enumeration (orc_exhaustive)."""
    X, Y = HI.make_pair(HI.PairSpec(n_x, n_y, d, HI.kappa_for(d), HI.kappa_for(d), 30.0, seed=5))
    total = math.comb(n_x + n_y, n_x)
    ref = orc.run_pair(X, Y, 10, SEED)
    counts, tot = orc.exhaustive(ref["Z"], n_x, ref["t_obs"], ref["tau"])
    assert tot == total
    g = ctx.permtest_pair(_cuda(X), _cuda(Y), total, SEED, exhaustive=True)
    fl = int(counts[2])
    assert abs(g["exceed_ge"] - int(counts[0])) <= fl
    assert abs(g["exceed_abs"] - int(counts[1])) <= fl
    assert g["exceed_ge"] >= 1  # the observed split itself is enumerated


def test_exhaustive_rejects_too_many_splits(hap, ctx):
    X, Y = HI.make_pair(HI.PairSpec(20, 20, 16, 20.0, 20.0, 30.0, seed=5))
    with pytest.raises(hap.HapError):
        ctx.permtest_pair(_cuda(X), _cuda(Y), 1000, SEED, exhaustive=True)


def test_gpu_type1_calibration_batch(ctx):
    """C5 recipe at test size: equal-kappa clouds with
    different mean directions.  Through hap_permtest_batch the aligned test rejects at the
    nominal rate (within 3 SE); the naive test (no reflection) is reported alongside."""
    R, B, alpha = 400, 999, 0.10
    pairs = [HI.make_pair(HI.PairSpec(60, 60, 32, 50.0, 50.0, 60.0, seed=78), rep) for rep in range(R)]
    Xp = np.concatenate([p[0] for p in pairs])
    Yp = np.concatenate([p[1] for p in pairs])
    cu = np.arange(R + 1, dtype=np.int64) * 60
    rates = {}
    for mode in (0, 1):
        res = ctx.permtest_batch(_cuda(Xp), cu, _cuda(Yp), cu, B, SEED, stream_id=0, mode=mode)
        rates[mode] = np.mean([r["p_value"] <= alpha for r in res])
    se = math.sqrt(alpha * (1 - alpha) / R)
    assert abs(rates[0] - alpha) <= 3 * se, rates


@pytest.mark.parametrize("shared", [False, True])
def test_config5_batch_full_size(ctx, orc, shared):
    """C5 at full size (n = 500/500, d = 768, B = 10^4) through hap_permtest_batch in the
    bench's launch configuration (waves of 3 / 4, two lanes): 4 replicates vs the oracle."""
    pairs = [HI.config_pair("C5", rep) for rep in range(4)]
    Xp = np.concatenate([p[0] for p in pairs])
    Yp = np.concatenate([p[1] for p in pairs])
    cu = np.arange(5, dtype=np.int64) * 500
    B, s0 = 10000, 40
    res = ctx.permtest_batch(_cuda(Xp), cu, _cuda(Yp), cu, B, SEED, stream_id=s0, shared=shared)
    for p in range(4):
        ref = orc.run_pair(pairs[p][0], pairs[p][1], B, SEED, s=s0 if shared else s0 + p)
        Ls = abs(ref["L_x"]) + abs(ref["L_y"])
        assert abs(res[p]["t_obs"] - ref["t_obs"]) <= 1e-10 * Ls
        assert abs(res[p]["gemm_t_obs"] - ref["t_obs"]) <= 1e-5 * Ls
        for k in ("exceed_ge", "exceed_abs"):
            assert abs(res[p][k] - ref[k]) <= ref["flagged"], (p, k)


_VARIANT_SCRIPT = r"""
import sys, json
sys.path.insert(0, sys.argv[1])
import numpy as np, torch
import hap_inputs as HI
import paper_2605_08048_b200 as hap
ctx = hap.Context(0)
sizes = [50, 300, 129, 1000, 64, 333]
Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=96)
res = ctx.permtest_batch(torch.from_numpy(Xp).cuda(), cnx, torch.from_numpy(Yp).cuda(), cny,
                         1200, HI.PERM_SEED, stream_id=9)
print(json.dumps([[r["exceed_ge"], r["exceed_abs"], r["flagged"], r["gemm_t_obs"]] for r in res]))
"""


@pytest.mark.parametrize("env", [{"HAP_K1_DRAWS": "1"}, {"HAP_BATCH_SPLIT": "1"},
                                 {"HAP_WAVE": "1"}, {"HAP_K3_DYNAMIC": "0"},
                                 {"HAP_K3_DYNAMIC": "0", "HAP_K3_ROUND_ROBIN": "1"},
                                 {"HAP_K2_NARROW": "1", "HAP_K2_PW": "1"},
                                 {"HAP_K2_NARROW": "1", "HAP_K2_PW": "2"},
                                 {"HAP_K2_NARROW": "1", "HAP_K2_PW": "4"},
                                 {"HAP_K2_WIDE_PW": "1"}, {"HAP_K2_WIDE_PW": "2"},
                                 {"HAP_K2_WIDE_PW": "4"}, {"HAP_K3_TILE_GROUP": "0"},
                                 {"HAP_K3_TILE_GROUP": "3"}])
def test_experimental_paths_bitwise_equal(env):
    """The alternative scheduling paths (draws staged by K1, split generator on the side
    stream, one test per wave, the static K3 split, round-robin K3 schedule, the u16-table
    generator with 1, 2 or 4 warps per permutation) give bitwise the default results."""
    import json
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))

    def run(extra):
        e = dict(os.environ)
        for k in ("HAP_K1_DRAWS", "HAP_BATCH_SPLIT", "HAP_WAVE", "HAP_K3_ROUND_ROBIN", "HAP_K3_DYNAMIC",
                  "HAP_K2_NARROW", "HAP_K2_PW", "HAP_K2_WIDE_PW", "HAP_K3_TILE_GROUP"):
            e.pop(k, None)
        e.update(extra)
        out = subprocess.run([sys.executable, "-c", _VARIANT_SCRIPT, root], env=e,
                             capture_output=True, text=True, timeout=600)
        assert out.returncode == 0, out.stderr[-2000:]
        return json.loads(out.stdout.strip().splitlines()[-1])

    assert run(env) == run({})


def test_gpu_power_broader_x(ctx):
    """NEXT-3: when X is genuinely broader (kappa_X < kappa_Y) the
    aligned one-sided test keeps its power (rejects in most replicates), like the naive one."""
    R, B = 60, 999
    pairs = [HI.make_pair(HI.PairSpec(100, 100, 32, 25.0, 60.0, 45.0, seed=79), rep) for rep in range(R)]
    Xp = np.concatenate([p[0] for p in pairs])
    Yp = np.concatenate([p[1] for p in pairs])
    cu = np.arange(R + 1, dtype=np.int64) * 100
    power = {}
    for mode in (0, 1):
        res = ctx.permtest_batch(_cuda(Xp), cu, _cuda(Yp), cu, B, SEED, mode=mode)
        power[mode] = np.mean([r["p_value"] <= 0.05 for r in res])
    assert power[0] >= 0.9, power


def test_config2_batch_full_size_bench_launch(ctx, orc):
    """C2 at full size in exactly the bench's launch configuration: one wave of 3 tests
    through hap_permtest_batch (generator streams as bench.py assigns them), every test's
    observed statistic, same-path T_obs and counts vs the oracle."""
    pairs = [HI.make_pair(HI.PairSpec(1000, 1000, 768, HI.kappa_for(768), HI.kappa_for(768), 30.0,
                                      seed=1002), rep=i) for i in range(3)]
    Xp = np.concatenate([p[0] for p in pairs])
    Yp = np.concatenate([p[1] for p in pairs])
    cu = np.arange(4, dtype=np.int64) * 1000
    B, s0 = 10000, 1_000_003
    res = ctx.permtest_batch(_cuda(Xp), cu, _cuda(Yp), cu, B, SEED, stream_id=s0, wave=3)
    for p in range(3):
        ref = orc.run_pair(pairs[p][0], pairs[p][1], B, SEED, s=s0 + p)
        Ls = abs(ref["L_x"]) + abs(ref["L_y"])
        assert abs(res[p]["t_obs"] - ref["t_obs"]) <= 1e-10 * Ls
        assert abs(res[p]["gemm_t_obs"] - ref["t_obs"]) <= 1e-5 * Ls
        for k in ("exceed_ge", "exceed_abs"):
            assert abs(res[p][k] - ref[k]) <= ref["flagged"], (p, k)


def _fuzz_cases(n=18, seed=20261018):
    rng = np.random.default_rng(seed)
    out = []
    for i in range(n):
        nx = int(rng.integers(2, 300))
        ny = int(rng.integers(2, 300))
        d = int(rng.choice([2, 3, 17, 31, 64, 100, 257, 768, 1024, 1540]))
        B = int(rng.integers(1, 1500))
        out.append((i, nx, ny, d, B, int(rng.integers(0, 2)), int(rng.choice([1, 2])),
                    int(rng.choice([0, 97])), [None, True, False][int(rng.integers(0, 3))]))
    return out


@pytest.mark.parametrize("case", _fuzz_cases(), ids=lambda c: f"fuzz{c[0]}")
def test_fuzz_shapes_vs_oracle(ctx, orc, case):
    """Seeded random shapes (tiny d, ragged n, odd B, both alignment modes, both K3 modes,
    forced multi-block, the Gram / plane / automatic K3 form): full parity bars against the
    oracle."""
    i, nx, ny, d, B, mode, pair_mode, block, gram = case
    X, Y = HI.make_pair(HI.PairSpec(nx, ny, d, 8.0 + d, 8.0 + d, 40.0, seed=900 + i))
    check_pair(ctx, orc, X, Y, B, s=i, mode=mode, block=block, pair_mode=pair_mode, gram=gram)


def _campaign_cases(seed=20261019):
    """Wider seeded shapes than _fuzz_cases: log-uniform group sizes 1..1500 (singletons
    included), d up to 4096 (the streaming ring K1 path once n_pad d >= 8 Mi), B scaled so the
    oracle stays within seconds.  FUZZ_CASES (default 6) sets the count: the suite runs 6; a
    campaign run (profiles/r02_fuzz_campaign.log) runs 120."""
    rng = np.random.default_rng(seed)
    out = []
    for i in range(int(os.environ.get("FUZZ_CASES", "6"))):
        nx = int(np.exp(rng.uniform(0.0, np.log(1500))))
        ny = int(np.exp(rng.uniform(0.0, np.log(1500))))
        if rng.uniform() < 0.15:  # ring-path sizes (n_pad d >= 8 Mi at d = 4096)
            nx, ny = int(rng.integers(1000, 1400)), int(rng.integers(1000, 1400))
            d = 4096
        else:
            d = int(rng.choice([2, 3, 17, 31, 64, 100, 257, 768, 1024, 1540, 2048, 4096]))
        B = int(max(1, min(int(rng.integers(1, 2500)), 3e9 // max(1, (nx + ny) * d))))
        out.append((i, nx, ny, d, B, int(rng.integers(0, 2)), int(rng.choice([1, 2])),
                    int(rng.choice([0, 97])), [None, True, False][int(rng.integers(0, 3))]))
    return out


@pytest.mark.parametrize("case", _campaign_cases(),
                         ids=lambda c: f"c{c[0]}_n{c[1]}x{c[2]}_d{c[3]}_B{c[4]}")
def test_fuzz_campaign_vs_oracle(hap, ctx, orc, case):
    """Seeded wide random shapes against the oracle.  Every case must meet the certified bar
    (R14: the kernel's own error bound covers its error on every permutation, every decision
    outside the widened band is the oracle's, counts within the GPU's flagged); the plain 1e-5
    bars of check_pair are reported per case (they fail where a tiny group's sums come from
    the complement t - sigma of a large one, or where d <= 3 makes L(r) ill-conditioned:
    DESIGN.md §4)."""
    i, nx, ny, d, B, mode, pair_mode, block, gram = case
    X, Y = HI.make_pair(HI.PairSpec(nx, ny, d, 8.0 + d, 8.0 + d, 40.0, seed=5000 + i))
    check_certified(hap, ctx, orc, X, Y, B, s=100 + i, mode=mode, block=block, pair_mode=pair_mode,
                    gram=gram)
    try:
        check_pair(ctx, orc, X, Y, B, s=100 + i, mode=mode, block=block, pair_mode=pair_mode, gram=gram)
        print(f"PLAIN-BARS ok   case {i} n {nx}x{ny} d {d}")
    except AssertionError:
        print(f"PLAIN-BARS miss case {i} n {nx}x{ny} d {d} (certified bar met)")


@pytest.mark.parametrize("seed", [1, 2, 3, 4, 5, 6])
def test_fuzz_batches_vs_oracle(ctx, orc, seed):
    """Seeded random varlen batches: random pair counts and sizes, wave size, alignment
    mode and shared / independent masks, every pair against the oracle."""
    rng = np.random.default_rng(seed)
    P = int(rng.integers(3, 10))
    d = int(rng.choice([16, 48, 130]))
    shared = bool(rng.integers(0, 2))
    if shared:  # runs of equal sizes (shared waves need equal n_x, n_y)
        base = [int(rng.integers(4, 150)) for _ in range(3)]
        sx = [base[int(rng.integers(0, 3))] for _ in range(P)]
        sy = list(sx)
    else:
        sx = [int(rng.integers(2, 200)) for _ in range(P)]
        sy = [int(rng.integers(2, 200)) for _ in range(P)]
    Xp, cnx, Yp, cny = HI.varlen_batch(sx, d=d, ny_sizes=sy, seed=3000 + seed)
    B, s0 = int(rng.integers(50, 900)), int(rng.integers(0, 1000))
    wave, mode = int(rng.integers(1, 5)), int(rng.integers(0, 2))
    gram = bool(rng.integers(0, 2))
    res = ctx.permtest_batch(_cuda(Xp), cnx, _cuda(Yp), cny, B, SEED, stream_id=s0, mode=mode,
                             wave=wave, shared=shared, gram=gram)
    for p in range(P):
        ref = orc.run_pair(Xp[cnx[p]:cnx[p + 1]], Yp[cny[p]:cny[p + 1]], B, SEED,
                           s=s0 if shared else s0 + p, mode=mode)
        Ls = abs(ref["L_x"]) + abs(ref["L_y"])
        assert abs(res[p]["t_obs"] - ref["t_obs"]) <= 1e-10 * Ls, p
        for k in ("exceed_ge", "exceed_abs"):
            assert abs(res[p][k] - ref[k]) <= ref["flagged"], (p, k, res[p][k], ref[k])


def test_batch_argument_errors(hap, ctx):
    """Synchronous argument errors of hap_permtest_batch (nothing enqueued)."""
    import torch
    sizes = [10, 12]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=16)
    X, Y = _cuda(Xp), _cuda(Yp)
    infos = torch.zeros((2, hap.INFO_BYTES), dtype=torch.uint8, device="cuda")
    counts = torch.zeros((2, 3), dtype=torch.int64, device="cuda")
    ok = hap.make_cfg(SEED, 100)
    with pytest.raises(hap.HapError):  # exhaustive mode is per pair only
        hap.hap_permtest_batch(ctx.h, X, cnx, Y, cny, 0, hap.make_cfg(SEED, 100, flags=hap.HAP_FLAG_EXHAUSTIVE),
                               infos, counts)
    with pytest.raises(hap.HapError):  # bad alignment mode
        hap.hap_permtest_batch(ctx.h, X, cnx, Y, cny, 7, ok, infos, counts)
    with pytest.raises(hap.HapError):  # pair_sel out of range
        hap.hap_permtest_batch(ctx.h, X, cnx, Y, cny, 0, ok, infos, counts, pair_sel=[0, 5])
    with pytest.raises(hap.HapError):  # a pair listed twice would add its counts twice
        hap.hap_permtest_batch(ctx.h, X, cnx, Y, cny, 0, ok, infos, counts, pair_sel=[1, 0, 1])
    with pytest.raises(hap.HapError):  # one input in host memory, the other on the device
        hap.hap_permtest_batch(ctx.h, torch.from_numpy(Xp), cnx, Y, cny, 0, ok, infos, counts)
    with pytest.raises(hap.HapError):  # b_end beyond 2^32
        hap.hap_permtest_batch(ctx.h, X, cnx, Y, cny, 0, hap.make_cfg(SEED, 1 << 33), infos, counts)
    hap.hap_permtest_batch(ctx.h, X, cnx, Y, cny, 0, ok, infos, counts)  # still usable
    hap.hap_sync(ctx.h)
    assert int(counts.sum()) > 0


@pytest.mark.parametrize("pinned", [True, False])
def test_batch_host_inputs_bitwise(ctx, pinned):
    """hap_permtest_batch with X_packed / Y_packed in host memory (pinned or pageable): the
    library copies each wave's rows itself; results are bitwise those of device inputs."""
    import torch
    sizes = [50, 300, 7, 129, 1000, 64, 2, 333]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=96)
    Xh, Yh = torch.from_numpy(Xp), torch.from_numpy(Yp)
    if pinned:
        Xh, Yh = Xh.pin_memory(), Yh.pin_memory()
    dev = ctx.permtest_batch(_cuda(Xp), cnx, _cuda(Yp), cny, 900, SEED, stream_id=5)
    host = ctx.permtest_batch(Xh, cnx, Yh, cny, 900, SEED, stream_id=5)
    assert host == dev


def test_batch_order_independent(ctx):
    """The batch processes pairs largest-first in waves; the results of every pair are the
    same bits whatever order pair_sel lists them in (own generator stream and workspace)."""
    sizes = [50, 300, 7, 129, 1000, 64, 2, 333, 129, 50]
    Xp, cnx, Yp, cny = HI.varlen_batch(sizes, d=96)
    X, Y = _cuda(Xp), _cuda(Yp)
    a = ctx.permtest_batch(X, cnx, Y, cny, 800, SEED, stream_id=3)
    perm = list(np.random.default_rng(1).permutation(len(sizes)))
    b = ctx.permtest_batch(X, cnx, Y, cny, 800, SEED, stream_id=3, pair_sel=perm)
    assert a == b


def test_max_pooled_size(ctx, orc):
    """N = n_x + n_y = 65535 (the ABI maximum; u16 generator table, 65536-row mask tiles):
    every statistic and count against the oracle."""
    X, Y = HI.make_pair(HI.PairSpec(40000, 25535, 16, 20.0, 30.0, 40.0, seed=65535))
    check_pair(ctx, orc, X, Y, 300, s=7)


def test_split_half_words_parity(ctx, orc):
    """Same-word split-half workload (App. E :852-858, Table 6): words of
    130-160 tokens split in halves, baseline (naive) and proposed (aligned) through
    hap_permtest_batch on the same permutations; counts within the flagged permutations of
    the oracle's, and the two tests' p-values close (the paper's finding)."""
    import sys
    sys.path.insert(0, __import__("os").path.join(__import__("os").path.dirname(__file__), "..", "tools"))
    import split_half as SH
    Xp, cnx, Yp, cny, ns, rs = SH.make_words(6, seed=11)
    B = 2000
    outs = {}
    for mode in (0, 1):
        outs[mode] = ctx.permtest_batch(_cuda(Xp), cnx, _cuda(Yp), cny, B, SEED, stream_id=0, mode=mode)
        for p in range(6):
            ref = orc.run_pair(Xp[cnx[p]:cnx[p + 1]], Yp[cny[p]:cny[p + 1]], B, SEED, s=p, mode=mode)
            g = outs[mode][p]
            assert abs(g["exceed_ge"] - ref["exceed_ge"]) <= ref["flagged"], (mode, p)
            assert abs(g["exceed_abs"] - ref["exceed_abs"]) <= ref["flagged"], (mode, p)
    dp = [abs(outs[0][p]["p_value"] - outs[1][p]["p_value"]) for p in range(6)]
    assert max(dp) < 0.03, dp
