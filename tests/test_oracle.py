"""Pins of the fp64 oracle against things other than itself (-m "not gpu").

Each test names what fixes the expected value: a published known-answer vector, a
worked example computed by independent code, a closed form from the
paper (PAPER.md line), a textbook identity, or brute force.  A plausible mistake in
the oracle (dropped term, sign, index, transposed operand, wrong stream word) fails
at least one of them.
"""
import itertools
import math

import numpy as np
import pytest

from conftest import read_golden
import hap_inputs as HI

SEED = HI.PERM_SEED


# ---------------------------------------------------------------- Philox / PERM-SPEC
def test_philox_kat(orc):
    """Random123 KATs (tests/golden/philox_kat.txt)."""
    for row in read_golden("philox_kat.txt"):
        w = [int(x, 16) for x in row.split()]
        out = orc.philox4x32_10(w[0:4], w[4:6])
        assert out.tolist() == w[6:10]


def test_permspec_golden_sets(orc):
    """SURVEY.md §8c golden sets (independent implementation)."""
    for row in read_golden("permspec_v1.txt"):
        lhs, rhs = row.split(":")
        seed, s, b, N, n = lhs.split()
        want = [int(x) for x in rhs.split()]
        g = orc.perm_set(int(seed, 16), int(s), int(b), int(N), int(n))
        assert np.nonzero(g)[0].tolist() == want


def test_permspec_exact_size_and_uniform(orc):
    """|G_b| = n_x always; all C(6,3)=20 subsets equally likely (chi^2, 19 dof;
    critical value at p=1e-3 is 43.82)."""
    counts = {}
    B = 20000
    for b in range(B):
        g = orc.perm_set(SEED, 0, b, 6, 3)
        assert g.sum() == 3
        key = tuple(np.nonzero(g)[0])
        counts[key] = counts.get(key, 0) + 1
    assert len(counts) == 20
    exp = B / 20
    chi2 = sum((c - exp) ** 2 / exp for c in counts.values())
    assert chi2 < 43.82


def test_permspec_marginals_large(orc):
    """Each row lands in group 1 with probability n/N (binomial 5-sigma), N=2000."""
    N, n, B = 2000, 1000, 400
    tot = np.zeros(N)
    for b in range(B):
        g = orc.perm_set(SEED, 3, b, N, n)
        assert g.sum() == n
        tot += g
    p = n / N
    z = (tot - B * p) / math.sqrt(B * p * (1 - p))
    assert np.abs(z).max() < 5.0
    # first-half share (X rows) is not biased
    assert abs(tot[:n].sum() / (B * n) - p) < 0.01


def test_permspec_stream_ids_differ(orc):
    a = orc.perm_set(SEED, 0, 5, 100, 50)
    b = orc.perm_set(SEED, 1, 5, 100, 50)
    c = orc.perm_set(SEED + 1, 0, 5, 100, 50)
    assert not np.array_equal(a, b) and not np.array_equal(a, c)


def test_permspec_lemire_rejection_path(orc):
    """The side stream is exercised: over many (b, N) the redraw count is > 0 for
    huge N (rejection prob ~ k/2^32), and sets stay exact-size."""
    tot = 0
    for b in range(200):
        r = orc.perm_set_redraws(SEED, 0, b, 3_000_000, 1500)
        assert r >= 0
        tot += r
    assert tot > 0


def _rejection_rows():
    """tests/golden/permspec_v1_rejections.txt (independent generator, see its header)."""
    out = []
    for row in read_golden("permspec_v1_rejections.txt"):
        if " sha: " in row:
            lhs, rhs = row.split(" sha: ")
            kind = "sha"
        else:
            lhs, rhs = row.split(":")
            kind = "set"
        seed, s, b, N, n, rej = lhs.split()
        out.append((int(seed, 16), int(s), int(b), int(N), int(n), int(rej), kind, rhs.strip()))
    return out


def test_permspec_side_stream_golden(orc):
    """Sets decided by Lemire rejections (side stream (q', b, s, 1 + i), R6) and
    the rejection counts, from an independent sparse Fisher-Yates + Philox in pure Python
    (tests/golden/gen_permspec_rejections.py): a wrong side-stream counter word, word order
    or threshold changes at least one of these sets."""
    import hashlib
    rows = _rejection_rows()
    assert len(rows) >= 10 and all(r[5] >= 1 for r in rows)
    for seed, s, b, N, n, rej, kind, want in rows:
        g = orc.perm_set(seed, s, b, N, n)
        members = np.nonzero(g)[0].tolist()
        assert len(members) == n
        if kind == "sha":
            assert hashlib.sha256(" ".join(map(str, members)).encode()).hexdigest() == want
        else:
            assert members == [int(x) for x in want.split()], (s, b, N, n)
        assert orc.perm_set_redraws(seed, s, b, N, n) == rej, (s, b, N, n)


# ---------------------------------------------------------------- SPEC worked numbers
def test_normalize_and_2d_axis(orc):
    """SPEC.md:48-50 (3,4)->(0.6,0.8); SPEC.md:68 axis (0.70711,-0.70711) and
    reflecting (1,0) gives (0,1)."""
    a = orc.align(np.array([[3, 4]], np.float32), np.array([[1, 0]], np.float32), mode=1)
    assert np.allclose(a.Z[0], [0.6, 0.8], atol=1e-15)
    a = orc.align(np.array([[1, 0]], np.float32), np.array([[0, 1]], np.float32), mode=0)
    assert np.allclose(a.u, [math.sqrt(0.5), -math.sqrt(0.5)], atol=1e-15)
    assert np.allclose(a.Z[0], [0.0, 1.0], atol=1e-15)


def test_kappa_closed_forms(orc):
    """kappa(0.5, d=3) = 0.5*2.75/0.75 = 1.833333.., v = 0.545454..;
    kappa(0) = 0 (L = -inf); clamp at 1 - 1e-9; monotone."""
    assert math.isclose(math.exp(orc.logkappa(0.5, 3)), 0.5 * 2.75 / 0.75, rel_tol=1e-14)
    assert math.isclose(math.exp(-orc.logkappa(0.5, 3)), 6.0 / 11.0, rel_tol=1e-14)
    assert orc.logkappa(0.0, 3) == -math.inf
    assert orc.logkappa(1.0, 768) == orc.logkappa(1 - 1e-9, 768)
    assert orc.logkappa(0.3, 128) < orc.logkappa(0.6, 128)


def test_pvalue_examples(orc):
    """SPEC.md:249-251 / PAPER.md:189."""
    assert orc.pvalue(0, 99) == 0.01
    assert orc.pvalue(99, 99) == 1.0
    assert orc.pvalue(49, 99) == 0.5


def test_worked_example(orc):
    """SURVEY.md §8c worked example: r_X, r_Y, u, t, T_obs and the exhaustive
    12/70 (24/70 two-sided); nearest other T is 0.0155 away."""
    rows = read_golden("worked_example.txt")
    X = np.array([[float(v) for v in r.split()[1:]] for r in rows if r.startswith("X ")],
                 np.float32)
    Y = np.array([[float(v) for v in r.split()[1:]] for r in rows if r.startswith("Y ")],
                 np.float32)
    val = {r.split()[0]: [float(v) for v in r.split()[1:]] for r in rows
           if not r.startswith(("X ", "Y "))}
    a = orc.align(X, Y, 0)
    ob = orc.observed(a.Z, 4)
    assert math.isclose(ob["r1"], val["r_x"][0], abs_tol=1e-11)
    assert math.isclose(ob["r2"], val["r_y"][0], abs_tol=1e-11)
    assert np.allclose(a.u, val["u"], atol=1e-11)
    assert np.allclose(a.Z.sum(0), val["t"], atol=1e-10)
    assert math.isclose(ob["T"], val["t_obs"][0], abs_tol=1e-11)
    counts, total = orc.exhaustive(a.Z, 4, ob["T"])
    assert total == int(val["exhaustive_total"][0])
    assert int(counts[0]) == int(val["exhaustive_ge"][0])
    assert int(counts[1]) == int(val["exhaustive_abs"][0])


# ---------------------------------------------------------------- Householder (§3.1)
@pytest.mark.parametrize("d", [2, 16, 256, 768])
def test_householder_identities(orc, d):
    """H = I - 2uu^T is symmetric, orthogonal, involutive;
    H mu_x = mu_y; rows of X' are H x (isometry: norms and pairwise distances kept,
    PAPER.md:161); Y unchanged; r(X') = r(X)."""
    rng = np.random.default_rng(d)
    spec = HI.PairSpec(40, 30, d, HI.kappa_for(d) if d >= 32 else 5.0,
                       HI.kappa_for(d) if d >= 32 else 5.0, 70.0, seed=d)
    X, Y = HI.make_pair(spec)
    a = orc.align(X, Y, 0)
    n = orc.align(X, Y, 1)  # naive: normalised, unreflected
    assert a.status == 0 and not a.is_identity
    H = np.eye(d) - 2.0 * np.outer(a.u, a.u)
    assert np.allclose(H, H.T, atol=1e-15)
    assert np.allclose(H @ H.T, np.eye(d), atol=1e-13)
    Xn, Yn = n.Z[:40], n.Z[40:]
    mu_x = Xn.mean(0) / np.linalg.norm(Xn.mean(0))
    mu_y = Yn.mean(0) / np.linalg.norm(Yn.mean(0))
    assert np.allclose(H @ mu_x, mu_y, atol=1e-12)
    assert np.allclose(H @ mu_y, mu_x, atol=1e-12)
    Xa = a.Z[:40]
    assert np.allclose(Xa, Xn @ H.T, atol=1e-13)  # x' = H x
    assert np.array_equal(a.Z[40:], Yn)  # Y unchanged
    assert np.allclose(np.linalg.norm(Xa, axis=1), 1.0, atol=1e-13)
    D0 = np.linalg.norm(Xn[:, None] - Xn[None], axis=2)
    D1 = np.linalg.norm(Xa[:, None] - Xa[None], axis=2)
    assert np.allclose(D0, D1, atol=1e-12)
    ma = Xa.mean(0)
    assert math.isclose(np.linalg.norm(ma), np.linalg.norm(Xn.mean(0)), rel_tol=1e-12)
    assert np.allclose(ma / np.linalg.norm(ma), mu_y, atol=1e-12)


def test_app_d_merged_mrl_closed_form(orc):
    """App. D: after H, t = (n||xbar|| + m||ybar||) mu_y and the
    merged MRL equals the upper bound (n||xbar|| + m||ybar||)/(n+m); no other
    orthogonal R (identity, random reflections) exceeds it."""
    spec = HI.PairSpec(50, 70, 64, 60.0, 60.0, 120.0, seed=5)
    X, Y = HI.make_pair(spec)
    a = orc.align(X, Y, 0)
    n = orc.align(X, Y, 1)
    t = a.Z.sum(0)
    Yn = n.Z[50:]
    mu_y = Yn.mean(0) / np.linalg.norm(Yn.mean(0))
    bound = 50 * a.norm_xbar + 70 * a.norm_ybar
    assert np.allclose(t, bound * mu_y, atol=1e-11)
    assert math.isclose(np.linalg.norm(t) / 120, bound / 120, rel_tol=1e-13)
    assert np.linalg.norm(n.Z.sum(0)) < np.linalg.norm(t)
    rng = np.random.default_rng(0)
    for _ in range(20):
        w = rng.standard_normal(64)
        w /= np.linalg.norm(w)
        R = np.eye(64) - 2 * np.outer(w, w)
        merged = np.linalg.norm(n.Z[:50] @ R.T + 0, axis=None)
        merged = np.linalg.norm((n.Z[:50] @ R.T).sum(0) + Yn.sum(0))
        assert merged <= np.linalg.norm(t) + 1e-9


def test_identity_and_degenerate(orc):
    """Coincident means -> identity (R3); antipodal cloud -> DegenerateMean; zero
    row -> ZeroVector with its index."""
    X = np.array([[1, 0, 0], [0, 1, 0]], np.float32)
    a = orc.align(X, X.copy(), 0)
    assert a.status == 0 and a.is_identity and np.array_equal(a.Z[:2], a.Z[2:])
    a = orc.align(np.array([[1, 0], [-1, 0]], np.float32), np.array([[0, 1]], np.float32), 0)
    assert a.status == orc.ORC_E_DEGENERATE_MEAN
    a = orc.align(np.array([[1, 0], [0, 0]], np.float32), np.array([[0, 1]], np.float32), 0)
    assert a.status == orc.ORC_E_ZERO_VECTOR and a.bad_row == 1


# ---------------------------------------------------------------- statistic
def test_statistic_rotation_invariance_and_antisymmetry(orc):
    """T_obs(aligned) = T_obs(naive) (r is rotation invariant);
    swapping X and Y negates T."""
    spec = HI.PairSpec(60, 45, 96, 80.0, 40.0, 50.0, seed=9)
    X, Y = HI.make_pair(spec)
    ta = orc.observed(orc.align(X, Y, 0).Z, 60)["T"]
    tn = orc.observed(orc.align(X, Y, 1).Z, 60)["T"]
    ts = orc.observed(orc.align(Y, X, 0).Z, 45)["T"]
    assert math.isclose(ta, tn, rel_tol=1e-11, abs_tol=1e-13)
    assert math.isclose(ta, -ts, rel_tol=1e-11, abs_tol=1e-13)


def test_statistic_brute_force_numpy(orc):
    """group_stats == an independent numpy evaluation via the +-1 sign-matrix
    route of PAPER.md:215-237 (U = S X, sigma = (t +- U)/2), which is a different
    formula from the oracle's direct group sums."""
    rng = np.random.default_rng(1)
    Z = rng.standard_normal((30, 12))
    Z /= np.linalg.norm(Z, axis=1, keepdims=True)
    n = 11
    for _ in range(20):
        g = np.zeros(30, np.uint8)
        g[rng.choice(30, n, replace=False)] = 1
        st = orc.group_stats(Z, n, g)
        s = np.where(g == 1, 1.0, -1.0)
        t = Z.sum(0)
        U = s @ Z
        r1 = np.linalg.norm((t + U) / 2 / n)
        r2 = np.linalg.norm((t - U) / 2 / (30 - n))
        L = lambda r: math.log(r * (12 - r * r) / (1 - r * r))
        assert math.isclose(st["r1"], r1, rel_tol=1e-12)
        assert math.isclose(st["r2"], r2, rel_tol=1e-12)
        assert math.isclose(st["T"], L(r2) - L(r1), rel_tol=1e-10, abs_tol=1e-12)


def test_zero_resultant_group(orc):
    """r1 = 0 -> L1 = -inf -> T = +inf, counted as an exceedance."""
    Z = np.array([[1, 0], [-1, 0], [0, 1], [0.6, 0.8]], float)
    g = np.array([1, 1, 0, 0], np.uint8)
    st = orc.group_stats(Z, 2, g)
    assert st["r1"] == 0.0 and st["T"] == math.inf


def test_monte_carlo_matches_exhaustive(orc):
    """MC p within 3 SE of the exhaustive p for tiny clouds, and
    p >= 1/(B+1)."""
    rng = np.random.default_rng(3)
    B = 4000
    for trial in range(6):
        N = int(rng.integers(5, 9))
        n = int(rng.integers(2, N - 1))
        X = rng.standard_normal((n, 3)).astype(np.float32)
        Y = (rng.standard_normal((N - n, 3)) + 0.5).astype(np.float32)
        r = orc.run_pair(X, Y, B, SEED, s=trial, nthreads=2)
        counts, total = orc.exhaustive(r["Z"], n, r["t_obs"])
        p_ex = counts[0] / total
        p_mc = r["exceed_ge"] / B
        se = math.sqrt(max(p_ex * (1 - p_ex), 1e-12) / B)
        assert abs(p_mc - p_ex) <= 3 * se + 1e-12
        assert r["p_value"] >= 1 / (B + 1)


def test_permuted_sum_moments(orc):
    """With unit rows and uniform n-subsets:
    E[sigma1] = (n/N) t and E||sigma1||^2 = n + n(n-1)(||t||^2 - N)/(N(N-1))."""
    rng = np.random.default_rng(4)
    N, n, d = 24, 9, 5
    Z = rng.standard_normal((N, d)) + 1.0
    Z /= np.linalg.norm(Z, axis=1, keepdims=True)
    t = Z.sum(0)
    B = 20000
    s1 = np.zeros(d)
    q = 0.0
    for b in range(B):
        g = orc.perm_set(SEED, 11, b, N, n).astype(bool)
        v = Z[g].sum(0)
        s1 += v
        q += v @ v
    s1 /= B
    q /= B
    want_q = n + n * (n - 1) * (t @ t - N) / (N * (N - 1))
    assert np.allclose(s1, n / N * t, atol=0.05)
    assert abs(q - want_q) / want_q < 0.01


def test_counts_accumulate_over_shards(orc):
    """Counts are additive over b-ranges (the sharding contract)."""
    X, Y = HI.make_pair(HI.PairSpec(30, 30, 16, 20.0, 20.0, 40.0, seed=2))
    full = orc.run_pair(X, Y, 600, SEED, nthreads=3)
    parts = [orc.run_pair(X, Y, 600, SEED, b_begin=b0, b_end=b1, nthreads=1)
             for b0, b1 in [(0, 100), (100, 350), (350, 600)]]
    for k in ("exceed_ge", "exceed_abs", "flagged"):
        assert full[k] == sum(p[k] for p in parts)


def test_flagged_counter_exact_ties(orc):
    """Pin of the `flagged` counter (R8) by combinatorics alone (tests/tiecase.py):
    a pool of 4 distinct rows with multiplicities (3, 2, 2, 3); the splits that reproduce the
    observed count vector tie T_obs and those with the mirrored vector tie -T_obs, so the
    exhaustive enumeration flags exactly prod C(m_k, c_k) + prod C(m_k, m_k - c_k) splits.
    Every other count vector is checked to lie far outside the tie band, so a flag that
    misses a boundary, double counts, or uses the wrong tau changes the number."""
    import tiecase
    X, Y, order = tiecase.pool()
    ref = orc.run_pair(X, Y, 10, SEED, mode=1)
    want, c_obs, mirror = tiecase.expected_flagged(order)
    # separation: every other count vector's T (one representative split each) is far
    # from both boundaries, so the tie band cannot catch it
    N = len(order)
    for c, mult in tiecase.count_vectors():
        if c in (c_obs, mirror):
            continue
        members, need = [], list(c)
        for i in range(N):
            if need[order[i]] > 0:
                members.append(i)
                need[order[i]] -= 1
        g = np.zeros(N, np.uint8)
        g[members] = 1
        T = orc.group_stats(ref["Z"], 5, g)["T"]
        assert abs(T - ref["t_obs"]) > 1e3 * ref["tau"] and abs(abs(T) - abs(ref["t_obs"])) > 1e3 * ref["tau"]
    assert sum(m for _, m in tiecase.count_vectors()) == math.comb(N, 5)
    counts, total = orc.exhaustive(ref["Z"], 5, ref["t_obs"], ref["tau"])
    assert total == math.comb(N, 5)
    assert int(counts[2]) == want, (int(counts[2]), want)
    # and by Monte Carlo: flagged / B estimates want / C(N, n_x)
    B = 20000
    mc = orc.run_pair(X, Y, B, SEED, mode=1)
    p = want / math.comb(N, 5)
    assert abs(mc["flagged"] / B - p) < 5 * math.sqrt(p * (1 - p) / B)


# ---------------------------------------------------------------- input generator
def test_vmf_generator_mrl():
    """The input generator hits E[MRL] = A_d(kappa) (= 0.75 at the configs' kappa;
    A_d = I_{d/2}/I_{d/2-1}, scipy.special.ive)."""
    from scipy.special import ive
    for d, kappa in [(32, 50.0), (768, 1315.34)]:
        rng = np.random.default_rng(d)
        mu = HI.random_unit(rng, d)
        x = HI.sample_vmf(rng, mu, kappa, 20000)
        A = ive(d / 2, kappa) / ive(d / 2 - 1, kappa)
        assert np.allclose(np.linalg.norm(x, axis=1), 1.0)
        assert abs(float((x @ mu).mean()) - A) < 5e-3


def test_type1_aligned_calibrated(orc):
    """Aligned test is calibrated on equal-kappa clouds with different means
    (PAPER.md:129-133): rejection rate at alpha=0.1 within 3 SE (R=150)."""
    R, B, alpha = 150, 199, 0.10
    rej = 0
    for rep in range(R):
        X, Y = HI.make_pair(HI.PairSpec(60, 60, 32, 50.0, 50.0, 60.0, seed=77), rep)
        r = orc.run_pair(X, Y, B, SEED, s=rep, nthreads=4)
        rej += r["p_value"] <= alpha
    se = math.sqrt(alpha * (1 - alpha) / R)
    assert abs(rej / R - alpha) <= 3 * se


def test_naive_inflates_type1_on_anisotropic_clouds(orc):
    """The north star's calibration pin (§1 Fig. 1: a mean-direction
    difference distorts the naive test's null; PAPER.md:445-448 anisotropy caveat; SURVEY.md
    App. B, R15): under H0 (equal concentration) with mean directions 60 deg apart
    and shared anisotropic noise (hap_inputs.anisotropic_pair), the two-sided rejection rate
    of the naive test at alpha = 0.10 is inflated by > 2.5 SE while the aligned test stays
    within 2 SE of alpha, on the same permutations (R = 600, n = 200/200, d = 768, B = 200).
    Seeded, so the outcome is fixed; the GPU sweep at R = 1000, B = 10^4 is
    profiles/r02_c5_sweep.json."""
    R, n, d, B, alpha = 600, 200, 768, 200, 0.10
    spec = HI.PairSpec(n, n, d, HI.kappa_for(d), HI.kappa_for(d), 60.0, seed=2005)
    rej = {0: 0, 1: 0}
    for rep in range(R):
        X, Y = HI.anisotropic_pair(spec, rep)
        for mode in (0, 1):
            r = orc.run_pair(X, Y, B, SEED, s=rep, mode=mode, nthreads=8)
            rej[mode] += orc.pvalue(r["exceed_abs"], B) <= alpha
    se = math.sqrt(alpha * (1 - alpha) / R)
    aligned, naive = rej[0] / R, rej[1] / R
    assert abs(aligned - alpha) <= 2 * se, (aligned, naive)
    assert naive - alpha >= 2.5 * se, (aligned, naive)
