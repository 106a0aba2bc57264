"""Seeded synthetic inputs shared by the oracle tests, the GPU parity tests, smoke()
and bench.py.

This module holds NONE of the method's arithmetic (no normalisation, means,
reflection, statistic, permutation or counting): it only draws raw embedding
clouds h_i = s_i * x_i with x_i ~ vMF(mu, kappa) (Wood 1994) and BERT-like raw
norms s_i ~ LogNormal(ln 20, 0.1), as recorded in DESIGN.md "Input recipe"
(SURVEY.md §8d).
"""
from __future__ import annotations

import math
from dataclasses import dataclass

import numpy as np

PERM_SEED = 0x0123456789ABCDEF


def random_unit(rng: np.random.Generator, d: int) -> np.ndarray:
    v = rng.standard_normal(d)
    return v / np.linalg.norm(v)


def at_angle(rng: np.random.Generator, mu: np.ndarray, theta_deg: float) -> np.ndarray:
    """A unit vector at angle theta from mu, in a random 2-plane containing mu."""
    w = rng.standard_normal(mu.shape[0])
    w -= mu * (w @ mu)
    w /= np.linalg.norm(w)
    th = math.radians(theta_deg)
    return math.cos(th) * mu + math.sin(th) * w


def sample_vmf(rng: np.random.Generator, mu: np.ndarray, kappa: float, n: int) -> np.ndarray:
    """n draws from vMF(mu, kappa) on S^{d-1} (Wood 1994 rejection sampler), fp64."""
    d = mu.shape[0]
    if kappa <= 0:
        v = rng.standard_normal((n, d))
        return v / np.linalg.norm(v, axis=1, keepdims=True)
    dm1 = d - 1.0
    b = dm1 / (2.0 * kappa + math.sqrt(4.0 * kappa * kappa + dm1 * dm1))
    x0 = (1.0 - b) / (1.0 + b)
    c = kappa * x0 + dm1 * math.log(1.0 - x0 * x0)
    w = np.empty(n)
    todo = np.arange(n)
    while todo.size:
        z = rng.beta(dm1 / 2.0, dm1 / 2.0, size=todo.size)
        ww = (1.0 - (1.0 + b) * z) / (1.0 - (1.0 - b) * z)
        u = rng.random(todo.size)
        ok = kappa * ww + dm1 * np.log(1.0 - x0 * ww) - c >= np.log(u)
        w[todo[ok]] = ww[ok]
        todo = todo[~ok]
    v = rng.standard_normal((n, d))
    v -= np.outer(v @ mu, mu)
    v /= np.linalg.norm(v, axis=1, keepdims=True)
    return w[:, None] * mu[None, :] + np.sqrt(np.clip(1.0 - w * w, 0.0, None))[:, None] * v


def raw_cloud(rng: np.random.Generator, mu: np.ndarray, kappa: float, n: int,
              norm_median: float = 20.0, norm_sigma: float = 0.1) -> np.ndarray:
    """Raw (non-unit) fp32 embeddings h_i = s_i x_i, s_i ~ LogNormal(ln 20, 0.1)."""
    x = sample_vmf(rng, mu, kappa, n)
    s = rng.lognormal(math.log(norm_median), norm_sigma, size=n)
    return (x * s[:, None]).astype(np.float32)


# kappa giving E[MRL] = A_d(kappa) = 0.75 (SURVEY.md §8c "vMF sampler" row)
KAPPA_R075 = {768: 1315.34, 4096: 7020.48, 32: 53.627}


def mrl_vmf(d: int, kappa: float) -> float:
    """E[MRL] of vMF(kappa) on S^{d-1}: A_d(kappa) = I_{d/2}(kappa) / I_{d/2-1}(kappa)."""
    import scipy.special as sp
    return float(sp.ive(d / 2.0, kappa) / sp.ive(d / 2.0 - 1.0, kappa))


def kappa_for_r(d: int, r: float) -> float:
    """kappa with A_d(kappa) = r (0.5 <= r < 1): the concentration of a cloud whose mean
    resultant length is r (narrow words r ~ 0.96, near-duplicate clouds r -> 1)."""
    import scipy.optimize as so
    return float(so.brentq(lambda k: mrl_vmf(d, k) - r, d * r,
                           2.0 * d / (1.0 - r) + 10.0, xtol=1e-9, rtol=1e-13))


def kappa_for(d: int) -> float:
    if d in KAPPA_R075:
        return KAPPA_R075[d]
    # A_d(k) ~ k/(k + (d-1)/2 ...) for large d: solve A = 0.75 approximately
    return 0.75 * (d - 1) / (1 - 0.75 ** 2) * 0.98


@dataclass
class PairSpec:
    n_x: int
    n_y: int
    d: int
    kappa_x: float
    kappa_y: float
    theta_deg: float = 30.0
    seed: int = 1000


def make_pair(spec: PairSpec, rep: int = 0):
    """Seeded pair (X, Y) of raw fp32 clouds: equal concentration, mean directions
    at angle theta (the H0 of PAPER.md:129-133 with E[X] != E[Y])."""
    rng = np.random.default_rng([spec.seed, rep])
    mu_x = random_unit(rng, spec.d)
    mu_y = at_angle(rng, mu_x, spec.theta_deg)
    X = raw_cloud(rng, mu_x, spec.kappa_x, spec.n_x)
    Y = raw_cloud(rng, mu_y, spec.kappa_y, spec.n_y)
    return X, Y


def anisotropic_pair(spec: PairSpec, rep: int = 0, n_coords: int = 16, scale: float = 6.0):
    """Anisotropic variant: shared noise scaled `scale`x on
    `n_coords` fixed coordinates, added before the raw-norm scaling."""
    rng = np.random.default_rng([spec.seed, rep, 7])
    mu_x = random_unit(rng, spec.d)
    mu_y = at_angle(rng, mu_x, spec.theta_deg)
    coords = np.arange(n_coords)

    def cloud(mu, kappa, n):
        x = sample_vmf(rng, mu, kappa, n)
        noise = rng.standard_normal((n, n_coords)) * (scale / math.sqrt(spec.d))
        x[:, coords] += noise
        s = rng.lognormal(math.log(20.0), 0.1, size=n)
        return (x * s[:, None]).astype(np.float32)

    return cloud(mu_x, spec.kappa_x, spec.n_x), cloud(mu_y, spec.kappa_y, spec.n_y)


# BASELINE.json configs (data seed = 1000 + config index)
CONFIGS = {
    "C1": dict(n_x=64, n_y=64, d=768, B=1000),
    "C2": dict(n_x=1000, n_y=1000, d=768, B=10000),
    "C3": dict(n_x=5000, n_y=5000, d=4096, B=100000),
    "C4": dict(P=10000, n_min=50, n_max=5000, d=768, B=10000),
    "C5": dict(R=1000, n_x=500, n_y=500, d=768, B=10000),
}


def config_pair(name: str, rep: int = 0, theta_deg: float = 30.0):
    c = CONFIGS[name]
    idx = int(name[1:])
    spec = PairSpec(c["n_x"], c["n_y"], c["d"], kappa_for(c["d"]), kappa_for(c["d"]),
                    theta_deg, seed=1000 + idx)
    return make_pair(spec, rep)


def c4_sizes(P: int, n_min: int = 50, n_max: int = 5000, seed: int = 1004) -> np.ndarray:
    """Log-uniform pair sizes n_p in [n_min, n_max] (Zipf-like frequencies)."""
    rng = np.random.default_rng(seed)
    return np.exp(rng.uniform(math.log(n_min), math.log(n_max), size=P)).astype(np.int64)


def duplicated_pair(spec: PairSpec, rep: int = 0, n_distinct_x: int = 8, n_distinct_y: int = 8,
                    frac: float = 0.5):
    """make_pair, then a fraction `frac` of each cloud's rows replaced by exact copies of
    that cloud's first n_distinct rows (identical contexts give identical embeddings)."""
    X, Y = make_pair(spec, rep)
    rng = np.random.default_rng([spec.seed, rep, 11])
    for M, nd in ((X, n_distinct_x), (Y, n_distinct_y)):
        n = M.shape[0]
        nd = max(1, min(nd, n))
        k = int(round(frac * (n - nd)))
        rows = rng.choice(np.arange(nd, n), size=k, replace=False) if k > 0 else []
        for i in rows:
            M[i] = M[int(rng.integers(0, nd))]
    return X, Y


def dyadic_pair(rng: np.random.Generator, n_x: int, n_y: int, d: int, ks=(1, 4, 16)):
    """Already-unit rows with k in `ks` nonzero entries of magnitude 1/sqrt(k)
    (1, 1/2, 1/4): exact in bf16 and all their group sums are exact, so with no
    reflection (naive mode) every sum on both sides is exact."""
    def rows(n):
        m = np.zeros((n, d), dtype=np.float32)
        for i in range(n):
            k = int(rng.choice([k for k in ks if k <= d]))
            cols = rng.choice(d, size=k, replace=False)
            m[i, cols] = rng.choice([-1.0, 1.0], size=k) / math.sqrt(k)
        return m
    return rows(n_x), rows(n_y)


def varlen_batch(sizes, d: int = 768, seed: int = 1004, theta_deg: float = 30.0,
                 ny_sizes=None):
    """Packed varlen batch (C4 recipe): pair p is an independent vMF pair
    with n_X = sizes[p], n_Y = ny_sizes[p] (default n_X), kappa(r=0.75) for d, mean
    directions at theta_deg.  Returns (X_packed, cu_nx, Y_packed, cu_ny) with cu_* the
    int64 prefix offsets [P+1] (FlashAttention-style)."""
    sizes = [int(s) for s in sizes]
    ny_sizes = sizes if ny_sizes is None else [int(s) for s in ny_sizes]
    Xs, Ys = [], []
    k = kappa_for(d)
    for p, (nx, ny) in enumerate(zip(sizes, ny_sizes)):
        X, Y = make_pair(PairSpec(nx, ny, d, k, k, theta_deg, seed=seed), rep=p)
        Xs.append(X)
        Ys.append(Y)
    cu_nx = np.concatenate([[0], np.cumsum(sizes)]).astype(np.int64)
    cu_ny = np.concatenate([[0], np.cumsum(ny_sizes)]).astype(np.int64)
    return (np.ascontiguousarray(np.concatenate(Xs)), cu_nx,
            np.ascontiguousarray(np.concatenate(Ys)), cu_ny)
