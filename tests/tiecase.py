"""A pooled cloud with exactly predictable near-ties, for pinning the `flagged` counter.

The pool holds K distinct raw rows v_k with multiplicities m_k (identical rows = identical
contexts).  In naive mode (no reflection) a split's statistic depends only on
its count vector c (c_k copies of v_k in group 1), so every split with the observed count
vector c_obs has T = T_obs, and with n_x = n_y every split with the mirrored vector
m - c_obs has T = -T_obs (the groups swap roles): both are near-ties of
DESIGN.md R8 (the first of T_obs, the second of |T_obs|).  The number of splits with count
vector c is prod_k C(m_k, c_k), so over the exhaustive enumeration

    flagged = prod_k C(m_k, c_obs_k) + prod_k C(m_k, m_k - c_obs_k)

provided no other count vector's T comes within the tie band of T_obs or -T_obs (checked
by the test with a wide margin).  Plain combinatorics; no statistic arithmetic.
"""
from __future__ import annotations

import itertools
import math

import numpy as np

MULT = (3, 2, 2, 3)           # m_k; N = 10
D = 5


def pool():
    """(X, Y) raw fp32 rows (n_x = n_y = 5) and the distinct-row index of every pooled row."""
    rng = np.random.default_rng(20261019)
    V = rng.standard_normal((len(MULT), D)) + 2.0 * np.eye(len(MULT), D)
    V *= rng.uniform(5.0, 20.0, size=(len(MULT), 1))     # raw (non-unit) norms
    kinds = [k for k, m in enumerate(MULT) for _ in range(m)]
    order = [0, 3, 1, 0, 2, 3, 1, 2, 0, 3]                   # a fixed interleaving
    assert sorted(order) == sorted(kinds)
    Z = V[order].astype(np.float32)
    return Z[:5].copy(), Z[5:].copy(), order


def count_vector(members, order):
    c = [0] * len(MULT)
    for i in members:
        c[order[i]] += 1
    return tuple(c)


def multiplicity(c):
    return math.prod(math.comb(m, k) for m, k in zip(MULT, c))


def expected_flagged(order, n_x=5):
    c_obs = count_vector(range(n_x), order)
    mirror = tuple(m - k for m, k in zip(MULT, c_obs))
    assert mirror != c_obs
    return multiplicity(c_obs) + multiplicity(mirror), c_obs, mirror


def count_vectors(n_x=5):
    """Every count vector with sum n_x and its multiplicity (sums to C(N, n_x))."""
    for c in itertools.product(*[range(m + 1) for m in MULT]):
        if sum(c) == n_x:
            yield c, multiplicity(c)
