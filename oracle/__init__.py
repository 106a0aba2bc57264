"""fp64 CPU ORACLE for the Householder-aligned permutation test (arXiv 2605.08048).

TEST INFRASTRUCTURE ONLY.  Only ``tests/``, ``__graft_entry__.smoke()`` and
``bench.py``'s ``cpu_baseline`` / ``--impl reference`` leg may import this
package.  The product path (``paper_2605_08048_b200``) never imports it, and the
two share no code: this module wraps ``hap_oracle.c`` (plain C, fp64, plain
loops) through ctypes and numpy.

Pins: see ``hap_oracle.h`` and ``tests/test_oracle_*.py``.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "hap_oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")

ORC_OK, ORC_E_ARG, ORC_E_ZERO_VECTOR, ORC_E_DEGENERATE_MEAN = 0, 1, 2, 3


def build(force: bool = False) -> str:
    """Compile the oracle with gcc (-O2, no fast-math: IEEE fp64 throughout)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < max(
            os.path.getmtime(_SRC), os.path.getmtime(os.path.join(_HERE, "hap_oracle.h"))):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", "-O2", "-std=c11", "-fPIC", "-shared", "-fno-fast-math",
                               "-ffp-contract=off", "-o", tmp, _SRC, "-lm", "-lpthread"])
        os.replace(tmp, _LIB)
    return _LIB


_lib = None


def lib():
    global _lib
    if _lib is None:
        L = ctypes.CDLL(build())
        P = ctypes.POINTER
        u8p, f32p, f64p, u32p, u64p = (P(ctypes.c_uint8), P(ctypes.c_float), P(ctypes.c_double),
                                       P(ctypes.c_uint32), P(ctypes.c_uint64))
        i64, u64, u32 = ctypes.c_int64, ctypes.c_uint64, ctypes.c_uint32
        L.orc_philox4x32_10.argtypes = [u32p, u32p, u32p]
        L.orc_perm_set.argtypes = [u64, u32, u32, i64, i64, u8p]
        L.orc_perm_set.restype = ctypes.c_int
        L.orc_align.argtypes = [f32p, i64, f32p, i64, i64, ctypes.c_int, f64p, f64p, f64p]
        L.orc_align.restype = ctypes.c_int
        L.orc_logkappa.argtypes = [ctypes.c_double, i64]
        L.orc_logkappa.restype = ctypes.c_double
        L.orc_group_stats.argtypes = [f64p, i64, i64, i64, u8p, f64p]
        L.orc_permtest.argtypes = [f64p, i64, i64, i64, u64, u32, u64, u64, ctypes.c_double,
                                   ctypes.c_double, ctypes.c_int, u64p, f64p]
        L.orc_exhaustive.argtypes = [f64p, i64, i64, i64, ctypes.c_double, ctypes.c_double, u64p]
        L.orc_exhaustive.restype = i64
        L.orc_pvalue.argtypes = [u64, u64]
        L.orc_pvalue.restype = ctypes.c_double
        _lib = L
    return _lib


def _ptr(a: np.ndarray, ct):
    return a.ctypes.data_as(ctypes.POINTER(ct))


def philox4x32_10(ctr, key) -> np.ndarray:
    c = np.ascontiguousarray(ctr, dtype=np.uint32)
    k = np.ascontiguousarray(key, dtype=np.uint32)
    o = np.zeros(4, dtype=np.uint32)
    lib().orc_philox4x32_10(_ptr(c, ctypes.c_uint32), _ptr(k, ctypes.c_uint32),
                            _ptr(o, ctypes.c_uint32))
    return o


def perm_set(seed: int, s: int, b: int, N: int, n_x: int) -> np.ndarray:
    """PERM-SPEC v1 group-1 membership (uint8[N])."""
    g = np.zeros(N, dtype=np.uint8)
    rc = lib().orc_perm_set(seed, s, b, N, n_x, _ptr(g, ctypes.c_uint8))
    if rc < 0:
        raise ValueError("bad perm_set arguments")
    return g


def perm_set_redraws(seed: int, s: int, b: int, N: int, n_x: int) -> int:
    g = np.zeros(N, dtype=np.uint8)
    return lib().orc_perm_set(seed, s, b, N, n_x, _ptr(g, ctypes.c_uint8))


class AlignResult:
    def __init__(self, Z, u, info, status, d, n_x, n_y):
        self.Z, self.u, self.status = Z, u, status
        self.norm_xbar, self.norm_ybar = float(info[0]), float(info[1])
        self.is_identity = bool(info[2] != 0.0)
        self.bad_row = int(info[3])
        self.d, self.n_x, self.n_y = d, n_x, n_y


def align(X: np.ndarray, Y: np.ndarray, mode: int = 0) -> AlignResult:
    X = np.ascontiguousarray(X, dtype=np.float32)
    Y = np.ascontiguousarray(Y, dtype=np.float32)
    n_x, d = X.shape
    n_y = Y.shape[0]
    Z = np.zeros((n_x + n_y, d), dtype=np.float64)
    u = np.zeros(d, dtype=np.float64)
    info = np.zeros(4, dtype=np.float64)
    st = lib().orc_align(_ptr(X, ctypes.c_float), n_x, _ptr(Y, ctypes.c_float), n_y, d, mode,
                         _ptr(Z, ctypes.c_double), _ptr(u, ctypes.c_double),
                         _ptr(info, ctypes.c_double))
    return AlignResult(Z, u, info, st, d, n_x, n_y)


def logkappa(r: float, d: int) -> float:
    return lib().orc_logkappa(float(r), int(d))


def group_stats(Z: np.ndarray, n_x: int, in_g1: np.ndarray) -> dict:
    Z = np.ascontiguousarray(Z, dtype=np.float64)
    g = np.ascontiguousarray(in_g1, dtype=np.uint8)
    N, d = Z.shape
    out = np.zeros(5, dtype=np.float64)
    lib().orc_group_stats(_ptr(Z, ctypes.c_double), N, d, n_x, _ptr(g, ctypes.c_uint8),
                          _ptr(out, ctypes.c_double))
    return dict(r1=out[0], r2=out[1], L1=out[2], L2=out[3], T=out[4])


def observed(Z: np.ndarray, n_x: int) -> dict:
    """T_obs on the observed split {0..n_x-1} (Alg. 1 step 4)."""
    g = np.zeros(Z.shape[0], dtype=np.uint8)
    g[:n_x] = 1
    return group_stats(Z, n_x, g)


def tie_tau(L1: float, L2: float, tie_rel: float = 1e-6) -> float:
    """Tie band tau = tie_rel * (|L(r_X)| + |L(r_Y)|) (R8)."""
    return tie_rel * (abs(L1) + abs(L2))


def permtest(Z: np.ndarray, n_x: int, seed: int, s: int, b_begin: int, b_end: int, t_obs: float,
             tau: float, nthreads: int | None = None, want_stats: bool = False):
    Z = np.ascontiguousarray(Z, dtype=np.float64)
    N, d = Z.shape
    counts = np.zeros(3, dtype=np.uint64)
    stats = np.zeros((max(b_end - b_begin, 0), 3), dtype=np.float64) if want_stats else None
    nthreads = nthreads or (os.cpu_count() or 1)
    lib().orc_permtest(_ptr(Z, ctypes.c_double), N, d, n_x, seed, s, b_begin, b_end,
                       float(t_obs), float(tau), nthreads, _ptr(counts, ctypes.c_uint64),
                       _ptr(stats, ctypes.c_double) if want_stats else None)
    return (counts, stats) if want_stats else counts


def exhaustive(Z: np.ndarray, n_x: int, t_obs: float, tau: float = 0.0):
    Z = np.ascontiguousarray(Z, dtype=np.float64)
    N, d = Z.shape
    counts = np.zeros(3, dtype=np.uint64)
    total = lib().orc_exhaustive(_ptr(Z, ctypes.c_double), N, d, n_x, float(t_obs), float(tau),
                                 _ptr(counts, ctypes.c_uint64))
    return counts, int(total)


def pvalue(exceed: int, B: int) -> float:
    return lib().orc_pvalue(int(exceed), int(B))


def run_pair(X, Y, B: int, seed: int, s: int = 0, mode: int = 0, tie_rel: float = 1e-6,
             nthreads: int | None = None, b_begin: int = 0, b_end: int | None = None,
             want_stats: bool = False) -> dict:
    """Alg. 1 end to end (normalise -> align -> T_obs -> permutations -> p)."""
    a = align(X, Y, mode)
    if a.status != ORC_OK:
        return dict(status=a.status, bad_row=a.bad_row)
    n_x = X.shape[0]
    ob = observed(a.Z, n_x)
    tau = tie_tau(ob["L1"], ob["L2"], tie_rel)
    b_end = B if b_end is None else b_end
    res = permtest(a.Z, n_x, seed, s, b_begin, b_end, ob["T"], tau, nthreads, want_stats)
    counts, stats = res if want_stats else (res, None)
    return dict(status=ORC_OK, t_obs=ob["T"], r_x=ob["r1"], r_y=ob["r2"], L_x=ob["L1"],
                L_y=ob["L2"], tau=tau, exceed_ge=int(counts[0]), exceed_abs=int(counts[1]),
                flagged=int(counts[2]), p_value=pvalue(int(counts[0]), B), stats=stats,
                is_identity=a.is_identity, Z=a.Z, u=a.u)
