"""TEST INFRASTRUCTURE ONLY -- NumPy restatement of the reference's NDCT for
the sizes where the C oracle's radix-2 chirp-z r2r backend is too slow or too
large (N = 2^20 .. 2^26 full vectors).

Same algorithm and operation order as the C restatement
(oracle/fastleg_oracle.c), which is pinned bit for bit to the compiled
reference; only the FFT boundary differs: FFTW's REDFT01 / RODFT01 /
REDFT10 / RODFT10 (absent from the image) are scipy.fft's
pocketfft dct/dst types 3 and 2 (unnormalised, the same definitions), run on
all host threads. This restatement is pinned against the C oracle at
moderate N by tests/test_oracle_pins.py (by tolerance: the FFT rounding
differs).

  trig.hpp:55-74   dct_iii            trig.hpp:100-116 dct_iii_transpose
  trig.hpp:76-95   dst_iii            trig.hpp:118-136 dst_iii_transpose
  ndct.hpp:77      taylor_sign        ndct.hpp:98-117  ndct_apply
  ndct.hpp:121-143 ndct_apply_transpose
"""
from __future__ import annotations

import os

import numpy as np
import scipy.fft as sf

CHEB1, CHEBSTAR = 0, 1
WORKERS = os.cpu_count() or 1


def _redft01(v):  # FFTW REDFT01: X_0 + 2 sum_{j>=1} X_j cos(pi j (k+1/2)/n)
    return sf.dct(v, type=3, workers=WORKERS)


def _rodft01(v):  # FFTW RODFT01: (-1)^k X_{n-1} + 2 sum_{j<n-1} X_j sin(pi (j+1)(k+1/2)/n)
    return sf.dst(v, type=3, workers=WORKERS)


def _redft10(v):  # FFTW REDFT10: 2 sum_j X_j cos(pi (j+1/2) k / n)
    return sf.dct(v, type=2, workers=WORKERS)


def _rodft10(v):  # FFTW RODFT10: 2 sum_j X_j sin(pi (j+1/2)(k+1) / n)
    return sf.dst(v, type=2, workers=WORKERS)


def dct_iii(c: np.ndarray, kind: int) -> np.ndarray:  # trig.hpp:55-74
    n = len(c)
    if kind == CHEB1:
        a = 0.5 * c
        a[0] = c[0]
        return _redft01(a)
    m = 2 * n + 1
    a = np.zeros(m)
    a[:n] = 0.5 * c
    a[0] = c[0]
    return _redft01(a)[1::2][:n]


def dst_iii(c: np.ndarray, kind: int) -> np.ndarray:  # trig.hpp:76-95
    n = len(c)
    if kind == CHEB1:
        if n == 1:
            return np.zeros(1)
        a = np.zeros(n)
        a[:n - 1] = 0.5 * c[1:]
        return _rodft01(a)
    m = 2 * n + 1
    a = np.zeros(m)
    a[:n - 1] = 0.5 * c[1:]
    return _rodft01(a)[1::2][:n]


def dct_iii_transpose(g: np.ndarray, kind: int) -> np.ndarray:  # trig.hpp:100-116
    n = len(g)
    if kind == CHEB1:
        return 0.5 * _redft10(g)
    m = 2 * n + 1
    a = np.zeros(m)
    a[1::2][:n] = g
    return 0.5 * _redft10(a)[:n]


def dst_iii_transpose(g: np.ndarray, kind: int) -> np.ndarray:  # trig.hpp:118-136
    n = len(g)
    out = np.zeros(n)
    if n == 1:
        return out
    if kind == CHEB1:
        out[1:] = 0.5 * _rodft10(g)[:n - 1]
        return out
    m = 2 * n + 1
    a = np.zeros(m)
    a[1::2][:n] = g
    out[1:] = 0.5 * _rodft10(a)[:n - 1]
    return out


def taylor_sign(l: int) -> float:  # ndct.hpp:77
    return 1.0 if ((l + 1) // 2) % 2 == 0 else -1.0


def ndct_apply(c, kind: int, num_terms: int, delta, lo: int = 0) -> np.ndarray:  # ndct.hpp:98-117
    """Taylor terms l in [lo, num_terms) (lo = 0: the whole ndct_apply)."""
    c = np.asarray(c, dtype=np.float64)
    delta = np.asarray(delta, dtype=np.float64)
    n = len(c)
    j = np.arange(n, dtype=np.float64)
    f = np.zeros(n)
    stage = c.copy()
    perturb = np.ones(n)
    for l in range(num_terms):
        if l > 0:
            stage *= j
            perturb *= delta / float(l)
        if l < lo:
            continue
        t = dct_iii(stage, kind) if l % 2 == 0 else dst_iii(stage, kind)
        f += taylor_sign(l) * perturb * t
    return f


def ndct_apply_transpose(v, kind: int, num_terms: int, delta, lo: int = 0) -> np.ndarray:  # ndct.hpp:121-143
    """Taylor terms l in [lo, num_terms) of ndct_apply_transpose."""
    v = np.asarray(v, dtype=np.float64)
    delta = np.asarray(delta, dtype=np.float64)
    n = len(v)
    j = np.arange(n, dtype=np.float64)
    out = np.zeros(n)
    degree = np.ones(n)
    perturb = np.ones(n)
    for l in range(num_terms):
        if l > 0:
            degree *= j
            perturb *= delta / float(l)
        if l < lo:
            continue
        h = perturb * v
        t = dct_iii_transpose(h, kind) if l % 2 == 0 else dst_iii_transpose(h, kind)
        out += taylor_sign(l) * degree * t
    return out


def leg2cheb_rows(c, s, rows) -> np.ndarray:
    """conversion.hpp:106-111 for chosen rows k (O(N) each): (2 - delta_k0)
    sum_{j: k+2j<N} s_j s_{k+j} c_{k+2j}, s = scaled Lambda table."""
    c = np.asarray(c, dtype=np.float64)
    n = len(c)
    out = []
    for k in rows:
        j = np.arange((n - k + 1) // 2)
        out.append((1.0 if k == 0 else 2.0) * np.sum(s[j] * s[k + j] * c[k + 2 * j]))
    return np.array(out)


def leg2cheb_transpose_rows(v, s, rows) -> np.ndarray:
    """conversion.hpp:126-133 for chosen rows m: 2 sum_{2j<m} s_j s_{m-j}
    v_{m-2j} + [m even] s_{m/2} s_{m-m/2} v_0."""
    v = np.asarray(v, dtype=np.float64)
    out = []
    for m in rows:
        j = np.arange((m + 1) // 2)
        acc = 2.0 * np.sum(s[j] * s[m - j] * v[m - 2 * j])
        if m % 2 == 0:
            acc += s[m // 2] * s[m - m // 2] * v[0]
        out.append(acc)
    return np.array(out)
