"""Closed-form Haar-basis reference — TEST INFRASTRUCTURE ONLY (see oracle/__init__.py).

An independent second definition of the same linear map as oracle/haar.py: instead of
iterating the filter bank, every coefficient is written as an explicit (signed) block sum of
the input, i.e. the orthonormal Haar basis functions (textbook form of the transform whose
Fast structure PAPER.md §III-§IV derives; basis normalisation fixed by the §II taps ±1/√2,
PAPER.md:54).  It pins the filter-bank oracle (tests/test_oracle_pins.py) and, on integer
inputs, gives EXACT dyadic-rational coefficients (int64 block sums, one power-of-two scale),
which the c3 bit-exactness check uses.

Conventions (readings R1, R2, R7, R8):
  1-D detail_j[k] = 2^(-j/2) (sum of first half - sum of second half of block [k 2^j, (k+1) 2^j))
  1-D approx_J[k] = 2^(-J/2) (sum of block [k 2^J, (k+1) 2^J))
  2-D level j, block (p, q) of size 2^j x 2^j with quadrants TL TR / BL BR:
      LL = 2^-j (TL+TR+BL+BR), HL = 2^-j (TL-TR+BL-BR), LH = 2^-j (TL+TR-BL-BR), HH = 2^-j (TL-TR-BL+BR)
  Mallat placement as in oracle/haar.py.
"""
from __future__ import annotations

import math

import numpy as np


def haar_matrix_1d(n: int, levels: int) -> np.ndarray:
    """Rows are the orthonormal Haar basis functions, in Mallat order [a_J | d_J | ... | d_1]."""
    assert levels >= 1 and n % (1 << levels) == 0
    m = np.zeros((n, n))
    bj = 1 << levels
    for k in range(n // bj):
        m[k, k * bj:(k + 1) * bj] = 2.0 ** (-levels / 2.0)
    for j in range(1, levels + 1):
        b = 1 << j
        base = n >> j
        for k in range(n // b):
            m[base + k, k * b:k * b + b // 2] = 2.0 ** (-j / 2.0)
            m[base + k, k * b + b // 2:(k + 1) * b] = -(2.0 ** (-j / 2.0))
    return m


def closed_form_1d(x, levels: int) -> np.ndarray:
    x = np.asarray(x, dtype=np.float64)
    return x @ haar_matrix_1d(x.shape[-1], levels).T


def _quadrant_sums(x, j):
    """Sums of the four 2^(j-1) x 2^(j-1) quadrants of every 2^j x 2^j block."""
    b, hb = 1 << j, 1 << (j - 1)
    h, w = x.shape[-2], x.shape[-1]
    blk = x.reshape(x.shape[:-2] + (h // b, 2, hb, w // b, 2, hb))
    q = blk.sum(axis=(-4, -1))            # (..., h/b, 2, w/b, 2): [row half, col half]
    return q[..., 0, :, 0], q[..., 0, :, 1], q[..., 1, :, 0], q[..., 1, :, 1]


def closed_form_2d(x, levels: int, exact_int: bool = False) -> np.ndarray:
    """Explicit block-sum formula for the whole L-level Mallat pyramid over the last two axes.

    exact_int=True: x must hold integers; sums are taken in int64 and scaled by 2^-j once,
    which is exact in fp64 (and in fp32 while the sums stay below 2^24)."""
    x = np.asarray(x)
    h, w = x.shape[-2], x.shape[-1]
    assert levels >= 1 and h % (1 << levels) == 0 and w % (1 << levels) == 0
    if exact_int:
        xi = x.astype(np.int64)
        assert np.array_equal(xi, x), "exact_int needs integer-valued input"
    else:
        xi = x.astype(np.float64)
    out = np.zeros(x.shape, dtype=np.float64)
    for j in range(1, levels + 1):
        tl, tr, bl, br = _quadrant_sums(xi, j)
        sc = 2.0 ** (-j)
        hj, wj = h >> j, w >> j
        out[..., :hj, wj:2 * wj] = (tl - tr + bl - br) * sc       # HL
        out[..., hj:2 * hj, :wj] = (tl + tr - bl - br) * sc       # LH
        out[..., hj:2 * hj, wj:2 * wj] = (tl - tr - bl + br) * sc  # HH
        if j == levels:
            out[..., :hj, :wj] = (tl + tr + bl + br) * sc         # LL_L
    return out


def closed_form_2d_block(x_block, levels: int) -> dict:
    """All coefficients of ONE 2^L x 2^L block, keyed (level, band) -> array, band in
    {'LL','HL','LH','HH'} (LL only at level L).  Used for sampled full-size parity checks."""
    x = np.asarray(x_block, dtype=np.float64)
    res = {}
    for j in range(1, levels + 1):
        tl, tr, bl, br = _quadrant_sums(x, j)
        sc = 2.0 ** (-j)
        res[(j, "HL")] = (tl - tr + bl - br) * sc
        res[(j, "LH")] = (tl + tr - bl - br) * sc
        res[(j, "HH")] = (tl - tr - bl + br) * sc
        if j == levels:
            res[(j, "LL")] = (tl + tr + bl + br) * sc
    return res


def sqrt2_power(e: float) -> float:
    return math.pow(2.0, e / 2.0)
