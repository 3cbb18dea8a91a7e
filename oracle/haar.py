"""fp64 CPU ORACLE of the paper's Haar filter bank — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg may
import this module.  The product path (paper_1002_2184_b200/) never imports it and shares no
code, constants or helpers with it; the two meet only through datagen/ (seeded inputs).

What it computes (plain definitions, written out, no blocking or fusion):

* ``direct_analysis`` — the DIRECT two-channel analysis bank of PAPER.md:58-74 (§III, Fig. 2,
  Eqs. (1)-(4)): full-rate convolution with the §II analysis taps
  b0 = [1/√2, 1/√2], b1 = [-1/√2, 1/√2], followed by ↓2 keeping phase n = 2k+1
  (reading R1 = SURVEY §8(c) A1).
* ``direct_synthesis`` — the DIRECT synthesis bank of PAPER.md:128-136 (§IV, Fig. 5, Eq. (13)):
  ↑2 by zero insertion, convolution with a0 = [1/√2, 1/√2], a1 = [1/√2, -1/√2],
  sum.  Unity gain: the factor 2 of Eq. (14) is not applied (reading R3 = A3).
* ``fast_analysis`` / ``fast_synthesis`` — the paper's polyphase "Fast Haar" banks (Fig. 4,
  PAPER.md:118-124; Fig. 7): split into even/odd polyphase components, one
  butterfly scaled by b00 = a00 = 1/√2.  Used only to pin the paper's own claim that the
  two structures agree and the op-count claim.
* ``decompose_1d`` / ``reconstruct_1d`` — Mallat recursion on the approximation band
  (not in the paper, reading R7 = A7), flat layout [a_J | d_J | ... | d_1].
* ``analyze_2d`` / ``synthesize_2d`` — separable 2-D application (§V; rows then
  columns, reading R8 = A8), Mallat quadrants [[LL, HL], [LH, HH]], recursion
  on LL.

Every function is pinned by tests/test_oracle_pins.py against values and identities that do
not come from this file: printed worked examples, hand-computed fixtures
(tests/golden/), an explicit closed-form Haar basis matrix, torch's avg_pool2d, perfect
reconstruction, energy, linearity and separability.  No function here is "parity unpinned".
"""
from __future__ import annotations

import math

import numpy as np


# --------------------------------------------------------------------------- errors
class OracleError(ValueError):
    pass


class OddLength(OracleError):
    pass


class EmptySignal(OracleError):
    pass


class InvalidLevels(OracleError):
    pass


class InsufficientLength(OracleError):
    pass


class LengthMismatch(OracleError):
    pass


class DimensionMismatch(OracleError):
    pass


# --------------------------------------------------------------------------- §II taps
S = 1.0 / math.sqrt(2.0)   # computed once in fp64


def filter_bank():
    """§II Haar coefficient sets.  Tap k multiplies x[n-k]."""
    return {
        "b0": (S, S),      # analysis LPF  [1/√2, 1/√2]
        "b1": (-S, S),     # analysis HPF  [-1/√2, 1/√2]
        "a0": (S, S),      # synthesis LPF [1/√2, 1/√2]
        "a1": (S, -S),     # synthesis HPF [1/√2, -1/√2]
        "b00": S,          # polyphase component b00(n) = a00(n) = 1/√2
        "M": 2,            # decimation factor
    }


class OpCounter:
    """Counts multiplications and additions on sample data."""

    def __init__(self):
        self.mul = 0
        self.add = 0


def _mul(c, x, ops):
    if ops is not None:
        ops.mul += x.size
    return c * x


def _add(x, y, ops, sign=1.0):
    if ops is not None:
        ops.add += x.size
    return x + y if sign > 0 else x - y


def _delay(x):
    """x[n-1] along the last axis with x[-1] = 0 (finite causal signal)."""
    out = np.zeros_like(x)
    out[..., 1:] = x[..., :-1]
    return out


def _check_even(n):
    if n == 0:
        raise EmptySignal("empty signal")
    if n % 2:
        raise OddLength(f"odd length {n}")


# --------------------------------------------------------------------------- one level
def direct_analysis(x, ops: OpCounter | None = None):
    """Fig. 2 / Eqs. (1)-(4): y_i[n] = b_i[0] x[n] + b_i[1] x[n-1] for every n, then keep n = 2k+1.

    Along the last axis.  Returns (approx d0, detail d1), each N/2 long.
    """
    x = np.asarray(x, dtype=np.float64)
    _check_even(x.shape[-1])
    fb = filter_bank()
    xd = _delay(x)
    b0, b1 = fb["b0"], fb["b1"]
    y0 = _add(_mul(b0[0], x, ops), _mul(b0[1], xd, ops), ops)   # full-rate LPF output
    y1 = _add(_mul(b1[0], x, ops), _mul(b1[1], xd, ops), ops)   # full-rate HPF output
    return y0[..., 1::2].copy(), y1[..., 1::2].copy()            # ↓2, phase n = 2k+1


def direct_synthesis(approx, detail, ops: OpCounter | None = None):
    """Fig. 5 / Eq. (13): D_R = A0(Z) D0(Z^2) + A1(Z) D1(Z^2), i.e. ↑2 (zero insertion),
    full-rate convolution with a0 / a1, sum.  Along the last axis; returns 2L samples."""
    a = np.asarray(approx, dtype=np.float64)
    d = np.asarray(detail, dtype=np.float64)
    if a.shape != d.shape:
        raise LengthMismatch(f"band shapes differ: {a.shape} vs {d.shape}")
    if a.shape[-1] == 0:
        raise EmptySignal("empty bands")
    fb = filter_bank()
    shape = a.shape[:-1] + (2 * a.shape[-1],)
    u0 = np.zeros(shape)
    u1 = np.zeros(shape)
    u0[..., 0::2] = a          # ↑2: subband sample k placed at time 2k
    u1[..., 0::2] = d
    a0, a1 = fb["a0"], fb["a1"]
    r0 = _add(_mul(a0[0], u0, ops), _mul(a0[1], _delay(u0), ops), ops)
    r1 = _add(_mul(a1[0], u1, ops), _mul(a1[1], _delay(u1), ops), ops)
    return _add(r0, r1, ops)


def split_polyphase(x):
    """Eq. (7), M = 2: even[k] = x[2k], odd[k] = x[2k+1]."""
    x = np.asarray(x)
    if x.shape[-1] % 2:
        raise OddLength(f"odd length {x.shape[-1]}")
    return x[..., 0::2].copy(), x[..., 1::2].copy()


def merge_polyphase(even, odd):
    """Interleave, inverse of split_polyphase."""
    even, odd = np.asarray(even), np.asarray(odd)
    if even.shape != odd.shape:
        raise LengthMismatch(f"{even.shape} vs {odd.shape}")
    out = np.empty(even.shape[:-1] + (2 * even.shape[-1],), dtype=np.result_type(even, odd))
    out[..., 0::2] = even
    out[..., 1::2] = odd
    return out


def fast_analysis(x, ops: OpCounter | None = None):
    """Fig. 4: ↓2 first (polyphase split), then one butterfly × b00 = 1/√2.
    Detail sign per §II taps (reading R2 = A2): d1 = b00 (x_e - x_o)."""
    x = np.asarray(x, dtype=np.float64)
    _check_even(x.shape[-1])
    even, odd = split_polyphase(x)
    b00 = filter_bank()["b00"]
    return _mul(b00, _add(even, odd, ops), ops), _mul(b00, _add(even, odd, ops, -1), ops)


def fast_synthesis(approx, detail, ops: OpCounter | None = None):
    """Fig. 7, Eq. (19) with A00 = A01 = a00 = 1/√2 and ↑2 moved to the output:
    even = a00 (d0 + d1), odd = a00 (d0 - d1), then merge (reading R4 = A4)."""
    a = np.asarray(approx, dtype=np.float64)
    d = np.asarray(detail, dtype=np.float64)
    if a.shape != d.shape:
        raise LengthMismatch(f"band shapes differ: {a.shape} vs {d.shape}")
    if a.shape[-1] == 0:
        raise EmptySignal("empty bands")
    a00 = filter_bank()["b00"]
    return merge_polyphase(_mul(a00, _add(a, d, ops), ops), _mul(a00, _add(a, d, ops, -1), ops))


_ANALYSIS = {"direct": direct_analysis, "fast": fast_analysis}
_SYNTHESIS = {"direct": direct_synthesis, "fast": fast_synthesis}


# --------------------------------------------------------------------------- validation
def check_levels_1d(n: int, levels: int):
    if levels < 1:
        raise InvalidLevels(f"levels={levels} < 1")
    if n == 0:
        raise EmptySignal("empty signal")
    if n % (1 << levels):
        raise InsufficientLength(f"n={n} not divisible by 2^{levels}")


def check_levels_2d(h: int, w: int, levels: int):
    if levels < 1:
        raise InvalidLevels(f"levels={levels} < 1")
    if h == 0 or w == 0:
        raise EmptySignal("empty image")
    if h % 2 or w % 2:
        raise OddLength(f"odd dimension {h}x{w}")
    if h % (1 << levels) or w % (1 << levels):
        raise InsufficientLength(f"{h}x{w} not divisible by 2^{levels}")


# --------------------------------------------------------------------------- 1-D multilevel
def decompose_1d(x, levels: int, mode: str = "direct", ops: OpCounter | None = None):
    """Mallat recursion: analyse the approximation band `levels` times.
    Flat layout along the last axis: [a_J | d_J | d_{J-1} | ... | d_1], d_j at [n/2^j, n/2^(j-1))."""
    x = np.asarray(x, dtype=np.float64)
    n = x.shape[-1]
    check_levels_1d(n, levels)
    out = np.empty_like(x)
    a = x
    for j in range(1, levels + 1):
        a, d = _ANALYSIS[mode](a, ops)
        out[..., n >> j:n >> (j - 1)] = d
    out[..., :n >> levels] = a
    return out


def reconstruct_1d(c, levels: int, mode: str = "direct", ops: OpCounter | None = None):
    """Inverse of decompose_1d, coarsest level first."""
    c = np.asarray(c, dtype=np.float64)
    n = c.shape[-1]
    check_levels_1d(n, levels)
    a = c[..., :n >> levels]
    for j in range(levels, 0, -1):
        a = _SYNTHESIS[mode](a, c[..., n >> j:n >> (j - 1)], ops)
    return a


# --------------------------------------------------------------------------- 2-D
def _along(fn, axis, *arrays, ops=None):
    moved = [np.moveaxis(np.asarray(a, dtype=np.float64), axis, -1) for a in arrays]
    res = fn(*moved, ops)
    if isinstance(res, tuple):
        return tuple(np.moveaxis(r, -1, axis) for r in res)
    return np.moveaxis(res, -1, axis)


def analyze2d_level(x, mode: str = "direct", ops: OpCounter | None = None):
    """One separable level: 1-D analysis along every row -> (L, H), then along
    every column of L -> (LL, LH) and of H -> (HL, HH).  Returns (LL, HL, LH, HH)."""
    x = np.asarray(x, dtype=np.float64)
    fn = _ANALYSIS[mode]
    lo, hi = _along(fn, -1, x, ops=ops)
    ll, lh = _along(fn, -2, lo, ops=ops)
    hl, hh = _along(fn, -2, hi, ops=ops)
    return ll, hl, lh, hh


def synthesize2d_level(ll, hl, lh, hh, mode: str = "direct", ops: OpCounter | None = None):
    """Inverse of analyze2d_level: columns first (LL+LH -> L, HL+HH -> H), then rows."""
    shapes = {np.shape(b) for b in (ll, hl, lh, hh)}
    if len(shapes) != 1:
        raise DimensionMismatch(f"subband shapes differ: {shapes}")
    fn = _SYNTHESIS[mode]
    lo = _along(fn, -2, ll, lh, ops=ops)
    hi = _along(fn, -2, hl, hh, ops=ops)
    return _along(fn, -1, lo, hi, ops=ops)


def analyze_2d(x, levels: int, mode: str = "direct", ops: OpCounter | None = None):
    """Multi-level 2-D (Mallat) pyramid over the last two axes.  At level j the region
    [0, h/2^(j-1)) x [0, w/2^(j-1)) holds [[LL_j, HL_j], [LH_j, HH_j]]; recursion on LL."""
    x = np.asarray(x, dtype=np.float64)
    h, w = x.shape[-2], x.shape[-1]
    check_levels_2d(h, w, levels)
    out = np.empty_like(x)
    cur = x
    for j in range(1, levels + 1):
        hh_, ww_ = h >> j, w >> j
        ll, hl, lh, hh = analyze2d_level(cur, mode, ops)
        out[..., :hh_, ww_:2 * ww_] = hl
        out[..., hh_:2 * hh_, :ww_] = lh
        out[..., hh_:2 * hh_, ww_:2 * ww_] = hh
        cur = ll
    out[..., :h >> levels, :w >> levels] = cur
    return out


def synthesize_2d(c, levels: int, mode: str = "direct", ops: OpCounter | None = None):
    """Inverse of analyze_2d, coarsest level first."""
    c = np.asarray(c, dtype=np.float64)
    h, w = c.shape[-2], c.shape[-1]
    check_levels_2d(h, w, levels)
    ll = c[..., :h >> levels, :w >> levels]
    for j in range(levels, 0, -1):
        hh_, ww_ = h >> j, w >> j
        ll = synthesize2d_level(ll, c[..., :hh_, ww_:2 * ww_], c[..., hh_:2 * hh_, :ww_],
                                c[..., hh_:2 * hh_, ww_:2 * ww_], mode, ops)
    return ll


# --------------------------------------------------------------------------- metrics (f3, f4)
def pointwise_error_db(candidate, reference, floor_db: float = -300.0):
    """20 log10(|c - o| / peak), peak = max|o| (1 if o is all zero), floored.
    Quantifies PAPER.md:186 ("-90dB") and :192 ("-160dB to -220dB")."""
    c = np.asarray(candidate, dtype=np.float64)
    o = np.asarray(reference, dtype=np.float64)
    if c.shape != o.shape:
        raise LengthMismatch(f"{c.shape} vs {o.shape}")
    peak = float(np.max(np.abs(o))) if o.size else 0.0
    if peak == 0.0:
        peak = 1.0
    diff = np.abs(c - o)
    with np.errstate(divide="ignore"):
        db = np.where(diff > 0, 20.0 * np.log10(np.where(diff > 0, diff, 1.0) / peak), floor_db)
    return np.maximum(db, floor_db)
