"""Pins of the fp64 oracle (oracle/) against things that are not the oracle itself.

Each test names the passage that fixes the expected value:
* printed worked examples (SPEC.md, tests/golden/spec_examples.json),
* hand-computed values (tests/golden/hand_computed.json),
* an explicit closed-form Haar basis (oracle/closed_form.py, independent formula),
* library routines (torch avg_pool1d/avg_pool2d: LL_L = 2^L * block mean),
* invariants of an orthonormal PR filter bank ("perfect reconstruction").
A plausible slip (dropped term, swapped sign, transposed operand, wrong decimation phase,
factor-2 gain) fails at least one of them.
"""
import json
import math
import os

import numpy as np
import pytest

import oracle as o
from oracle.closed_form import closed_form_1d, closed_form_2d, haar_matrix_1d

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _ev(s):
    return float(eval(str(s), {"__builtins__": {}}, {"sqrt": math.sqrt}))


def _load(name):
    with open(os.path.join(GOLD, name)) as f:
        return json.load(f)


# ------------------------------------------------------------------ SPEC worked examples
def test_spec_analysis_examples():
    g = _load("spec_examples.json")
    for case in g["analysis_1d"]:
        for mode in ("direct", "fast"):
            fn = o.direct_analysis if mode == "direct" else o.fast_analysis
            a, d = fn(case["x"])
            np.testing.assert_allclose(a, [_ev(v) for v in case["approx"]], atol=1e-12, err_msg=case["cite"])
            np.testing.assert_allclose(d, [_ev(v) for v in case["detail"]], atol=1e-12, err_msg=case["cite"])


def test_spec_synthesis_examples():
    g = _load("spec_examples.json")
    for case in g["synthesis_1d"]:
        for fn in (o.direct_synthesis, o.fast_synthesis):
            r = fn([_ev(v) for v in case["approx"]], [_ev(v) for v in case["detail"]])
            np.testing.assert_allclose(r, case["x"], atol=1e-12, err_msg=case["cite"])


def test_spec_decompose_example():
    g = _load("spec_examples.json")
    for case in g["decompose_1d"]:
        c = o.decompose_1d(case["x"], case["levels"])
        np.testing.assert_allclose(c, [_ev(v) for v in case["mallat"]], atol=1e-12)
        np.testing.assert_allclose(o.reconstruct_1d(c, case["levels"]), case["x"], atol=1e-12)


def test_spec_2d_examples():
    g = _load("spec_examples.json")
    cst = g["analysis_2d_constant"]
    x = np.full((cst["size"], cst["size"]), float(cst["value"]))
    c = o.analyze_2d(x, 1)
    h = cst["size"] // 2
    np.testing.assert_allclose(c[:h, :h], cst["LL"], atol=1e-12)
    assert np.all(c[:h, h:] == 0) and np.all(c[h:, :] == 0)      # exactly zero details
    np.testing.assert_allclose(o.synthesize_2d(c, 1), x, atol=1e-12)
    q = g["analysis_2d_2x2"]
    c = o.analyze_2d(np.array(q["x"], dtype=float), 1)
    assert c[0, 0] == pytest.approx(_ev(q["LL"]), abs=1e-12)
    assert c[1, 1] == pytest.approx(_ev(q["HH"]), abs=1e-12)
    ll = g["synthesis_2d_ll_only"]
    coeffs = np.array([[2 * ll["c"], 0.0], [0.0, 0.0]])
    np.testing.assert_allclose(o.synthesize_2d(coeffs, 1), np.full((2, 2), ll["c"]), atol=1e-12)


def test_spec_error_db_example():
    g = _load("spec_examples.json")["error_db"]
    db = o.pointwise_error_db(g["candidate"], g["oracle"])
    np.testing.assert_allclose(db, g["db"], atol=1e-6)
    assert np.all(o.pointwise_error_db([0.5, 2.0], [0.5, 2.0]) == -300.0)


def test_spec_op_counts():
    """direct 4N mul + 2N add, fast N mul + N add per level; ratio 1/4."""
    for case in _load("spec_examples.json")["op_counts"]:
        ops = o.OpCounter()
        o.decompose_1d(np.arange(case["n"], dtype=float), case["levels"], case["mode"], ops)
        assert ops.mul == case["mul"], case["cite"]
        if "add" in case:
            assert ops.add == case["add"], case["cite"]
    for n in (2, 8, 64, 1024):
        for lv in (1, 2, 3):
            if n % (1 << lv):
                continue
            od, of = o.OpCounter(), o.OpCounter()
            x = np.arange(n, dtype=float)
            o.decompose_1d(x, lv, "direct", od)
            o.decompose_1d(x, lv, "fast", of)
            assert of.mul * 4 == od.mul                      # "less than quarter", read as <= 1/4
            assert (of.mul + of.add) * 3 == od.mul + od.add  # total-op ratio 1/3


# ------------------------------------------------------------------ hand-computed fixtures
def test_hand_computed_1d():
    g = _load("hand_computed.json")
    s = g["signal_1_to_8"]
    for j in (1, 2, 3):
        c = o.decompose_1d(s["x"], j)
        np.testing.assert_allclose(c, [_ev(v) for v in s[f"J{j}"]], atol=1e-12)
    c3 = o.decompose_1d(s["x"], 3)
    assert np.sum(c3 ** 2) == pytest.approx(s["energy"], rel=1e-13)
    assert c3[0] ** 2 == pytest.approx(162) and c3[1] ** 2 == pytest.approx(32)
    t = g["signal_3_1"]
    np.testing.assert_allclose(o.decompose_1d(t["x"], 1), [_ev(v) for v in t["J1"]], atol=1e-12)


def test_hand_computed_2d():
    g = _load("hand_computed.json")["image_4x4"]
    x = np.array(g["x"], dtype=float)
    np.testing.assert_allclose(o.analyze_2d(x, 1), g["L1"], atol=1e-12)
    np.testing.assert_allclose(o.analyze_2d(x, 2), g["L2"], atol=1e-12)
    assert np.sum(o.analyze_2d(x, 2) ** 2) == pytest.approx(g["energy"], rel=1e-13)


# ------------------------------------------------------------------ closed-form basis
@pytest.mark.parametrize("n", [2, 4, 8, 16, 64, 256])
def test_closed_form_1d_all_levels(n):
    rng = np.random.default_rng(n)
    x = rng.standard_normal((3, n))
    for j in range(1, int(math.log2(n)) + 1):
        np.testing.assert_allclose(o.decompose_1d(x, j, "direct"), closed_form_1d(x, j), atol=1e-12)
        np.testing.assert_allclose(o.decompose_1d(x, j, "fast"), closed_form_1d(x, j), atol=1e-12)


def test_closed_form_basis_is_orthonormal():
    for n, j in [(8, 3), (64, 4), (256, 8)]:
        m = haar_matrix_1d(n, j)
        np.testing.assert_allclose(m @ m.T, np.eye(n), atol=1e-12)


@pytest.mark.parametrize("h,w", [(2, 2), (4, 4), (8, 32), (16, 64), (64, 16), (64, 64)])
def test_closed_form_2d_all_levels(h, w):
    rng = np.random.default_rng(h * 1000 + w)
    x = rng.standard_normal((2, h, w))
    for lv in range(1, int(math.log2(min(h, w))) + 1):
        np.testing.assert_allclose(o.analyze_2d(x, lv), closed_form_2d(x, lv), atol=1e-12)
        np.testing.assert_allclose(o.analyze_2d(x, lv, "fast"), closed_form_2d(x, lv), atol=1e-12)


# ------------------------------------------------------------------ library special cases
def test_ll_is_scaled_avg_pool():
    """LL_L = 2^L * avg_pool2d(x, 2^L); approx_J = 2^(J/2) * avg_pool1d(x, 2^J)  (torch, CPU fp64)."""
    import torch
    rng = np.random.default_rng(5)
    x = rng.uniform(0, 1, (3, 64, 128))
    for lv in range(1, 7):
        c = o.analyze_2d(x, lv)
        ref = (2.0 ** lv) * torch.nn.functional.avg_pool2d(torch.from_numpy(x)[:, None], 1 << lv)[:, 0].numpy()
        np.testing.assert_allclose(c[:, :64 >> lv, :128 >> lv], ref, rtol=1e-13, atol=1e-13)
    s = rng.standard_normal((4, 512))
    for j in range(1, 10):
        c = o.decompose_1d(s, j)
        ref = (2.0 ** (j / 2)) * torch.nn.functional.avg_pool1d(torch.from_numpy(s)[:, None], 1 << j)[:, 0].numpy()
        np.testing.assert_allclose(c[:, :512 >> j], ref, rtol=1e-12, atol=1e-12)


def test_single_pair_is_scaled_hadamard():
    """One level on a pair is the 2x2 Hadamard matrix / sqrt(2), with the section II detail sign."""
    h2 = np.array([[1.0, 1.0], [1.0, -1.0]]) / math.sqrt(2.0)
    rng = np.random.default_rng(9)
    for _ in range(10):
        x = rng.standard_normal(2)
        np.testing.assert_allclose(np.concatenate(o.direct_analysis(x)), h2 @ x, atol=1e-15)


# ------------------------------------------------------------------ invariants
def test_perfect_reconstruction_all_combinations():
    """PAPER.md:54 ("perfect reconstruction"); {direct,fast} x {direct,fast}."""
    rng = np.random.default_rng(11)
    for n in (2, 4, 6, 10, 1024, 4096):
        x = rng.standard_normal((5, n))
        for am in (o.direct_analysis, o.fast_analysis):
            for sm in (o.direct_synthesis, o.fast_synthesis):
                np.testing.assert_allclose(sm(*am(x)), x, atol=1e-12 * max(1, np.abs(x).max()))
    x = rng.standard_normal((2, 1 << 12))
    for j in (1, 5, 12):
        for mode in ("direct", "fast"):
            np.testing.assert_allclose(o.reconstruct_1d(o.decompose_1d(x, j, mode), j, mode), x, atol=j * 1e-12 * 4)
    img = rng.uniform(0, 255, (2, 64, 96))
    for lv in (1, 3, 5):
        np.testing.assert_allclose(o.synthesize_2d(o.analyze_2d(img, lv), lv), img, atol=1e-10)


def test_no_aliasing_zero_delay():
    """Aliasing cancelled and zero delay (reading R1): an impulse at every position reconstructs exactly
    in place, including the last sample of a finite block (the paper's even-phase chain loses it)."""
    n = 16
    for p in range(n):
        x = np.zeros(n)
        x[p] = 1.0
        np.testing.assert_allclose(o.reconstruct_1d(o.decompose_1d(x, 4), 4), x, atol=1e-15)


def test_energy_linearity_constant():
    rng = np.random.default_rng(12)
    x, y = rng.standard_normal((2, 4, 512))
    for j in (1, 4, 9):
        cx = o.decompose_1d(x, j)
        np.testing.assert_allclose(np.sum(cx ** 2, -1), np.sum(x ** 2, -1), rtol=1e-12)
        np.testing.assert_allclose(o.decompose_1d(2.5 * x - 0.75 * y, j), 2.5 * cx - 0.75 * o.decompose_1d(y, j),
                                   atol=1e-12 * 8)
    cst = np.full(64, 3.7)
    a, d = o.fast_analysis(cst)
    assert np.all(d == 0.0)
    img = rng.uniform(0, 1, (32, 64))
    c = o.analyze_2d(img, 4)
    assert np.sum(c ** 2) == pytest.approx(np.sum(img ** 2), rel=1e-12)


def test_rank1_separability():
    """analyze2d(outer(u, v)) has LL = outer(approx(u), approx(v)) (every level)."""
    rng = np.random.default_rng(13)
    u, v = rng.standard_normal(32), rng.standard_normal(64)
    for lv in (1, 3, 5):
        c = o.analyze_2d(np.outer(u, v), lv)
        au = o.decompose_1d(u, lv)[:32 >> lv]
        av = o.decompose_1d(v, lv)[:64 >> lv]
        np.testing.assert_allclose(c[:32 >> lv, :64 >> lv], np.outer(au, av), atol=1e-12)
        # full separability: the whole pyramid's level-1 HH is outer(d1(u), d1(v))
        c1 = o.analyze_2d(np.outer(u, v), 1)
        np.testing.assert_allclose(c1[16:, 32:], np.outer(o.direct_analysis(u)[1], o.direct_analysis(v)[1]), atol=1e-12)


def test_shift_covariance():
    """Shifting the input by a multiple of 2^J shifts every band by the corresponding amount."""
    rng = np.random.default_rng(14)
    n, J = 256, 4
    x = rng.standard_normal(n)
    xs = np.roll(x, 16)                 # 16 = 2^J: block-aligned circular shift
    c, cs = o.decompose_1d(x, J), o.decompose_1d(xs, J)
    for j in range(1, J + 1):
        band = slice(n >> j, n >> (j - 1))
        np.testing.assert_allclose(cs[band], np.roll(c[band], 16 >> j), atol=1e-12)
    np.testing.assert_allclose(cs[:n >> J], np.roll(c[:n >> J], 1), atol=1e-12)


def test_row_band_sharding_invariance():
    """2^L-aligned row bands transform independently (no halo)."""
    rng = np.random.default_rng(15)
    h, w, lv, parts = 128, 64, 4, 4
    img = rng.uniform(0, 1, (h, w))
    full = o.analyze_2d(img, lv)
    hb = h // parts
    for r in range(parts):
        band = o.analyze_2d(img[r * hb:(r + 1) * hb], lv)
        for j in range(1, lv + 1):
            bh, gh = hb >> j, h >> j
            bw = w >> j
            rows_g = slice(r * bh, (r + 1) * bh)
            np.testing.assert_allclose(band[:bh, bw:2 * bw], full[rows_g, bw:2 * bw], atol=1e-13)            # HL
            np.testing.assert_allclose(band[bh:2 * bh, :bw], full[gh + r * bh:gh + (r + 1) * bh, :bw], atol=1e-13)  # LH
        np.testing.assert_allclose(band[:hb >> lv, :w >> lv], full[r * (hb >> lv):(r + 1) * (hb >> lv), :w >> lv], atol=1e-13)


# ------------------------------------------------------------------ the paper's own comparison
def test_fast_matches_direct_paper_db():
    """PAPER.md:186 (-90 dB, approximation) and :192 (-160 dB, detail): fast vs direct in fp64."""
    rng = np.random.default_rng(16)
    for _ in range(20):
        x = rng.uniform(-1, 1, 4096)
        ad, dd = o.direct_analysis(x)
        af, df = o.fast_analysis(x)
        assert o.pointwise_error_db(af, ad).max() <= -90.0
        assert o.pointwise_error_db(df, dd).max() <= -160.0
        assert np.abs(af - ad).max() <= 1e-12 * max(1, np.abs(x).max())


# ------------------------------------------------------------------ exactness on integer images
def test_integer_image_exact():
    """integer-valued images give dyadic-rational coefficients; the oracle is within
    1e-12 of the exact int64 closed form."""
    import datagen
    img = datagen.c3_image(64, seed=2184)
    exact = closed_form_2d(img, 3, exact_int=True)
    np.testing.assert_allclose(o.analyze_2d(img, 3), exact, atol=1e-12)
    assert np.array_equal(exact.astype(np.float32).astype(np.float64), exact)   # fp32-representable


# ------------------------------------------------------------------ error paths
def test_error_paths():
    with pytest.raises(o.OddLength):
        o.direct_analysis([1.0, 2.0, 3.0])
    with pytest.raises(o.EmptySignal):
        o.fast_analysis([])
    with pytest.raises(o.LengthMismatch):
        o.direct_synthesis([1.0], [1.0, 2.0])
    with pytest.raises(o.InvalidLevels):
        o.decompose_1d(np.ones(8), 0)
    with pytest.raises(o.InsufficientLength):
        o.decompose_1d(np.ones(12), 3)
    with pytest.raises(o.OddLength):
        o.analyze_2d(np.ones((3, 4)), 1)
    with pytest.raises(o.InsufficientLength):
        o.analyze_2d(np.ones((8, 12)), 3)
    with pytest.raises(o.EmptySignal):
        o.analyze_2d(np.ones((0, 4)), 1)
    with pytest.raises(o.DimensionMismatch):
        o.synthesize2d_level(np.ones((2, 2)), np.ones((2, 2)), np.ones((2, 3)), np.ones((2, 2)))
