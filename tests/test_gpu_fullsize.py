"""Full-size GPU parity at BASELINE.json's sizes, in bench.py's launch configuration (plans,
one analysis + one synthesis launch of the whole config).  The oracle checks sampled units one by
one (signals, images, 2^L-aligned 256x256 blocks, which are independent by reading R1); every unit
is checked by properties that hold at any size (round trip, energy of the orthonormal transform).
"""
import numpy as np
import pytest

import datagen
import oracle as o

torch = pytest.importorskip("torch")
pytestmark = [pytest.mark.gpu, pytest.mark.slow]

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1002_2184_b200 as fhwt  # noqa: E402

TOL = 1e-5


def _rel(a, b, scale):
    return float(np.abs(np.asarray(a, np.float64) - np.asarray(b, np.float64)).max()) / scale


def _properties(x, c, r, dims):
    """Round trip and energy, per unit, computed on the GPU in fp64 (no transform arithmetic)."""
    xd = x.double()
    scale = xd.abs().amax(dim=dims)
    rt = (r.double() - xd).abs().amax(dim=dims) / scale
    e_in = (xd * xd).sum(dim=dims)
    e_out = (c.double() ** 2).sum(dim=dims)
    assert float(rt.max()) <= TOL, f"round trip {float(rt.max()):.3e}"
    assert float(((e_out - e_in).abs() / e_in).max()) <= 1e-5   # energy: fp32 outputs, rel 1e-5


def test_c2_full():
    cfg = datagen.CONFIGS["c2"]
    host = datagen.generate("c2")
    x = torch.from_numpy(host).cuda()
    plan = fhwt.Plan1d(cfg["n"], cfg["batch"], cfg["levels"])
    c = plan.analyze(x)
    r = plan.synthesize(c)
    torch.cuda.synchronize()
    _properties(x, c, r, (1,))
    for i in (0, 1, 1234, 2047, 3000, 4095):
        ref = o.decompose_1d(host[i], cfg["levels"])
        assert _rel(c[i].cpu().numpy(), ref, np.abs(host[i]).max()) <= TOL, i


def test_c4_full():
    cfg = datagen.CONFIGS["c4"]
    host = datagen.generate("c4")
    x = torch.from_numpy(host).cuda()
    plan = fhwt.Plan2d(cfg["h"], cfg["w"], cfg["batch"], cfg["levels"])
    c = plan.analyze(x)
    r = plan.synthesize(c)
    torch.cuda.synchronize()
    _properties(x, c, r, (1, 2))
    for i in (0, 77, 255):
        ref = o.analyze_2d(host[i], cfg["levels"])
        assert _rel(c[i].cpu().numpy(), ref, np.abs(host[i]).max()) <= TOL, i


def _block_coeffs(c, r0, c0, b, levels, H, W):
    """Gather the global Mallat coefficients of the b x b input block at (r0, c0) into the block's
    own Mallat layout (the layout definition of oracle/haar.py, written out here)."""
    out = np.zeros((b, b))
    for j in range(1, levels + 1):
        hb, hj, wj, rr, cc = b >> j, H >> j, W >> j, r0 >> j, c0 >> j
        out[:hb, hb:2 * hb] = c[rr:rr + hb, wj + cc:wj + cc + hb].cpu().numpy()
        out[hb:2 * hb, :hb] = c[hj + rr:hj + rr + hb, cc:cc + hb].cpu().numpy()
        out[hb:2 * hb, hb:2 * hb] = c[hj + rr:hj + rr + hb, wj + cc:wj + cc + hb].cpu().numpy()
    hb = b >> levels
    out[:hb, :hb] = c[r0 >> levels:(r0 >> levels) + hb, c0 >> levels:(c0 >> levels) + hb].cpu().numpy()
    return out


def test_c5_full():
    cfg = datagen.CONFIGS["c5"]
    H, W, L = cfg["h"], cfg["w"], cfg["levels"]
    host = datagen.generate("c5")
    x = torch.from_numpy(host).cuda()
    plan = fhwt.Plan2d(H, W, 1, L)
    c = plan.analyze(x)
    r = plan.synthesize(c)
    torch.cuda.synchronize()
    _properties(x[None], c[None], r[None], (1, 2))
    scale = float(np.abs(host).max())
    b = 1 << L
    for (br, bc) in ((0, 0), (17, 93), (127, 127), (64, 1)):
        r0, c0 = br * b, bc * b
        ref = o.analyze_2d(host[r0:r0 + b, c0:c0 + b], L)
        assert _rel(_block_coeffs(c, r0, c0, b, L, H, W), ref, scale) <= TOL, (r0, c0)
