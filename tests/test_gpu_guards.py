"""Out-of-bounds write checks without compute-sanitizer: every output buffer sits inside a larger
allocation whose guard bands (before and after) hold a NaN sentinel pattern, and must be untouched
after the call.  Covers the paths with the most index arithmetic: overlapped last tiles of ragged
widths, odd band offsets, shifted synthesis boxes, the cooperative coarse levels, whole-image and
short-signal chunk kernels (short last chunks), and the LL-only lowpass paths."""
import numpy as np
import pytest

torch = pytest.importorskip("torch")
pytestmark = pytest.mark.gpu

if not torch.cuda.is_available():  # pragma: no cover
    pytest.skip("needs a CUDA device", allow_module_level=True)

import paper_1002_2184_b200 as fhwt  # noqa: E402

GUARD = 4096   # floats on each side (16 KB: a multiple of 16 B keeps the payload aligned)


def guarded(shape, dtype=torch.float32):
    n = int(np.prod(shape))
    buf = torch.full((n + 2 * GUARD,), float("nan"), dtype=dtype, device="cuda")
    return buf, buf[GUARD:GUARD + n].view(shape)


def assert_guards(buf):
    torch.cuda.synchronize()
    head, tail = buf[:GUARD], buf[-GUARD:]
    assert bool(torch.isnan(head).all()) and bool(torch.isnan(tail).all()), "write outside the output buffer"


@pytest.mark.parametrize("b,h,w,levels", [(2, 40, 1000, 3), (3, 32, 800, 3), (1, 48, 1600, 4), (2, 64, 1160, 3),
                                          (1, 256, 1280, 7), (33, 32, 32, 5), (301, 16, 64, 4), (5, 64, 64, 6),
                                          (2, 128, 512, 7), (3, 8, 24, 3), (2, 1000, 1000, 3), (1, 1080, 512, 3),
                                          (1, 360, 256, 3), (2, 64, 1064, 3), (1, 64, 1088, 6)])
def test_2d_outputs_stay_in_bounds(b, h, w, levels):
    x = torch.rand(b, h, w, device="cuda")
    cbuf, c = guarded((b, h, w))
    fhwt.analyze_2d(x, levels, out=c)
    assert_guards(cbuf)
    rbuf, r = guarded((b, h, w))
    fhwt.synthesize_2d(c, levels, out=r)
    assert_guards(rbuf)
    assert float((r - x).abs().max()) <= 1e-5 * float(x.abs().max())


@pytest.mark.parametrize("n,batch,levels", [(256, 77, 8), (96, 55, 5), (12, 333, 2), (1040, 3, 4), (3072, 2, 10),
                                            (1 << 14, 2, 14)])
def test_1d_outputs_stay_in_bounds(n, batch, levels):
    x = torch.rand(batch, n, device="cuda")
    cbuf, c = guarded((batch, n))
    fhwt.analyze_1d(x, levels, out=c)
    assert_guards(cbuf)
    rbuf, r = guarded((batch, n))
    fhwt.synthesize_1d(c, levels, out=r)
    assert_guards(rbuf)
    assert float((r - x).abs().max()) <= 1e-5 * float(x.abs().max())


@pytest.mark.parametrize("h,w,levels", [(512, 512, 2), (512, 512, 5), (512, 512, 7), (72, 1000, 3)])
def test_lowpass_outputs_stay_in_bounds(h, w, levels):
    u8 = torch.randint(0, 256, (3, h, w), dtype=torch.uint8, device="cuda")
    for src, fn in ((u8, fhwt.lowpass_2d_u8), (u8.to(torch.bfloat16), fhwt.lowpass_2d_bf16)):
        buf, ll = guarded((3, h >> levels, w >> levels))
        fn(src, levels, out=ll)
        assert_guards(buf)
