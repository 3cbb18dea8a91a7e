"""Small shapes that exercise every kernel variant once (for compute-sanitizer runs)."""
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402

torch.manual_seed(0)
cases2d = [(64, 512, 2, 5), (64, 256, 1, 3), (96, 320, 2, 5), (256, 512, 1, 8), (16, 24, 1, 3), (6, 10, 1, 1),
           (64, 128, 2, 2),
           # ragged widths (overlapped last tile, odd band offsets, shifted synthesis boxes), 8-row tiles
           (40, 1000, 1, 3), (32, 800, 2, 3), (48, 1600, 1, 4), (64, 1160, 1, 3), (256, 1280, 1, 7),
           # small images (whole-image chunk kernels) incl. a short last chunk
           (32, 32, 33, 5), (16, 64, 301, 4), (64, 64, 5, 6)]
for h, w, b, L in cases2d:
    x = torch.rand(b, h, w, device="cuda")
    r = fhwt.synthesize_2d(fhwt.analyze_2d(x, L), L)
    torch.cuda.synchronize()
    assert float((r - x).abs().max()) < 1e-5, (h, w, b, L)
for n, b, J in [(1024, 3, 10), (1 << 12, 2, 12), (1040, 2, 4), (6, 2, 1), (3072, 1, 10),
                (256, 77, 8), (96, 55, 5), (12, 333, 2)]:   # short signals: chunk kernels
    x = torch.rand(b, n, device="cuda")
    r = fhwt.synthesize_1d(fhwt.analyze_1d(x, J), J)
    torch.cuda.synchronize()
    assert float((r - x).abs().max()) < 1e-5, (n, b, J)
c = fhwt.analyze_2d(torch.rand(2, 64, 64, device="cuda"), 3)
fhwt.pack_ll_2d(c, 3)
u8 = torch.randint(0, 256, (3, 512, 512), dtype=torch.uint8, device="cuda")
for L in (2, 5, 7):
    fhwt.lowpass_2d_u8(u8, L)
    fhwt.lowpass_2d_bf16(u8.to(torch.bfloat16), L)
for knob in ("FHWT_ANA_FUSED=3", "FHWT_SYN_MODE=2", "FHWT_SYN_MODE=0", "FHWT_COOP=0"):
    k, v = knob.split("=")
    os.environ[k] = v
    x = torch.rand(2, 128, 512, device="cuda")
    r = fhwt.synthesize_2d(fhwt.analyze_2d(x, 7), 7)
    torch.cuda.synchronize()
    assert float((r - x).abs().max()) < 1e-5, knob
    del os.environ[k]
torch.cuda.synchronize()
print("sanitize case ok")
