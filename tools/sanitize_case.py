"""Small shapes that exercise every kernel variant once (for compute-sanitizer runs)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402

torch.manual_seed(0)
cases2d = [(64, 512, 2, 5), (64, 256, 1, 3), (96, 320, 2, 5), (256, 512, 1, 8), (16, 24, 1, 3), (6, 10, 1, 1),
           (64, 128, 2, 2)]
for h, w, b, L in cases2d:
    x = torch.rand(b, h, w, device="cuda")
    r = fhwt.synthesize_2d(fhwt.analyze_2d(x, L), L)
    torch.cuda.synchronize()
    assert float((r - x).abs().max()) < 1e-5, (h, w, b, L)
for n, b, J in [(1024, 3, 10), (1 << 12, 2, 12), (1040, 2, 4), (6, 2, 1), (3072, 1, 10)]:
    x = torch.rand(b, n, device="cuda")
    r = fhwt.synthesize_1d(fhwt.analyze_1d(x, J), J)
    torch.cuda.synchronize()
    assert float((r - x).abs().max()) < 1e-5, (n, b, J)
c = fhwt.analyze_2d(torch.rand(2, 64, 64, device="cuda"), 3)
fhwt.pack_ll_2d(c, 3)
torch.cuda.synchronize()
print("sanitize case ok")
