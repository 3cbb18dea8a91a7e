"""Isolate the 1000 x 1000 slowdown: same bytes, one dimension at a time."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402
from tools.ab_shapes import t  # noqa: E402

buf = [torch.rand(2**28, device="cuda") for _ in range(2)]
for (b, h, w, L) in ((256, 1000, 1000, 3), (256, 1024, 1000, 3), (256, 1000, 1024, 3), (256, 1024, 1024, 3),
                     (256, 1000, 1008, 3), (256, 1008, 1008, 3), (256, 1000, 1000, 1), (256, 1000, 1000, 2)):
    n = b * h * w
    x, c = (q[:n].view(b, h, w) for q in buf)
    p = fhwt.Plan2d(h, w, b, L)
    print(b, h, w, L, round(8 * n / t(lambda: p.analyze(x, out=c)) / 1e6), flush=True)
