"""Power-of-two vs other widths at equal bytes: does the band layout's power-of-two stride matter?"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402
from tools.ab_shapes import t  # noqa: E402

buf = [torch.rand(2**30, device="cuda") for _ in range(3)]
for rnd in range(2):
    for (b, h, w, L) in ((256, 2048, 2048, 5), (200, 2304, 2304, 5), (256, 2048, 2304, 5), (256, 2304, 2048, 5),
                         (160, 2560, 2560, 5), (128, 2048, 4096, 5), (64, 4096, 4096, 5), (1, 32768, 32768, 5)):
        n = b * h * w
        if n > 2**30:
            continue
        x, c, r = (q[:n].view(b, h, w) for q in buf)
        p = fhwt.Plan2d(h, w, b, L)
        ta = t(lambda: p.analyze(x, out=c))
        ts = t(lambda: p.synthesize(c, out=r))
        print(rnd, b, h, w, L, round(8 * n / ta / 1e6), round(8 * n / ts / 1e6), flush=True)
