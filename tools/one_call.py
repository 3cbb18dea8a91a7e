"""One warm-up + N analysis calls of a c4-shaped plan at level L (for ncu launch timing)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402

L, N = int(sys.argv[1]), int(sys.argv[2]) if len(sys.argv) > 2 else 3
x = torch.rand(256, 2048, 2048, device="cuda")
p = fhwt.Plan2d(2048, 2048, 256, L)
c = p.analyze(x)
for _ in range(N):
    p.analyze(x, out=c)
torch.cuda.synchronize()
