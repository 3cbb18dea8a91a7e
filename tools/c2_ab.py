"""c2 analysis / synthesis GB/s (4096 x 65536, J = 10), CUDA events over 20 launches."""
import torch

import paper_1002_2184_b200 as fhwt

x = torch.rand(4096, 65536, device="cuda")
p = fhwt.Plan1d(65536, 4096, 10)
c = p.analyze(x)
r = p.synthesize(c)
res = []
for rep in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(20):
        p.analyze(x, out=c)
    e[1].record()
    for _ in range(20):
        p.synthesize(c, out=r)
    e[2].record()
    torch.cuda.synchronize()
    S = x.numel()
    res.append(f"{8 * S / (e[0].elapsed_time(e[1]) / 20) / 1e6:.0f}/{8 * S / (e[1].elapsed_time(e[2]) / 20) / 1e6:.0f}")
print(" ".join(res))
