"""GB/s of the short-signal chunk kernels for a few lengths (analysis / synthesis)."""
import torch

import paper_1002_2184_b200 as fhwt

out = []
for (b, n, J) in ((1048576, 256, 8), (262144, 512, 9), (2097152, 128, 7), (4194304, 64, 6), (1048576, 256, 3)):
    x = torch.rand(b, n, device="cuda")
    p = fhwt.Plan1d(n, b, J)
    c = p.analyze(x)
    r = p.synthesize(c)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize()
    e[0].record()
    for _ in range(10):
        p.analyze(x, out=c)
    e[1].record()
    for _ in range(10):
        p.synthesize(c, out=r)
    e[2].record()
    torch.cuda.synchronize()
    S = x.numel()
    out.append(f"{n}J{J}:{8 * S / (e[0].elapsed_time(e[1]) / 10) / 1e6:.0f}/{8 * S / (e[1].elapsed_time(e[2]) / 10) / 1e6:.0f}")
print(" ".join(out))
