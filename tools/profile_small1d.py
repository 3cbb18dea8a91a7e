import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402
import paper_1002_2184_b200 as fhwt  # noqa: E402
x = torch.rand(1 << 20, 256, device="cuda")
p = fhwt.Plan1d(256, 1 << 20, 8)
c = p.analyze(x); r = p.synthesize(c)
torch.cuda.synchronize()
print("ok", float((r - x).abs().max()))
