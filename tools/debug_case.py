"""Run one transform case in isolation (for localising device faults): python tools/debug_case.py 2d|1d ana|syn h w batch L"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402

kind, op = sys.argv[1], sys.argv[2]
args = [int(a) for a in sys.argv[3:]]
if kind == "2d":
    h, w, b, L = args
    x = torch.rand(b, h, w, device="cuda")
    y = fhwt.analyze_2d(x, L) if op == "ana" else fhwt.synthesize_2d(x, L)
else:
    n, b, L = args
    x = torch.rand(b, n, device="cuda")
    y = fhwt.analyze_1d(x, L) if op == "ana" else fhwt.synthesize_1d(x, L)
torch.cuda.synchronize()
print("ok", kind, op, args)
