"""Practical ceiling for the 2-D access pattern: torch copy_ of the same bytes vs the fused kernels
at L = 1..5 (L=1 is a single strided read+write pass).  python tools/ceiling_2d.py"""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402

x = torch.rand(256, 2048, 2048, device="cuda")
c = torch.empty_like(x)
r = torch.empty_like(x)
S = x.numel()


def timeit(fn, reps=10):
    for _ in range(3):
        fn()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


t = timeit(lambda: c.copy_(x))
print(json.dumps({"op": "torch copy_ 4 GiB fp32", "gbs": 8 * S / t / 1e6}), flush=True)
for st in ("2",):
    os.environ["FHWT_ANA_STAGES"] = os.environ["FHWT_SYN_STAGES"] = st
    for L in (1, 2, 3, 4, 5):
        p = fhwt.Plan2d(2048, 2048, 256, L)
        ta = timeit(lambda: p.analyze(x, out=c))
        ts = timeit(lambda: p.synthesize(c, out=r))
        print(json.dumps({"stages": st, "L": L, "ana_gbs": 8 * S / ta / 1e6, "syn_gbs": 8 * S / ts / 1e6}), flush=True)
