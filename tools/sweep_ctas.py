"""Persistent-grid size sweep: CTAs per SM x levels, both 2-D kernels, c4-shaped data."""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def timeit(fn, reps=int(os.environ.get("FHWT_TIMEIT_REPS", "10"))):
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


def main():
    x = torch.rand(256, 2048, 2048, device="cuda")
    c = torch.empty_like(x)
    r = torch.empty_like(x)
    S = x.numel()
    for L in (1, 2, 3, 4, 5):
        p = fhwt.Plan2d(2048, 2048, 256, L)
        row = {"L": L}
        for cap in (0, 1, 2, 3, 4):
            os.environ["FHWT_CTAS_PER_SM"] = str(cap)
            ta = timeit(lambda: p.analyze(x, out=c))
            ts = timeit(lambda: p.synthesize(c, out=r))
            row[f"cap{cap}"] = [round(8 * S / ta / 1e6), round(8 * S / ts / 1e6)]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
