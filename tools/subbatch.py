"""Does the working-set size change streaming efficiency?  c4-shaped analysis / synthesis of 256
images in one call vs k calls of 256/k images (same bytes), interleaved, CUDA events."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    x = torch.rand(256, 2048, 2048, device="cuda")
    c = torch.empty_like(x)
    r = torch.empty_like(x)
    res = {}
    plans = {k: fhwt.Plan2d(2048, 2048, 256 // k, 5) for k in (1, 2, 4, 8)}
    for rnd in range(5):
        for k, pl in plans.items():
            n = 256 // k

            def ana():
                for i in range(k):
                    pl.analyze(x[i * n:(i + 1) * n], out=c[i * n:(i + 1) * n])

            def syn():
                for i in range(k):
                    pl.synthesize(c[i * n:(i + 1) * n], out=r[i * n:(i + 1) * n])

            for fn, name in ((ana, "ana"), (syn, "syn")):
                fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                res.setdefault(f"{name} k={k}", []).append(8 * x.numel() / (e0.elapsed_time(e1) / 10) / 1e6)
    for key, v in res.items():
        print(json.dumps({"case": key, "median_gbs": round(statistics.median(v))}))


if __name__ == "__main__":
    main()
