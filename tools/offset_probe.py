"""Does the relative placement of the input and output buffers change K1 / K4 throughput?
The c4 analysis (x -> c) and synthesis (c -> r) are timed with c placed at several byte offsets
inside one larger allocation (x and r fixed), interleaved rounds in one process; a torch copy
x -> c at the same offsets is the control.  python tools/offset_probe.py [offsets in KiB ...]"""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402
from tools.sweep_ctas import timeit  # noqa: E402


def main():
    offs = [int(v) for v in sys.argv[1:]] or [0, 4, 64, 512, 1024, 2048, 4096, 32768]
    B, H, W = 256, 2048, 2048
    n = B * H * W
    x = torch.rand(B, H, W, device="cuda")
    r = torch.empty_like(x)
    big = torch.empty(n + max(offs) * 256 + 1024, device="cuda")
    plan = fhwt.Plan2d(H, W, B, 5)
    res = {}
    for rnd in range(int(os.environ.get("ROUNDS", "5"))):
        for o in offs:
            c = big[o * 256: o * 256 + n].view(B, H, W)
            ta = timeit(lambda: plan.analyze(x, out=c))
            ts = timeit(lambda: plan.synthesize(c, out=r))
            tc = timeit(lambda: c.copy_(x))
            for k, t in (("ana", ta), ("syn", ts), ("copy", tc)):
                res.setdefault((o, k), []).append(8 * n / t / 1e6)
    for (o, k), v in sorted(res.items()):
        print(json.dumps({"offset_kib": o, "kernel": k, "median_gbs": round(statistics.median(v)),
                          "min": round(min(v)), "max": round(max(v))}), flush=True)


if __name__ == "__main__":
    main()
