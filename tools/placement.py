"""Does physical placement matter?  The same L=5 analysis on three different (x, c) buffer pairs
of the same shape, interleaved per call."""
import json
import statistics
import sys
import os

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    n = 128
    pairs = [(torch.rand(n, 2048, 2048, device="cuda"), torch.empty(n, 2048, 2048, device="cuda")) for _ in range(3)]
    plan = fhwt.Plan2d(2048, 2048, n, 5)
    ev = {i: [] for i in range(3)}
    for it in range(40):
        for i, (x, c) in enumerate(pairs):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            plan.analyze(x, out=c)
            e1.record()
            ev[i].append((e0, e1))
    torch.cuda.synchronize()
    for i in range(3):
        ms = [a.elapsed_time(b) for a, b in ev[i][2:]]
        print(json.dumps({"pair": i, "addr_x": hex(pairs[i][0].data_ptr()), "median_ms": round(statistics.median(ms), 4),
                          "gbs": round(8 * n * 2048 * 2048 / statistics.median(ms) / 1e6)}))


if __name__ == "__main__":
    main()
