"""1-D throughput across signal lengths (multiples and non-multiples of the 1024-sample chunk)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    for (b, n, J) in ((4096, 65536, 10), (4096, 65536, 14), (2730, 98304, 10), (8192, 48000, 7), (5952, 44100 * 2 // 2 * 1, 2),
                      (1, 2**28, 10), (1, 2**28, 20), (65536, 4096, 12), (262144, 1024, 10), (1048576, 256, 8)):
        if n % (1 << J):
            continue
        x = torch.rand(b, n, device="cuda")
        plan = fhwt.Plan1d(n, b, J)
        ws = torch.empty(max(plan.workspace_bytes, 1), dtype=torch.uint8, device="cuda")
        c = plan.analyze(x, workspace=ws)
        r = plan.synthesize(c, workspace=ws)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        torch.cuda.synchronize()
        e[0].record()
        for _ in range(10):
            plan.analyze(x, out=c, workspace=ws)
        e[1].record()
        for _ in range(10):
            plan.synthesize(c, out=r, workspace=ws)
        e[2].record()
        torch.cuda.synchronize()
        S = x.numel()
        ta, ts = e[0].elapsed_time(e[1]) / 10, e[1].elapsed_time(e[2]) / 10
        print(f"{b}x{n} J={J}: analysis {8 * S / ta / 1e6:.0f} GB/s, synthesis {8 * S / ts / 1e6:.0f} GB/s, "
              f"rt err {float((r - x).abs().max()):.2e}", flush=True)
        del x, c, r


if __name__ == "__main__":
    main()
