"""Throughput of shapes that do not take the compile-time fast path (ragged tiles, odd levels)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    shapes = ((64, 1080, 1920, 3), (32, 2160, 3840, 4), (256, 2048, 2048, 3), (256, 2048, 2048, 7),
              (16, 4096, 4096, 8), (1024, 512, 768, 6))
    if os.environ.get("SMALL"):
        shapes = ((65536, 32, 32, 5), (16384, 64, 64, 6), (16384, 64, 64, 3), (4096, 128, 128, 7), (4096, 128, 128, 5),
                  (1024, 256, 256, 8), (65536, 16, 64, 4))
    if os.environ.get("RAGGED"):
        shapes = ((256, 1000, 1000, 3), (128, 720, 1280, 4), (512, 600, 800, 3), (64, 1200, 1600, 4), (32, 3000, 4000, 3))
    if os.environ.get("SHAPES"):   # "b,h,w,L;b,h,w,L;..."
        shapes = tuple(tuple(int(v) for v in t.split(",")) for t in os.environ["SHAPES"].split(";"))
    for (b, h, w, L) in shapes:
        x = torch.rand(b, h, w, device="cuda")
        plan = fhwt.Plan2d(h, w, b, L)
        c = plan.analyze(x)
        r = plan.synthesize(c)
        e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
        for _ in range(3):
            plan.analyze(x, out=c)
            plan.synthesize(c, out=r)
        torch.cuda.synchronize()
        e[0].record()
        for _ in range(10):
            plan.analyze(x, out=c)
        e[1].record()
        for _ in range(10):
            plan.synthesize(c, out=r)
        e[2].record()
        torch.cuda.synchronize()
        S = x.numel()
        ta, ts = e[0].elapsed_time(e[1]) / 10, e[1].elapsed_time(e[2]) / 10
        print(f"{b}x{h}x{w} L={L}: analysis {8 * S / ta / 1e6:.0f} GB/s, synthesis {8 * S / ts / 1e6:.0f} GB/s, "
              f"rt err {float((r - x).abs().max()):.2e}", flush=True)
        del x, c, r


if __name__ == "__main__":
    main()
