"""Same bytes, different 2-D shapes (row stride effects): analysis / synthesis GB/s at L = 5."""
import json
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    L = int(os.environ.get("L", "5"))
    shapes = [(256, 2048, 2048), (1, 32768, 32768), (16, 8192, 8192), (64, 4096, 4096), (1024, 1024, 1024),
              (4, 4096, 65536 // 1), (1, 131072, 8192)]
    x = torch.rand(2**30, device="cuda")
    c = torch.empty_like(x)
    r = torch.empty_like(x)
    res = {}
    for rnd in range(3):
        for (b, h, w) in shapes:
            n = b * h * w
            if n > x.numel():
                continue
            xv, cv, rv = x[:n].view(b, h, w), c[:n].view(b, h, w), r[:n].view(b, h, w)
            pl = fhwt.Plan2d(h, w, b, L)
            ws = torch.empty(max(pl.workspace_bytes, 1), dtype=torch.uint8, device="cuda")
            for name, fn in (("ana", lambda: pl.analyze(xv, out=cv, workspace=ws)),
                             ("syn", lambda: pl.synthesize(cv, out=rv, workspace=ws))):
                fn()
                torch.cuda.synchronize()
                e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
                e0.record()
                for _ in range(10):
                    fn()
                e1.record()
                torch.cuda.synchronize()
                res.setdefault(f"{name} {b}x{h}x{w}", []).append(8 * n / (e0.elapsed_time(e1) / 10) / 1e6)
    for k, v in res.items():
        print(json.dumps({"case": k, "L": L, "median_gbs": round(statistics.median(v))}))


if __name__ == "__main__":
    main()
