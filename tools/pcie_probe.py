"""PCIe ceiling on the GPU box: pinned 4 GiB H2D alone, D2H alone, and both at once on two streams
(CUDA events), next to the library's host round trip (fhwt_roundtrip_2d_host) on the c4 shape.
python tools/pcie_probe.py"""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402


def timed(fn, reps=3):
    best = None
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1)
        best = t if best is None else min(best, t)
    return best


def main():
    n = 256 * 2048 * 2048
    hin = torch.rand(n).pin_memory()
    hout = torch.empty(n).pin_memory()
    d0 = torch.empty(n, device="cuda")
    d1 = torch.rand(n, device="cuda")
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    nb = 4 * n

    def h2d():
        d0.copy_(hin, non_blocking=True)

    def d2h():
        hout.copy_(d1, non_blocking=True)

    def both():
        cur = torch.cuda.current_stream()
        s1.wait_stream(cur)
        s2.wait_stream(cur)
        with torch.cuda.stream(s1):
            d0.copy_(hin, non_blocking=True)
        with torch.cuda.stream(s2):
            hout.copy_(d1, non_blocking=True)
        cur.wait_stream(s1)
        cur.wait_stream(s2)

    for name, fn, by in (("h2d", h2d, nb), ("d2h", d2h, nb), ("duplex", both, 2 * nb)):
        ms = timed(fn)
        print(json.dumps({"copy": name, "ms": round(ms, 2), "gbs": round(by / ms / 1e6, 2)}), flush=True)
    import paper_1002_2184_b200 as fhwt
    host = hin.view(256, 2048, 2048)
    out = hout.view(256, 2048, 2048)
    fhwt.roundtrip_2d_host(host, 5, out=out)
    import time
    for _ in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        fhwt.roundtrip_2d_host(host, 5, out=out)
        t = time.perf_counter() - t0
        print(json.dumps({"roundtrip_ms": round(t * 1e3, 2), "per_direction_gbs": round(nb / t / 1e9, 2)}), flush=True)


if __name__ == "__main__":
    main()
