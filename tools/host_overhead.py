"""Host-side cost per call (wall µs, GPU work is tiny): Python binding vs the bare C-ABI call, for
the c1 (1 x 1024, J=1) and c3 (512^2, L=3) plans."""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def per_call(fn, n=2000):
    for _ in range(50):
        fn()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(n):
        fn()
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    return round((t1 - t0) / n * 1e6, 2), round((t2 - t0) / n * 1e6, 2)


def main():
    L = fhwt.lib()
    out = {}
    for name, shape, plan in (("c1", (1, 1024), fhwt.Plan1d(1024, 1, 1)), ("c3", (1, 512, 512), fhwt.Plan2d(512, 512, 1, 3))):
        x = torch.rand(shape, device="cuda")
        c = torch.empty_like(x)
        r = torch.empty_like(x)
        s = ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
        xp, cp, rp = (ctypes.c_void_p(t.data_ptr()) for t in (x, c, r))
        ws = ctypes.c_void_p(0)
        out[name] = {
            "py_analyze_us(host,total)": per_call(lambda: plan.analyze(x, out=c)),
            "py_synthesize_us": per_call(lambda: plan.synthesize(c, out=r)),
            "c_analyze_us": per_call(lambda: L.fhwt_plan_analyze(plan._h, xp, cp, ws, s)),
            "c_synthesize_us": per_call(lambda: L.fhwt_plan_synthesize(plan._h, cp, rp, ws, s)),
            "torch_empty_like_us": per_call(lambda: torch.empty_like(x)),
            "current_stream_us": per_call(lambda: torch.cuda.current_stream()),
        }
    print(json.dumps(out, indent=1))


if __name__ == "__main__":
    main()
