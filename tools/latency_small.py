"""Latency (µs per DWT+IDWT, CUDA graph replay and eager) of small 2-D problems under env knobs.
python tools/latency_small.py 'FHWT_SMALL_TILES=0' 'FHWT_SMALL_TILES=1'"""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def lat(plan, x, iters=300):
    c, r = torch.empty_like(x), torch.empty_like(x)

    def step():
        plan.analyze(x, out=c)
        plan.synthesize(c, out=r)

    for _ in range(20):
        step()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(iters):
        step()
    e1.record()
    torch.cuda.synchronize()
    eager = e0.elapsed_time(e1) / iters * 1e3
    g = torch.cuda.CUDAGraph()
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        step()
    torch.cuda.current_stream().wait_stream(s)
    with torch.cuda.graph(g):
        step()
    for _ in range(20):
        g.replay()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(iters):
        g.replay()
    e1.record()
    torch.cuda.synchronize()
    return round(eager, 2), round(e0.elapsed_time(e1) / iters * 1e3, 2), float((r - x).abs().max())


def main():
    base = dict(os.environ)
    for spec in sys.argv[1:]:
        os.environ.clear()
        os.environ.update(base)
        for kv in spec.split(","):
            if "=" in kv:
                k, v = kv.split("=")
                os.environ[k] = v
        for (b, h, w, L) in ((1, 512, 512, 3), (1, 1024, 1024, 5), (4, 512, 512, 3), (1, 2048, 2048, 5)):
            x = torch.rand(b, h, w, device="cuda")
            e, gr, err = lat(fhwt.Plan2d(h, w, b, L), x)
            print(json.dumps({"knobs": spec, "shape": [b, h, w], "L": L, "eager_us": e, "graph_us": gr, "rt_err": err}),
                  flush=True)


if __name__ == "__main__":
    main()
