"""Analysis / synthesis time of one 2-D plan as CUDA-graph replays (the bench's timing context):
python tools/graph_time.py B H W L [reps]  -> JSON with GB/s of algorithmic bytes per kernel."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    B, H, W, L = (int(a) for a in sys.argv[1:5])
    reps = int(sys.argv[5]) if len(sys.argv) > 5 else 10
    x = torch.rand(B, H, W, device="cuda")
    c = torch.empty_like(x)
    r = torch.empty_like(x)
    plan = fhwt.Plan2d(H, W, B, L)
    ws = torch.empty(max(plan.workspace_bytes, 16), dtype=torch.uint8, device="cuda")
    s = torch.cuda.Stream()
    out = {"shape": [B, H, W], "levels": L}
    for name, fn in (("analysis", lambda: plan.analyze(x, out=c, workspace=ws)),
                     ("synthesis", lambda: plan.synthesize(c, out=r, workspace=ws))):
        with torch.cuda.stream(s):
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=s):
                for _ in range(reps):
                    fn()
            g.replay()
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(s)
            g.replay()
            e1.record(s)
            torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / reps
        out[name + "_ms"] = ms
        out[name + "_gbs"] = 8 * x.numel() / ms / 1e6
    print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
