"""Interleaved A/B of env knob settings on several 2-D shapes (median GB/s over rounds, same
process and buffers).  python tools/ab_shapes.py 'FHWT_SYN_RAGGED_FAST=0' 'FHWT_SYN_RAGGED_FAST=1'"""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402

SHAPES = ((256, 1000, 1000, 3), (128, 720, 1280, 4), (512, 600, 800, 3), (64, 1200, 1600, 4), (32, 3000, 4000, 3),
          (64, 1080, 1920, 3), (32, 2160, 3840, 4), (256, 2048, 2048, 5))


def t(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def main():
    specs = sys.argv[1:]
    base = dict(os.environ)
    buf = [torch.rand(2**30, device="cuda") for _ in range(3)]
    for (b, h, w, L) in SHAPES:
        n = b * h * w
        x, c, r = (t_[:n].view(b, h, w) for t_ in buf)
        plan = fhwt.Plan2d(h, w, b, L)
        ws = torch.empty(max(plan.workspace_bytes, 1), dtype=torch.uint8, device="cuda")
        res = {sp: ([], []) for sp in specs}
        for rnd in range(int(os.environ.get("ROUNDS", "4"))):
            for sp in specs:
                os.environ.clear()
                os.environ.update(base)
                os.environ.update(dict(kv.split("=") for kv in sp.split(",") if "=" in kv))
                res[sp][0].append(8 * n / t(lambda: plan.analyze(x, out=c, workspace=ws)) / 1e6)
                res[sp][1].append(8 * n / t(lambda: plan.synthesize(c, out=r, workspace=ws)) / 1e6)
        err = float((r - x).abs().max())
        print(json.dumps({"shape": [b, h, w], "L": L, "rt_err": err,
                          **{sp: [round(statistics.median(a)), round(statistics.median(s_))] for sp, (a, s_) in res.items()}}),
              flush=True)


if __name__ == "__main__":
    main()
