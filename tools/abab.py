"""Interleaved per-call timing of several plans/knob settings (ABAB... order cancels drift):
python tools/abab.py 'L=5' 'L=8' 'L=8,FHWT_COOP=0' ...   (analysis unless SYN=1 in the spec)"""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    B, H, W = (int(v) for v in os.environ.get("SHAPE", "256,2048,2048").split(","))
    x = torch.rand(B, H, W, device="cuda")
    c = torch.empty_like(x)
    r = torch.empty_like(x)
    base = dict(os.environ)
    cases = []
    for spec in sys.argv[1:]:
        kv = dict(t.split("=") for t in spec.split(","))
        L = int(kv.pop("L", "5"))
        syn = kv.pop("SYN", "0") == "1"
        plan = fhwt.Plan2d(H, W, B, L)
        ws = torch.empty(max(plan.workspace_bytes, 1), dtype=torch.uint8, device="cuda")
        cases.append((spec, plan, ws, kv, syn))
    times = {c[0]: [] for c in cases}
    for it in range(int(os.environ.get("ITERS", "30"))):
        for spec, plan, ws, kv, syn in cases:
            os.environ.clear()
            os.environ.update(base)
            os.environ.update(kv)
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            if syn:
                plan.synthesize(c, out=r, workspace=ws)
            else:
                plan.analyze(x, out=c, workspace=ws)
            e1.record()
            times[spec].append(e0)
            times[spec].append(e1)
    torch.cuda.synchronize()
    for spec, ev in times.items():
        ms = [ev[i].elapsed_time(ev[i + 1]) for i in range(2, len(ev), 2)]
        print(json.dumps({"case": spec, "median_ms": round(statistics.median(ms), 4),
                          "gbs": round(8 * x.numel() / statistics.median(ms) / 1e6)}))


if __name__ == "__main__":
    main()
