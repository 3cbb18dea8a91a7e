"""Per-launch time series after an idle period: for each variant, sleep, then time N back-to-back
launches individually (CUDA events) with NVML SM clock / power samples, to separate burst from
power-capped behaviour.  python tools/timeseries.py L N 'ANA:FHWT_ANA_WARP=0' ..."""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    import pynvml as nv
    nv.nvmlInit()
    h = nv.nvmlDeviceGetHandleByIndex(0)
    L, N = int(sys.argv[1]), int(sys.argv[2])
    x = torch.rand(256, 2048, 2048, device="cuda")
    c = torch.empty_like(x)
    r = torch.empty_like(x)
    plan = fhwt.Plan2d(2048, 2048, 256, L)
    c0 = plan.analyze(x)
    base = dict(os.environ)
    for spec in sys.argv[3:]:
        os.environ.clear()
        os.environ.update(base)
        for kv in spec.split(":", 1)[1].split(","):
            if "=" in kv:
                k, v = kv.split("=")
                os.environ[k] = v
        fn = (lambda: c.copy_(x)) if spec.startswith("COPY") else \
             (lambda: plan.analyze(x, out=c)) if spec.startswith("ANA") else (lambda: plan.synthesize(c0, out=r))
        fn()
        torch.cuda.synchronize()
        time.sleep(2.0)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(N + 1)]
        ev[0].record()
        for i in range(N):
            fn()
            ev[i + 1].record()
        clk = []
        t_end = time.time() + 0.001
        while not ev[N].query():
            clk.append((nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), round(nv.nvmlDeviceGetPowerUsage(h) / 1e3)))
            time.sleep(0.01)
        torch.cuda.synchronize()
        gbs = [round(8 * x.numel() / ev[i].elapsed_time(ev[i + 1]) / 1e6) for i in range(N)]
        print(json.dumps({"case": spec, "gbs": gbs, "clk": clk[:: max(1, len(clk) // 12)]}), flush=True)


if __name__ == "__main__":
    main()
