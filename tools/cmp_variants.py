"""A/B of 2-D kernel variants selected by env knobs, interleaved rounds in one process on c4-shaped
data (256 x 2048^2): median / min / max GB/s per case, plus bitwise equality of every variant's
output with the first variant's.
python tools/cmp_variants.py L 'ANA:FHWT_ANA_WARP=0' 'ANA:FHWT_ANA_WARP=1' 'SYN:FHWT_SYN_MODE=2' ..."""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import statistics
import sys
import threading
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402
from tools.sweep_ctas import timeit  # noqa: E402


_MB = None


def membench(kind, x, y):
    import ctypes
    import subprocess
    global _MB
    if _MB is None:
        here = os.path.dirname(os.path.abspath(__file__))
        so = os.path.join(here, "membench.so")
        if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(here, "membench.cu")):
            subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared",
                                   "-Xcompiler", "-fPIC", os.path.join(here, "membench.cu"), "-o", so])
        _MB = ctypes.CDLL(so)
        _MB.mb_tile_tma.restype = ctypes.c_float
        _MB.mb_tile_ldg.restype = ctypes.c_float
    B, H, W = x.shape
    vp, i64 = ctypes.c_void_p, ctypes.c_int64
    reps = int(os.environ.get("FHWT_TIMEIT_REPS", "10"))
    if kind.startswith("tma"):   # tma[:box rows[:stages]]
        parts = kind.split("/")
        bh = int(parts[1]) if len(parts) > 1 else 1
        st = int(parts[2]) if len(parts) > 2 else 3
        iss = int(parts[3]) if len(parts) > 3 else 1   # warps issuing the one-row boxes
        order = int(parts[4]) if len(parts) > 4 else 0   # 1: global tile order (atomic counter)
        bw = int(parts[5]) if len(parts) > 5 else 256    # box width in floats
        return _MB.mb_tile_tma(vp(x.data_ptr()), vp(y.data_ptr()), i64(H), i64(W), i64(B), 296, st, reps, bw, bh, 0,
                               iss, order)
    return _MB.mb_tile_ldg(vp(x.data_ptr()), vp(y.data_ptr()), i64(H), i64(W), i64(B), 592, reps)


class Nvml:
    """SM clock / power / throttle reasons polled every 5 ms, tagged with the current case."""

    def __init__(self):
        import pynvml as nv
        nv.nvmlInit()
        self.nv, self.h = nv, nv.nvmlDeviceGetHandleByIndex(torch.cuda.current_device())
        self.tag, self.samples, self.stop = None, {}, False
        self.th = threading.Thread(target=self.run, daemon=True)
        self.th.start()

    def run(self):
        nv, h = self.nv, self.h
        while not self.stop:
            if self.tag is not None:
                try:
                    s = (nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM), nv.nvmlDeviceGetPowerUsage(h) / 1e3,
                         nv.nvmlDeviceGetCurrentClocksEventReasons(h))
                    self.samples.setdefault(self.tag, []).append(s)
                except Exception:  # noqa: BLE001
                    pass
            time.sleep(0.005)

    def summary(self, tag):
        s = self.samples.get(tag, [])
        if not s:
            return {}
        reasons = 0
        for x in s:
            reasons |= x[2]
        return {"sm_mhz_med": statistics.median(x[0] for x in s), "sm_mhz_min": min(x[0] for x in s),
                "power_w_med": round(statistics.median(x[1] for x in s)), "reasons": hex(reasons), "n": len(s)}


def main():
    L = int(sys.argv[1])
    cases = sys.argv[2:]
    B = int(os.environ.get("BATCH", "256"))
    H = W = int(os.environ.get("SIZE", "2048"))
    x = torch.rand(B, H, W, device="cuda")
    c = torch.empty_like(x)
    r = torch.empty_like(x)
    plan = fhwt.Plan2d(H, W, B, L)
    ws = torch.empty(max(plan.workspace_bytes, 1), dtype=torch.uint8, device="cuda")
    base_env = {k: v for k, v in os.environ.items()}
    c_ref = plan.analyze(x, workspace=ws)
    r_ref = plan.synthesize(c_ref, workspace=ws)
    res, same = {k: [] for k in cases}, {}
    mon = Nvml()

    def setenv(spec):
        os.environ.clear()
        os.environ.update(base_env)
        for kv in spec.split(":", 1)[1].split(","):
            if "=" in kv:
                k, v = kv.split("=")
                os.environ[k] = v

    for rnd in range(int(os.environ.get("ROUNDS", "5"))):
        k0 = rnd % len(cases)   # rotate the order every round: no case always runs first
        for spec in cases[k0:] + cases[:k0]:
            setenv(spec)
            time.sleep(float(base_env.get("SLEEP", "0")))   # SLEEP > 0: burst (power-cap recovered) timing
            mon.tag = spec
            if spec.startswith("COPY"):
                t = timeit(lambda: c.copy_(x))
                same[spec] = True
            elif spec.startswith("MB"):   # tools/membench.cu pattern: MB:tma | MB:ldg
                t = membench(spec.split(":", 1)[1], x, c)
                same[spec] = None
            elif spec.startswith("ANA"):
                t = timeit(lambda: plan.analyze(x, out=c, workspace=ws))
                if spec not in same:
                    same[spec] = bool(torch.equal(c, c_ref))
            else:
                t = timeit(lambda: plan.synthesize(c_ref, out=r, workspace=ws))
                if spec not in same:
                    same[spec] = bool(torch.equal(r, r_ref))
            res[spec].append(8 * x.numel() / t / 1e6)
            mon.tag = None
    for k, v in res.items():
        print(json.dumps({"L": L, "case": k, "median_gbs": round(statistics.median(v)), "min": round(min(v)),
                          "max": round(max(v)), "bitwise_equal_default": same[k], "clocks": mon.summary(k)}), flush=True)


if __name__ == "__main__":
    main()
