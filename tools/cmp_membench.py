"""Same-process comparison: membench TMA-row + level-1 band-store pattern vs the real analysis kernel
(L=1 and L=5) under stage / L2-hint knobs; 5 interleaved rounds, median GB/s per case."""
import ctypes
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import statistics
import subprocess
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402
from tools.sweep_ctas import timeit  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "membench.so")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(HERE, "membench.cu")):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", os.path.join(HERE, "membench.cu"), "-o", so])
MB = ctypes.CDLL(so)
MB.mb_tile_tma.restype = ctypes.c_float
B, H, W = 256, 2048, 2048
x = torch.rand(B, H, W, device="cuda")
y = torch.empty_like(x)
r = torch.empty_like(x)
n = x.numel()
vp, i64 = ctypes.c_void_p, ctypes.c_int64
plans = {L: fhwt.Plan2d(H, W, B, L) for L in (1, 5)}


def case_membench(st):
    return lambda: MB.mb_tile_tma(vp(x.data_ptr()), vp(y.data_ptr()), i64(H), i64(W), i64(B), 296, st, 10, 256, 1, 0, 1, 0)


def case_ana(L, st, hint):
    def f():
        os.environ.update(FHWT_ANA_STAGES=str(st), FHWT_ANA_L2HINT=str(hint))
        return timeit(lambda: plans[L].analyze(x, out=y))
    return f


def case_syn(L, st):
    def f():
        os.environ.update(FHWT_SYN_STAGES=str(st))
        return timeit(lambda: plans[L].synthesize(y, out=r))
    return f


cases = {"membench tma256x1 st3": case_membench(3), "membench tma256x1 st2": case_membench(2)}
for L in (1, 5):
    for st in (2, 3):
        for hint in (1, 0):
            cases[f"ana L{L} st{st} hint{hint}"] = case_ana(L, st, hint)
    cases[f"syn L{L} st2"] = case_syn(L, 2)
res = {k: [] for k in cases}
for rnd in range(int(os.environ.get("ROUNDS", "5"))):
    for k, f in cases.items():
        res[k].append(8 * n / f() / 1e6)
for k, v in res.items():
    print(json.dumps({"case": k, "median_gbs": round(statistics.median(v)), "min": round(min(v)), "max": round(max(v))}),
          flush=True)
