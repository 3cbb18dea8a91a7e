"""Width dependence of the TMA row-box stream (tools/membench.cu k_tile_tma, one-row 1-KB boxes,
global tile order, band-scatter stores): 1 Gi samples as 256 x 2048^2, 16 x 8192^2, 1 x 32768^2.
python tools/membench_widths.py"""
import ctypes
import json
import os
import subprocess

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "membench.so")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(HERE, "membench.cu")):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", os.path.join(HERE, "membench.cu"), "-o", so])
L = ctypes.CDLL(so)
L.mb_tile_tma.restype = ctypes.c_float
x = torch.rand(1 << 30, device="cuda")
y = torch.empty_like(x)
vp, i64 = ctypes.c_void_p, ctypes.c_int64
for rep in range(2):
    for B, H, W in ((256, 2048, 2048), (16, 8192, 8192), (1, 32768, 32768), (64, 2048, 8192), (4, 2048, 131072)):
        for stages in (2, 3):
            ms = L.mb_tile_tma(vp(x.data_ptr()), vp(y.data_ptr()), i64(H), i64(W), i64(B), 296, stages, 10, 256, 1, 0,
                               1, 1)
            print(json.dumps({"shape": [B, H, W], "stages": stages, "gbs": round(8 * x.numel() / ms / 1e6, 1)}),
                  flush=True)
