"""Runs tools/membench.cu patterns on 4 GiB (c4-shaped) buffers and prints GB/s (read+write)."""
import ctypes
import json
import os
import subprocess
import sys

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
so = os.path.join(HERE, "membench.so")
if not os.path.exists(so) or os.path.getmtime(so) < os.path.getmtime(os.path.join(HERE, "membench.cu")):
    subprocess.check_call(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-O3", "-shared", "-Xcompiler",
                           "-fPIC", os.path.join(HERE, "membench.cu"), "-o", so])
L = ctypes.CDLL(so)
for f in ("mb_linear", "mb_tile_ldg", "mb_tile_tma"):
    getattr(L, f).restype = ctypes.c_float
B, H, W = 256, 2048, 2048
x = torch.rand(B, H, W, device="cuda")
y = torch.empty_like(x)
n = x.numel()
gb = lambda ms: 8 * n / ms / 1e6  # noqa: E731
vp = ctypes.c_void_p
for blocks, thr in ((148 * 8, 256), (148 * 4, 512), (148 * 16, 128), (148 * 64, 256)):
    ms = L.mb_linear(vp(x.data_ptr()), vp(y.data_ptr()), ctypes.c_int64(n), blocks, thr, 10)
    print(json.dumps({"pattern": "linear float4", "blocks": blocks, "threads": thr, "gbs": gb(ms)}), flush=True)
for blocks in (148 * 2, 148 * 4, 148 * 8):
    ms = L.mb_tile_ldg(vp(x.data_ptr()), vp(y.data_ptr()), ctypes.c_int64(H), ctypes.c_int64(W), ctypes.c_int64(B),
                       blocks, 10)
    print(json.dumps({"pattern": "tile LDG + band scatter", "blocks": blocks, "gbs": gb(ms)}), flush=True)
for blocks, st, bw, bh, bulk in ((148 * 2, 3, 256, 32, 0), (148 * 2, 3, 256, 8, 0), (148 * 2, 3, 128, 32, 0),
                                  (148 * 2, 3, 64, 32, 0), (148 * 2, 3, 256, 1, 0), (148 * 2, 3, 0, 0, 1),
                                  (148 * 3, 2, 256, 8, 0), (148 * 3, 2, 0, 0, 1), (148 * 4, 1, 256, 8, 0)):
    ms = L.mb_tile_tma(vp(x.data_ptr()), vp(y.data_ptr()), ctypes.c_int64(H), ctypes.c_int64(W), ctypes.c_int64(B),
                       blocks, st, 10, bw or 256, bh or 32, bulk, 1, 0)
    print(json.dumps({"pattern": "tile bulk-copy rows" if bulk else f"tile TMA box {bw}x{bh}", "blocks": blocks,
                      "stages": st, "gbs": gb(ms)}), flush=True)
