"""Checks that membench's TMA variants produce the same output as the LDG variant."""
import ctypes
import os

import torch

HERE = os.path.dirname(os.path.abspath(__file__))
L = ctypes.CDLL(os.path.join(HERE, "membench.so"))
for f in ("mb_linear", "mb_tile_ldg", "mb_tile_tma"):
    getattr(L, f).restype = ctypes.c_float
B, H, W = 256, 2048, 2048
x = torch.rand(B, H, W, device="cuda")
y0 = torch.zeros_like(x)
vp, i64 = ctypes.c_void_p, ctypes.c_int64
L.mb_tile_ldg(vp(x.data_ptr()), vp(y0.data_ptr()), i64(H), i64(W), i64(B), 592, 1)
for bw, bh, bulk in ((256, 32, 0), (256, 1, 0, 1, 0), (256, 8, 0), (0, 0, 1)):
    y = torch.zeros_like(x)
    ms = L.mb_tile_tma(vp(x.data_ptr()), vp(y.data_ptr()), i64(H), i64(W), i64(B), 296, 3, 10, bw or 256, bh or 32, bulk, 1, 0)
    torch.cuda.synchronize()
    print(bw, bh, bulk, "equal:", torch.equal(y, y0), "GB/s", 8 * x.numel() / ms / 1e6)
