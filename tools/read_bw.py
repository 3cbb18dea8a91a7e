"""Pure-read HBM bandwidth (the lowpass path reads 1 B/px and writes 1/1024 of that): torch
reductions over 4 GiB, best of 10, CUDA events, next to the lowpass kernel on c4 uint8 images."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def best(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ts = []
    for _ in range(reps):
        e0.record()
        fn()
        e1.record()
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts)


def main():
    a = torch.rand(2**30, device="cuda")
    u8 = torch.randint(0, 256, (256, 2048, 2048), dtype=torch.uint8, device="cuda")
    out = torch.empty((256, 64, 64), device="cuda")
    res = {
        "sum_f32_4GiB_gbs": 4 * 2**30 / best(lambda: a.sum()) / 1e6,
        "amax_u8_1GiB_gbs": 2**30 / best(lambda: u8.amax()) / 1e6,
        "copy_f32_4GiB_gbs": 8 * 2**30 / best(lambda: a.clone()) / 1e6,
        "lowpass_u8_L5_gbs": (u8.numel() * (1 + 4 / 4**5)) / best(lambda: fhwt.lowpass_2d_u8(u8, 5, out=out)) / 1e6,
    }
    print(json.dumps({k: round(v) for k, v in res.items()}))


if __name__ == "__main__":
    main()
