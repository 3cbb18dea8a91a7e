"""Lowpass (f1) timing on the c4 uint8 batch."""
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():

    d = torch.from_numpy(datagen.generate("c4u8")).cuda()
    for blocks, L in [(0, L) for L in (1, 2, 3, 4, 5, 8)]:
        os.environ["FHWT_LP_BLOCKS"] = str(blocks)
        out = torch.empty((256, 2048 >> L, 2048 >> L), device="cuda")
        for _ in range(3):
            fhwt.lowpass_2d_u8(d, L, out=out)
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            fhwt.lowpass_2d_u8(d, L, out=out)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        S = d.numel()
        print("blocks", blocks or "exact", "L", L, f"{ms:.4f} ms", f"{(S + 4 * S / 4 ** L) / ms / 1e6:.0f} GB/s")
    x = torch.empty(S // 4, dtype=torch.float32, device="cuda")
    for _ in range(3):
        x.sum()
    torch.cuda.synchronize()
    e0.record()
    for _ in range(10):
        x.sum()
    e1.record()
    torch.cuda.synchronize()
    print("torch sum of 1 GiB (read-only reference):", f"{S / (e0.elapsed_time(e1) / 10) / 1e6:.0f} GB/s")


if __name__ == "__main__":
    main()
