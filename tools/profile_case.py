"""Small driver for ncu captures: one warm-up + one profiled DWT+IDWT of a reduced workload.
python tools/profile_case.py c4 <images> | c2 <signals> | c5 <rows>"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():

    kind, count = sys.argv[1], int(sys.argv[2])
    if kind == "c4":
        x = torch.from_numpy(datagen.generate("c4", count=count)).cuda()
        plan = fhwt.Plan2d(2048, 2048, count, 5)
    elif kind == "c2":
        x = torch.from_numpy(datagen.generate("c2", count=count)).cuda()
        plan = fhwt.Plan1d(65536, count, 10)
    else:
        x = torch.from_numpy(datagen.generate("c5", r0=0, r1=count)).cuda()
        plan = fhwt.Plan2d(count, 32768, 1, 8)
    for _ in range(2):
        c = plan.analyze(x)
        r = plan.synthesize(c)
    torch.cuda.synchronize()
    print("ok", kind, count, float((r - x).abs().max()))


if __name__ == "__main__":
    main()
