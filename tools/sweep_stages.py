"""Stage-count x levels sweep of both 2-D kernels on c4-shaped data (256 x 2048^2)."""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402
from tools.sweep_ctas import timeit  # noqa: E402


def main():
    x = torch.rand(256, 2048, 2048, device="cuda")
    c = torch.empty_like(x)
    r = torch.empty_like(x)
    S = x.numel()
    levels = [int(a) for a in sys.argv[1:]] or [1, 2, 3, 4, 5]
    for L in levels:
        p = fhwt.Plan2d(2048, 2048, 256, L)
        row = {"L": L}
        for st in (2, 3, 4):
            os.environ["FHWT_ANA_STAGES"] = str(st)
            os.environ["FHWT_SYN_STAGES"] = str(st)
            try:
                ta = timeit(lambda: p.analyze(x, out=c))
                ts = timeit(lambda: p.synthesize(c, out=r))
                err = float((r - x).abs().max())
                row[f"st{st}"] = [round(8 * S / ta / 1e6), round(8 * S / ts / 1e6), err]
            except Exception as ex:  # noqa: BLE001
                row[f"st{st}"] = str(ex)[:80]
        print(json.dumps(row), flush=True)


if __name__ == "__main__":
    main()
