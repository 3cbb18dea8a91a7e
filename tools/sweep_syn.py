"""Synthesis variant sweep (same process, same box): TMA level-1 boxes vs LDG level 1, tiles, stages."""
import itertools
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():

    x = torch.from_numpy(datagen.generate("c4")).cuda()
    plan = fhwt.Plan2d(2048, 2048, 256, 5)
    c = plan.analyze(x)
    r = torch.empty_like(x)
    S = x.numel()


    def timeit(fn, reps=10):
        for _ in range(3):
            fn()
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        s.record()
        for _ in range(reps):
            fn()
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e) / reps


    for ldg, tc, st in [(0, 256, 2), (2, 256, 2), (0, 512, 2), (0, 512, 3), (2, 512, 2), (2, 512, 3)]:
        os.environ.update(FHWT_SYN_MODE=str(ldg), FHWT_SYN_TC=str(tc), FHWT_SYN_STAGES=str(st))
        try:
            t = timeit(lambda: plan.synthesize(c, out=r))
            err = float((r - x).abs().max())
            print(json.dumps({"mode": ldg, "tc": tc, "stages": st, "syn_gbs": 8 * S / t / 1e6, "rt_err": err}), flush=True)
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"mode": ldg, "tc": tc, "stages": st, "error": str(ex)[:160]}), flush=True)


if __name__ == "__main__":
    main()
