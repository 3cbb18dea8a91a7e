"""Tile / stage sweep of the fused 2-D kernels (env overrides read by libfhwt at call time).
python tools/sweep_2d.py [c4|c5]"""
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

    kind = sys.argv[1] if len(sys.argv) > 1 else "c4"
    if kind == "c4":
        x = torch.from_numpy(datagen.generate("c4")).cuda()
        plan = fhwt.Plan2d(2048, 2048, 256, 5)
    else:
        x = torch.from_numpy(datagen.generate("c5")).cuda()
        plan = fhwt.Plan2d(32768, 32768, 1, 8)
    c = torch.empty_like(x)
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


    res = []
    for tc, st in itertools.product((256,), (2, 3)):
        if tc == 256 and st > 4:
            continue
        os.environ["FHWT_ANA_TC"], os.environ["FHWT_ANA_STAGES"] = str(tc), str(st)
        os.environ["FHWT_SYN_TC"], os.environ["FHWT_SYN_STAGES"] = str(tc), str(st)
        try:
            ta = timeit(lambda: plan.analyze(x, out=c))
            ts = timeit(lambda: plan.synthesize(c, out=r))
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"tc": tc, "stages": st, "error": str(ex)[:200]}), flush=True)
            continue
        err = float((r - x).abs().max())
        row = {"tc": tc, "stages": st, "ana_ms": ta, "syn_ms": ts, "ana_gbs": 8 * S / ta / 1e6, "syn_gbs": 8 * S / ts / 1e6,
               "rt_err": err}
        res.append(row)
        print(json.dumps(row), flush=True)

    # alternating analysis/synthesis (the bench step), per-kernel events
    for k in ("FHWT_ANA_TC", "FHWT_ANA_STAGES", "FHWT_SYN_TC", "FHWT_SYN_STAGES"):
        os.environ.pop(k, None)
    for rep in range(2):
        evs = [[torch.cuda.Event(enable_timing=True) for _ in range(3)] for _ in range(10)]
        for _ in range(3):
            plan.analyze(x, out=c)
            plan.synthesize(c, out=r)
        torch.cuda.synchronize()
        for e in evs:
            e[0].record()
            plan.analyze(x, out=c)
            e[1].record()
            plan.synthesize(c, out=r)
            e[2].record()
        torch.cuda.synchronize()
        ta = sum(e[0].elapsed_time(e[1]) for e in evs) / 10
        ts = sum(e[1].elapsed_time(e[2]) for e in evs) / 10
        print(json.dumps({"alternating": rep, "ana_ms": ta, "syn_ms": ts, "ana_gbs": 8 * S / ta / 1e6,
                          "syn_gbs": 8 * S / ts / 1e6}), flush=True)


if __name__ == "__main__":
    main()
