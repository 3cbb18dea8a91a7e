"""c5 strong-scaling projection on one GPU: the per-rank work of a P-way row-band split
(32768/P x 32768, L = 8: analysis, LL pack, synthesis) timed alone for P = 1, 2, 4, 8, and the
efficiency T(1) / (P * T(P)) it implies before any communication (the all-gather of the 64 KiB
coarsest LL runs beside the synthesis pass).  Not a multi-GPU measurement."""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import datagen  # noqa: E402
import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    N, L = 32768, 8
    full = torch.from_numpy(datagen.generate("c5", r0=0, r1=N)).cuda()
    res, t1 = [], None
    for P in (1, 2, 4, 8):
        h = N // P
        x = full[:h]
        c = torch.empty_like(x)
        r = torch.empty_like(x)
        plan = fhwt.Plan2d(h, N, 1, L)
        ws = torch.empty(max(plan.workspace_bytes, 1), dtype=torch.uint8, device="cuda")
        ll = torch.empty((h >> L, N >> L), device="cuda")

        def step():
            plan.analyze(x, out=c, workspace=ws)
            fhwt.pack_ll_2d(c, L, out=ll)
            plan.synthesize(c, out=r, workspace=ws)

        n0 = fhwt.launch_count()
        step()
        launches = fhwt.launch_count() - n0
        for _ in range(3):
            step()
        torch.cuda.synchronize()
        reps = 10 * P
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(reps):
            step()
        e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / reps
        t1 = t1 or t
        ok = bool(torch.equal(r, x)) or float((r - x).abs().max()) <= 1e-5 * float(x.abs().max())
        res.append({"P": P, "band_rows": h, "ms_per_rank_step": round(t, 4),
                    "gbs_per_rank": round(16 * x.numel() / t / 1e6), "projected_efficiency": round(t1 / (P * t), 4),
                    "roundtrip_ok": ok, "launches_per_step": launches,
                    "coop": os.environ.get("FHWT_COOP", "1")})
        print(json.dumps(res[-1]), flush=True)


if __name__ == "__main__":
    main()
