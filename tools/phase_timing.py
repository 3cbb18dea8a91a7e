"""Phase breakdown of the fused 2-D analysis tile chain (K1) from the diagnostic build
(-DFHWT_PHASE_TIMING: clock64() marks in haar2d.cu, thread 0 = warp 0 and thread 224 = warp 7):
mean SM cycles per tile of each phase.  Builds paper_1002_2184_b200/libfhwt_phase.so if missing.
python tools/phase_timing.py [images=256] [levels=5]"""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
LIB = os.path.join(ROOT, "paper_1002_2184_b200", "libfhwt_phase.so")
os.environ["FHWT_TUNING"] = "1"
os.environ["FHWT_LIB"] = LIB

NAMES = {0: "wait (stage mbarrier)", 1: "level 1", 2: "barrier 1", 3: "refill issue", 4: "levels 2+3",
         5: "barrier 2", 6: "levels 4+5", 7: "loop top (after the tile)"}


def main():
    if not os.path.exists(LIB):
        from paper_1002_2184_b200 import _build
        _build.build(force=True, out=LIB, defines=["FHWT_PHASE_TIMING"])
    import torch

    import paper_1002_2184_b200 as fhwt
    B = int(sys.argv[1]) if len(sys.argv) > 1 else 256
    L = int(sys.argv[2]) if len(sys.argv) > 2 else 5
    raw = ctypes.CDLL(LIB)
    buf = (ctypes.c_ulonglong * 32)()
    x = torch.rand(B, 2048, 2048, device="cuda")
    c = torch.empty_like(x)
    plan = fhwt.Plan2d(2048, 2048, B, L)
    for variant in os.environ.get("VARIANTS", "1").split(","):
        os.environ["FHWT_ANA_FUSED"] = variant
        for _ in range(3):
            plan.analyze(x, out=c)
        torch.cuda.synchronize()
        raw.fhwt_debug_phases(buf, 1)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(10):
            plan.analyze(x, out=c)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 10
        raw.fhwt_debug_phases(buf, 1)
        out = {"variant": variant, "gbs": 8 * x.numel() / ms / 1e6, "ms": ms}
        for w, name in ((0, "warp0"), (1, "warp7")):
            n = buf[16 * w + 15] or 1
            out[name] = {NAMES[k]: round(buf[16 * w + k] / n, 1) for k in range(8)}
            out[name]["tiles"] = buf[16 * w + 15]
        print(json.dumps(out), flush=True)


if __name__ == "__main__":
    main()
