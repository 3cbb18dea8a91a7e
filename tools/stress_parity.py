"""Extended randomized parity stress (not part of the test suite): N random 1-D / 2-D problems over
every dispatch path (fast / ragged-clamped / masked / generic tiles, small-image and short-signal
chunks, cooperative and two-pass coarse levels, kernel-variant knobs), each against the fp64 oracle
at the north_star tolerance, plus bitwise determinism.  python tools/stress_parity.py [N] [seed]"""
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import oracle as o  # noqa: E402
import paper_1002_2184_b200 as fhwt  # noqa: E402

KNOBS = [{}, {"FHWT_ANA_FUSED": "0"}, {"FHWT_ANA_FUSED": "3"}, {"FHWT_SYN_MODE": "2"}, {"FHWT_SYN_MODE": "0"},
         {"FHWT_COOP": "0"}, {"FHWT_CLAMP_LAST": "0"}, {"FHWT_SMALL_IMAGES": "0"}, {"FHWT_SMALL_SIGNALS": "0"},
         {"FHWT_CLAMP_ROWS": "0"}, {"FHWT_TC256_CLAMP": "0"}, {"FHWT_SYN_SHIFT": "0"}, {"FHWT_1D_TAIL": "0"},
         {"FHWT_ANA_TILE_TABLE": "0", "FHWT_SYN_TILE_TABLE": "0"}, {"FHWT_ANA_FUSED": "6"}, {"FHWT_ANA_FUSED": "1"},
         {"FHWT_SYN_WARP128": "1"}, {"FHWT_SYN_WARP128": "0"},
         {"FHWT_ANA_DYN": "0", "FHWT_SYN_PROD": "0"}, {"FHWT_SYN_PROD": "1"}, {"FHWT_ANA_LEAN": "0"},
         {"FHWT_SYN_DYN": "1", "FHWT_SYN_PROD": "0"}, {"FHWT_SYN_SWZ": "0"}]


def main():
    n = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 7)
    worst, fails = 0.0, []
    for i in range(n):
        knob = KNOBS[rng.integers(len(KNOBS))]
        for k in [k for v in KNOBS for k in v]:
            os.environ.pop(k, None)
        os.environ.update(knob)
        if rng.random() < 0.5:
            L = int(rng.integers(1, 9))
            blk = 1 << L
            h = blk * int(rng.integers(1, max(2, 1100 // blk)))
            w = blk * int(rng.integers(1, max(2, 2100 // blk)))
            while h * w > 1 << 20:
                h = max(blk, h // 2 // blk * blk)
            w = w if w % 4 == 0 or L == 1 else w
            b = int(rng.integers(1, 4))
            if rng.random() < 0.3:   # the c4 / c5 kernels' tiles (32 x 256, LP = 5, swizzled K4 boxes)
                L = int(rng.integers(5, 9))
                h = 32 * int(rng.integers(1, 24)) * (1 << max(0, L - 5))
                w = 256 * int(rng.integers(1, 9)) if rng.random() < 0.7 else max(128, 1 << L) * int(rng.integers(2, 17))
                while h * w > 1 << 20:
                    h = max(1 << L, h // 2 // (1 << L) * (1 << L))
            x = (rng.standard_normal((b, h, w)) * rng.choice([1e-3, 1.0, 1e3])).astype(np.float32)
            xd = torch.from_numpy(x).cuda()
            c = fhwt.analyze_2d(xd, L)
            r = fhwt.synthesize_2d(c, L)
            c2 = fhwt.analyze_2d(xd, L)
            torch.cuda.synchronize()
            ref = o.analyze_2d(x, L)
            scale = np.abs(x).max(axis=(1, 2), keepdims=True)
            e1 = float((np.abs(c.double().cpu().numpy() - ref) / scale).max())
            e2 = float((np.abs(r.double().cpu().numpy() - x) / scale).max())
            det = bool(torch.equal(c, c2))
            case = ("2d", b, h, w, L, knob)
        else:
            J = int(rng.integers(1, 15))
            blk = 1 << J
            nn = blk * int(rng.integers(1, max(2, (1 << 16) // blk)))
            b = int(rng.integers(1, 40))
            if rng.random() < 0.2:   # full decompositions of 2048-8192 samples (levels inside the CTA)
                nn = int(rng.choice([2048, 4096, 8192]))
                J = int(rng.integers(11, nn.bit_length()))
                b = 8 * int(rng.integers(1, 5)) if rng.random() < 0.7 else int(rng.integers(1, 12))
            while nn * b > 1 << 21:
                b = max(1, b // 2)
                if b == 1:
                    break
            x = (rng.standard_normal((b, nn)) * rng.choice([1e-3, 1.0, 1e3])).astype(np.float32)
            xd = torch.from_numpy(x).cuda()
            c = fhwt.analyze_1d(xd, J)
            r = fhwt.synthesize_1d(c, J)
            c2 = fhwt.analyze_1d(xd, J)
            torch.cuda.synchronize()
            ref = o.decompose_1d(x, J)
            scale = np.abs(x).max(axis=1, keepdims=True)
            e1 = float((np.abs(c.double().cpu().numpy() - ref) / scale).max())   # fp64 levels 1-3 for J > 10
            e2 = float((np.abs(r.double().cpu().numpy() - x) / scale).max())
            det = bool(torch.equal(c, c2))
            case = ("1d", b, nn, J, knob)
        worst = max(worst, e1, e2)
        if e1 > 1e-5 or e2 > 1e-5 or not det:
            fails.append((case, e1, e2, det))
            print("FAIL", case, e1, e2, det, flush=True)
    print(f"{n} cases, worst error {worst:.3e} (bar 1e-5), failures {len(fails)}")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
