"""Host-buffer round trip (fhwt_roundtrip_2d_host) on the c4 workload: chunk size x stream count."""
import json
import os
os.environ.setdefault("FHWT_TUNING", "1")   # the library honours FHWT_* knobs only behind this gate
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1002_2184_b200 as fhwt  # noqa: E402


def main():
    host = torch.rand(256, 2048, 2048).pin_memory()
    out = torch.empty_like(host).pin_memory()
    fhwt.roundtrip_2d_host(host, 5, out=out)
    for mb, ns in ((256, 2), (64, 2), (64, 3), (32, 3), (128, 3), (64, 4)):
        os.environ.update(FHWT_RT_CHUNK_MB=str(mb), FHWT_RT_STREAMS=str(ns))
        ts = []
        for _ in range(4):
            t0 = time.perf_counter()
            fhwt.roundtrip_2d_host(host, 5, out=out)
            ts.append(time.perf_counter() - t0)
        t = statistics.median(ts)
        print(json.dumps({"chunk_mb": mb, "streams": ns, "ms": round(t * 1e3, 2), "gbs": round(16 * host.numel() / t / 1e9, 1)}),
              flush=True)
    print("rt err", float((out - host).abs().max()))


if __name__ == "__main__":
    main()
