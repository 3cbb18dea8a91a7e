"""Sustained vs burst HBM bandwidth: torch copy_ of 4 GiB repeated for ~20 s; per-second GB/s next
to nvidia-smi memory temperature, memory/SM clocks and power."""
import json
import subprocess
import sys
import time

import torch


def smi():
    q = "temperature.gpu,temperature.memory,clocks.mem,clocks.sm,power.draw,clocks_event_reasons.active"
    out = subprocess.run(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits", "-i", "0"],
                         capture_output=True, text=True).stdout.strip()
    return out


def main(seconds=float(sys.argv[1]) if len(sys.argv) > 1 else 20.0):
    a = torch.rand(2**30, device="cuda")
    b = torch.empty_like(a)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_end = time.time() + seconds
    while time.time() < t_end:
        e0.record()
        for _ in range(200):
            b.copy_(a)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / 200
        print(json.dumps({"t": round(seconds - (t_end - time.time()), 1), "copy_gbs": round(8 * 2**30 / ms / 1e6),
                          "smi": smi()}), flush=True)


if __name__ == "__main__":
    main()
