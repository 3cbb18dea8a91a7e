VARIANTS=1,9 python tools/phase_timing.py 256 5 > gpurun_out/phase.jsonl 2> gpurun_out/phase.err; cat gpurun_out/phase.jsonl; tail -3 gpurun_out/phase.err
