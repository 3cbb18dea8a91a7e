export FHWT_TUNING=1
ROUNDS=4 python tools/cmp_variants.py 5 'MB:tma/1/2/1/0/256' 'MB:tma/1/2/1/1/256' 'MB:tma/1/3/1/1/256' 'MB:tma/1/2/1/1/128' 'MB:tma/1/3/1/1/128' 'MB:tma/16/3/1/1/128' 'MB:tma/1/2/1/0/128' 'COPY:' > gpurun_out/mb2.jsonl 2>gpurun_out/mb2.err; cat gpurun_out/mb2.jsonl; tail -2 gpurun_out/mb2.err
python -m pytest tests/test_gpu_parity.py -q -x -k "tile_counter_workspace" -p no:cacheprovider 2>&1 | tail -1
