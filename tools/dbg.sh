export CUDA_LAUNCH_BLOCKING=1
export FHWT_TUNING=1   # the library honours FHWT_* knobs only behind this gate
for c in "4 4 3 2" "8 8 2 3" "32 4 2 2" "16 24 1 3" "32 32 1 5" "96 320 2 5" "64 64 2 6" "96 512 1 5" "96 320 1 3" "32 288 1 5" "32 256 1 5" "32 512 1 5" "64 512 1 5"; do
  timeout 60 python tools/debug_case.py 2d syn $c 2>&1 | tail -1
done
