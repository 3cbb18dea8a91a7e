# Small-image chunk kernels: chunk size x ring depth (analysis / synthesis GB/s)
export FHWT_TUNING=1   # the library honours FHWT_* knobs only behind this gate
for ch in 4096 8192 16384; do for st in 2 3; do
  echo "chunk=$ch stages=$st $(FHWT_SMALL_CHUNK=$ch FHWT_SMALL_STAGES=$st SMALL=1 SHAPES="65536,32,32,5;16384,64,64,6;65536,16,64,4;16384,64,64,3" timeout 100 python tools/generic_shapes.py 2>&1 | sed 's/ L=.: analysis / /; s/ GB.s, synthesis /\//; s/ GB.s, rt err.*//' | tr '\n' ' ')"
done; done
