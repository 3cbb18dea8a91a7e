# Synthesis on 32 x 128 tiles: cp.async (FHWT_SYN_WARP128=0) vs the warp-decoupled kernel (=1), table
export FHWT_TUNING=1   # the library honours FHWT_* knobs only behind this gate
# defaults (GB/s synthesis)
S="${S:-1024,480,640,3;512,600,800,3;256,1152,1152,3;512,768,896,3;256,1000,1152,3;512,480,640,4;256,1152,1152,4;512,480,640,5}"
run() { echo "$1 $(env $2 SHAPES="$S" timeout 100 python tools/generic_shapes.py 2>&1 | sed 's/ L=\(.\): analysis [0-9]* GB.s, synthesis /:L\1 /; s/ GB.s, rt err.*//' | tr '\n' ' ')"; }
for r in 1 2; do run cpasync "FHWT_SYN_WARP128=0"; run warp "FHWT_SYN_WARP128=1"; run default "X=1"; done
