# Analysis ring depth x CTAs/SM for the narrower fast tiles (32 x 128, 16 x 128, 16 x 256)
export FHWT_TUNING=1   # the library honours FHWT_* knobs only behind this gate
S="${S:-1024,400,544,3;128,720,1280,4;32,2160,3840,4;64,1200,1600,4}"
for st in ${STAGES:-2 3 4}; do for c in ${CTAS:-2 3 4 99}; do
  echo "stages=$st ctas=$c $(FHWT_ANA_STAGES=$st FHWT_ANA_CTAS_PER_SM=$c SHAPES="$S" timeout 100 python tools/generic_shapes.py 2>&1 | sed 's/, synthesis.*//; s/ L=.: analysis / /' | tr '\n' ' ')"
done; done
