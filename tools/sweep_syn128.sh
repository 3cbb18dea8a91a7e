# Synthesis ring depth x CTAs/SM for the narrower fast tiles (cp.async variant)
export FHWT_TUNING=1   # the library honours FHWT_* knobs only behind this gate
S="${S:-1024,480,640,3;512,600,800,3;256,1152,1152,3;1024,400,544,3;64,1200,1600,4}"
for st in ${STAGES:-2 3 4}; do for c in ${CTAS:-2 3 4}; do
  echo "stages=$st ctas=$c $(FHWT_SYN_STAGES=$st FHWT_CTAS_PER_SM=$c FHWT_ANA_CTAS_PER_SM=0 SHAPES="$S" timeout 100 python tools/generic_shapes.py 2>&1 | sed 's/ L=.: analysis [0-9]* GB.s, synthesis / /; s/, rt err.*//' | tr '\n' ' ')"
done; done
