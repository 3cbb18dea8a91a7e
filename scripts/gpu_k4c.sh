export FHWT_TUNING=1
python - <<'PY'
import os, torch, sys
sys.path.insert(0, '.')
import paper_1002_2184_b200 as fhwt
for L, shape in ((5, (8, 2048, 2048)), (8, (1, 4096, 4096))):
    x = torch.rand(*shape, device='cuda')
    c = fhwt.analyze_2d(x, L); r0 = fhwt.synthesize_2d(c, L)
    os.environ['FHWT_SYN_TC'] = '512'; os.environ['FHWT_DEBUG_LAUNCH'] = '1'
    for st in ('2', '3'):
        os.environ['FHWT_SYN_STAGES'] = st
        r = fhwt.synthesize_2d(c, L); torch.cuda.synchronize()
        print('L', L, 'stages', st, 'bitwise', bool(torch.equal(r, r0)), flush=True)
    del os.environ['FHWT_SYN_TC'], os.environ['FHWT_DEBUG_LAUNCH'], os.environ['FHWT_SYN_STAGES']
PY
ROUNDS=6 python tools/cmp_variants.py 5 'SYN:' 'SYN:FHWT_SYN_TC=512' 'SYN:FHWT_SYN_TC=512,FHWT_SYN_STAGES=3' 'ANA:' > gpurun_out/k4c.jsonl 2>gpurun_out/k4c.err; cat gpurun_out/k4c.jsonl; tail -3 gpurun_out/k4c.err
BATCH=1 SIZE=32768 ROUNDS=4 python tools/cmp_variants.py 8 'SYN:' 'SYN:FHWT_SYN_TC=512' 'SYN:FHWT_SYN_TC=512,FHWT_SYN_STAGES=3' > gpurun_out/k4c_c5.jsonl 2>>gpurun_out/k4c.err; cat gpurun_out/k4c_c5.jsonl
