# Short-signal chunk kernels: chunk size x ring depth x CTAs/SM (analysis / synthesis GB/s)
export FHWT_TUNING=1   # the library honours FHWT_* knobs only behind this gate
for ch in 4096 8192 16384; do for st in 2 3; do for c in 0 2 4 6; do
  echo "chunk=$ch stages=$st ctas=$c $(FHWT_SMALL1D_CHUNK=$ch FHWT_SMALL_STAGES=$st FHWT_SMALL_CTAS=$c python - <<'PY'
import torch, paper_1002_2184_b200 as fhwt
out = []
for (b, n, J) in ((1048576, 256, 8), (262144, 512, 9), (2097152, 128, 7)):
    x = torch.rand(b, n, device="cuda"); p = fhwt.Plan1d(n, b, J)
    c = p.analyze(x); r = p.synthesize(c)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize(); e[0].record()
    for _ in range(10): p.analyze(x, out=c)
    e[1].record()
    for _ in range(10): p.synthesize(c, out=r)
    e[2].record(); torch.cuda.synchronize()
    S = x.numel(); out.append(f"{n}:{8*S/(e[0].elapsed_time(e[1])/10)/1e6:.0f}/{8*S/(e[1].elapsed_time(e[2])/10)/1e6:.0f}")
print(" ".join(out))
PY
)"
done; done; done
