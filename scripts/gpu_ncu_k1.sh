# ncu --set full of the analysis kernels: default (fused) vs the warp-specialised variant
export FHWT_TUNING=1
ncu --set full --clock-control none --import-source on -k regex:ana2d -c 1 -o gpurun_out/k1_default -f python tools/profile_case.py c4 64 > gpurun_out/k1_ncu_default.log 2>&1; echo "rc=$?"
FHWT_ANA_FUSED=8 ncu --set full --clock-control none --import-source on -k regex:ana2d -c 1 -o gpurun_out/k1_ws8 -f python tools/profile_case.py c4 64 > gpurun_out/k1_ncu_ws8.log 2>&1; echo "rc=$?"
ncu --set full --clock-control none -k regex:copy -c 1 -o gpurun_out/k1_copy -f python -c "
import torch; x=torch.rand(64,2048,2048,device='cuda'); y=torch.empty_like(x); y.copy_(x); y.copy_(x); torch.cuda.synchronize()" > gpurun_out/k1_ncu_copy.log 2>&1; echo "rc=$?"
ls -la gpurun_out/
