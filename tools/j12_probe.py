import torch, sys, os
sys.path.insert(0, os.getcwd())
import paper_1002_2184_b200 as fhwt
x = torch.rand(65536, 4096, device="cuda")
for J in (10, 11, 12):
    plan = fhwt.Plan1d(4096, 65536, J)
    ws = torch.empty(max(plan.workspace_bytes, 1), dtype=torch.uint8, device="cuda")
    c = plan.analyze(x, workspace=ws); r = plan.synthesize(c, workspace=ws)
    e = [torch.cuda.Event(enable_timing=True) for _ in range(3)]
    torch.cuda.synchronize(); e[0].record()
    for _ in range(10): plan.analyze(x, out=c, workspace=ws)
    e[1].record()
    for _ in range(10): plan.synthesize(c, out=r, workspace=ws)
    e[2].record(); torch.cuda.synchronize()
    print(J, e[0].elapsed_time(e[1]) / 10, e[1].elapsed_time(e[2]) / 10)
