FHWT_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-breakdown --no-direct --sustained 0 > gpurun_out/tr2_c4.json 2> gpurun_out/tr2_c4.err; echo "tr2 c4 rc=$?"
FHWT_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --workload c5 --no-breakdown --no-direct --no-e2e --sustained 0 > gpurun_out/tr2_c5.json 2> gpurun_out/tr2_c5.err; echo "tr2 c5 rc=$?"
for w in c4 c5; do python -c "
import json; d=json.loads(open('gpurun_out/tr2_$w.json').read().strip().splitlines()[-1]); print('$w', round(d['value']), d['config']['global_batch'], d['config']['per_rank'], d['parity'], d.get('multi_gpu'))"; done
tail -3 gpurun_out/tr2_c5.err
