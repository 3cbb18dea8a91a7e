set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/r2_pytest.log 2>&1; echo "pytest rc=$?" >> gpurun_out/r2_pytest.log
tail -5 gpurun_out/r2_pytest.log
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/r2_smoke.log 2>&1; echo "smoke rc=$?"
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2_bench.json 2> gpurun_out/r2_bench.err; echo "bench rc=$?"
tail -3 gpurun_out/r2_bench.err
FHWT_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29611 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-breakdown --no-direct --sustained 0 > gpurun_out/r2_torchrun2_c4.json 2> gpurun_out/r2_torchrun2_c4.err; echo "tr2 c4 rc=$?"
FHWT_BENCH_ONE_DEVICE=1 timeout 900 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29612 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --workload c5 --no-breakdown --no-direct --no-e2e --sustained 0 > gpurun_out/r2_torchrun2_c5.json 2> gpurun_out/r2_torchrun2_c5.err; echo "tr2 c5 rc=$?"
tail -3 gpurun_out/r2_torchrun2_c5.err
