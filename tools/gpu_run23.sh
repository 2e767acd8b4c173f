mkdir -p gpurun_out
timeout 600 python -m pytest tests/test_tp_gpu.py -q -x > gpurun_out/pytest_tp.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --layers 4 --prefill-layers 1 --backend gloo --one-device --no-graph --skip-e2e > gpurun_out/bench_tp2.log 2>&1
echo "bench tp2 exit $?" >> gpurun_out/status.txt
