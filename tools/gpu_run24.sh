mkdir -p gpurun_out
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 3 --warmup 3 --layers 4 --prefill-layers 1 --backend gloo --one-device --no-graph --skip-e2e > gpurun_out/bench_tp2.log 2>&1
echo "bench tp2 exit $?" >> gpurun_out/status.txt
timeout 300 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29534 bench.py --impl reference --gpus 2 --steps 2 --warmup 1 > gpurun_out/ref_tp2.log 2>&1
echo "ref tp2 exit $?" >> gpurun_out/status.txt
