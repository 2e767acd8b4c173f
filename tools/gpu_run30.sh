mkdir -p gpurun_out
timeout 300 python tools/cublas_ref.py > gpurun_out/cublas.log 2>&1
nvidia-smi --query-gpu=clocks.sm,clocks.max.sm,power.draw --format=csv >> gpurun_out/cublas.log
timeout 300 python tools/quick_bench.py --prefill --pm 2048 >> gpurun_out/cublas.log 2>&1
