mkdir -p gpurun_out/base
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > gpurun_out/base/smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/base/pytest_gpu.log 2>&1; echo "pytest exit $?" >> gpurun_out/base/status.txt
timeout 600 python bench.py > gpurun_out/base/bench.log 2>&1; echo "bench exit $?" >> gpurun_out/base/status.txt
