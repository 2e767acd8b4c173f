mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 -x > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 400 python tools/decode_timing.py --tail 0,0.05 > gpurun_out/dt.log 2>&1
echo "dt exit $?" >> gpurun_out/status.txt
timeout 600 python bench.py --skip-cpu > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/status.txt
