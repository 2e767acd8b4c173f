mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 -x > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 300 python tools/quick_bench.py --decode > gpurun_out/qb_dec.log 2>&1
echo "qb exit $?" >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/status.txt
