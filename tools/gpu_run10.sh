mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 -x > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 300 python tools/decode_timing.py > gpurun_out/dt.log 2>&1
echo "dt exit $?" >> gpurun_out/status.txt
timeout 300 python tools/decode_trace.py > gpurun_out/trace.log 2>&1
echo "trace exit $?" >> gpurun_out/status.txt
