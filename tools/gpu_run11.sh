mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 -x -k "decode or chain" > gpurun_out/pytest_dec.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 400 python tools/decode_timing.py --tail 0,0.05,0.1,0.2 > gpurun_out/dt.log 2>&1
echo "dt exit $?" >> gpurun_out/status.txt
