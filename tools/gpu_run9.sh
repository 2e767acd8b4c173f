mkdir -p gpurun_out
timeout 300 python tools/decode_trace.py > gpurun_out/trace.log 2>&1
echo "trace exit $?" >> gpurun_out/status.txt
