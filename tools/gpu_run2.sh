mkdir -p gpurun_out
timeout 120 python tools/diag_prefill.py > gpurun_out/diag.log 2>&1
echo "diag exit $?" >> gpurun_out/status.txt
