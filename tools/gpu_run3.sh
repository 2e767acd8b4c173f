mkdir -p gpurun_out
timeout 120 python tools/diag_prefill.py > gpurun_out/diag.log 2>&1
echo "diag exit $?" >> gpurun_out/status.txt
timeout 900 python -m pytest tests -m gpu -q --timeout 120 > gpurun_out/pytest_all.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 200 python tools/quick_bench.py --prefill --pm 512,2048,4096 > gpurun_out/qb_pre.log 2>&1
echo "qbpre exit $?" >> gpurun_out/status.txt
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/status.txt
