mkdir -p gpurun_out
nvidia-smi > gpurun_out/smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -q --timeout 120 -k "not prefill and not p13 and not auto" > gpurun_out/pytest_dec.log 2>&1
echo "dec exit $?" >> gpurun_out/status.txt
timeout 300 python tools/quick_bench.py --decode --quant > gpurun_out/qb_dec.log 2>&1
echo "qb exit $?" >> gpurun_out/status.txt
timeout 400 python -m pytest tests -m gpu -q --timeout 60 -x -k "prefill or p13 or auto" > gpurun_out/pytest_pre.log 2>&1
echo "pre exit $?" >> gpurun_out/status.txt
timeout 200 python tools/quick_bench.py --prefill > gpurun_out/qb_pre.log 2>&1
echo "qbpre exit $?" >> gpurun_out/status.txt
timeout 120 python __graft_entry__.py smoke > gpurun_out/smoke.log 2>&1
echo "smoke exit $?" >> gpurun_out/status.txt
