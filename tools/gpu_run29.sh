mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q -x -k "prefill or p13 or auto or zero" > gpurun_out/pytest_p.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 900 python tools/ab_decode.py --prefill paper_2312_03788_b200/_lib/variants/libsq_prefill_old.so paper_2312_03788_b200/_lib/variants/libsq_base.so > gpurun_out/ab.log 2>&1
echo "ab exit $?" >> gpurun_out/status.txt
