mkdir -p gpurun_out
SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_pair.so timeout 300 python tools/diag_prefill.py > gpurun_out/diag.log 2>&1
echo "diag exit $?" >> gpurun_out/status.txt
SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_pair.so timeout 400 python -m pytest tests -m gpu -q -x --timeout 60 -k "prefill or p13 or auto or zero" > gpurun_out/pytest_pair.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 600 python tools/ab_decode.py --prefill paper_2312_03788_b200/_lib/variants/libsq_base.so paper_2312_03788_b200/_lib/variants/libsq_pair.so > gpurun_out/ab.log 2>&1
echo "ab exit $?" >> gpurun_out/status.txt
