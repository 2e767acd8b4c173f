mkdir -p gpurun_out
timeout 900 python tools/ab_decode.py paper_2312_03788_b200/_lib/variants/libsq_base.so paper_2312_03788_b200/_lib/variants/libsq_gpw2.so paper_2312_03788_b200/_lib/variants/libsq_gpw2c1.so > gpurun_out/ab.log 2>&1
echo "ab exit $?" >> gpurun_out/status.txt
SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_gpw2.so timeout 600 python -m pytest tests -m gpu -q -x -k "decode" > gpurun_out/pytest_g.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
