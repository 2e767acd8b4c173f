mkdir -p gpurun_out
timeout 600 python tools/ab_decode.py paper_2312_03788_b200/_lib/variants/libsq_v3.so paper_2312_03788_b200/_lib/variants/libsq_v5.so > gpurun_out/ab.log 2>&1
echo "ab exit $?" >> gpurun_out/status.txt
