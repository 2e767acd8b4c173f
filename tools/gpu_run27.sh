mkdir -p gpurun_out
timeout 900 python tools/ab_decode.py paper_2312_03788_b200/_lib/variants/libsq_base.so paper_2312_03788_b200/_lib/variants/libsq_noload.so paper_2312_03788_b200/_lib/variants/libsq_noload_abl2.so > gpurun_out/ab.log 2>&1
echo "ab exit $?" >> gpurun_out/status.txt
