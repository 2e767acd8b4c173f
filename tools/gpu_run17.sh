mkdir -p gpurun_out
timeout 900 python tools/ab_decode.py paper_2312_03788_b200/_lib/variants/libsq_base.so paper_2312_03788_b200/_lib/variants/libsq_sx.so > gpurun_out/ab.log 2>&1
echo "ab exit $?" >> gpurun_out/status.txt
SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_sx.so timeout 600 python -m pytest tests -m gpu -q -x -k "decode or chain" > gpurun_out/pytest_sx.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_sx.so timeout 300 ncu --set full --clock-control none -k regex:decode -s 2 -c 1 -o gpurun_out/prof_sx python tools/ncu_target.py decode --M 1 --N 44032 --K 8192 --reps 3 > gpurun_out/ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/status.txt
