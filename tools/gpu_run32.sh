mkdir -p gpurun_out
SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_pair.so timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill -s 1 -c 1 -o gpurun_out/prof_pair python tools/ncu_target.py prefill --M 2048 --N 8192 --K 8192 --reps 2 > gpurun_out/ncu.log 2>&1
echo "ncu exit $?" >> gpurun_out/status.txt
