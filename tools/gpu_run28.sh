mkdir -p gpurun_out
SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_noload.so timeout 300 ncu --set full --clock-control none -k regex:decode -s 2 -c 1 -o gpurun_out/prof_noload python tools/ncu_target.py decode --M 1 --N 44032 --K 8192 --reps 3 > gpurun_out/ncu.log 2>&1
SQ_LIB=paper_2312_03788_b200/_lib/variants/libsq_noload.so timeout 300 ncu --set full --clock-control none -k regex:decode -s 2 -c 1 -o gpurun_out/prof_noload16 python tools/ncu_target.py decode --M 16 --N 44032 --K 8192 --reps 3 > gpurun_out/ncu16.log 2>&1
echo "ncu exit $?" >> gpurun_out/status.txt
