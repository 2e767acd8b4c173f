mkdir -p gpurun_out
timeout 300 python tools/decode_timing.py > gpurun_out/dt.log 2>&1
echo "dt exit $?" >> gpurun_out/status.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode -s 2 -c 1 -o gpurun_out/prof_dec_o_m1 python tools/ncu_target.py decode --M 1 --N 8192 --K 8192 --reps 3 > gpurun_out/ncu1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode -s 2 -c 1 -o gpurun_out/prof_dec_g_m16 python tools/ncu_target.py decode --M 16 --N 22016 --K 8192 --reps 3 > gpurun_out/ncu2.log 2>&1
echo "ncu exit $?" >> gpurun_out/status.txt
