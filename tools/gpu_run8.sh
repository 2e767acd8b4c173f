mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -q --timeout 120 -x -k "decode or chain or p13 or auto" > gpurun_out/pytest_dec.log 2>&1
echo "pytest exit $?" >> gpurun_out/status.txt
timeout 300 python tools/decode_timing.py > gpurun_out/dt.log 2>&1
echo "dt exit $?" >> gpurun_out/status.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode -s 2 -c 1 -o gpurun_out/prof_dec_g_m1 python tools/ncu_target.py decode --M 1 --N 22016 --K 8192 --reps 3 > gpurun_out/ncu1.log 2>&1
echo "ncu exit $?" >> gpurun_out/status.txt
