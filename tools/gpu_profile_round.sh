# One-shot evidence capture: launch list of a short bench, ncu --set full of each hot kernel.
mkdir -p gpurun_out
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layers 2 --prefill-layers 1 --skip-e2e --skip-cpu --no-graph > gpurun_out/bench_ncu.log 2>&1
echo "launches exit $?" >> gpurun_out/status.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode -s 2 -c 1 -o gpurun_out/prof_decode_m1 python tools/ncu_target.py decode --M 1 --N 44032 --K 8192 --reps 3 > gpurun_out/ncu_d1.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode -s 2 -c 1 -o gpurun_out/prof_decode_m16 python tools/ncu_target.py decode --M 16 --N 44032 --K 8192 --reps 3 > gpurun_out/ncu_d16.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill -s 1 -c 1 -o gpurun_out/prof_prefill python tools/ncu_target.py prefill --M 2048 --N 22016 --K 8192 --reps 2 > gpurun_out/ncu_p.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize -s 1 -c 1 -o gpurun_out/prof_quant python tools/ncu_target.py quant --N 22016 --K 8192 --reps 2 > gpurun_out/ncu_q.log 2>&1
timeout 300 ncu --set full --clock-control none --import-source on -k regex:colabsmax -s 1 -c 1 -o gpurun_out/prof_smooth python tools/ncu_target.py smooth --N 22016 --K 8192 --reps 2 > gpurun_out/ncu_s.log 2>&1
echo "ncu exit $?" >> gpurun_out/status.txt
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/status.txt
