mkdir -p gpurun_out
timeout 600 python bench.py > gpurun_out/bench.log 2>&1
echo "bench exit $?" >> gpurun_out/status.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/launches.csv python bench.py --steps 2 --warmup 1 --layers 2 --skip-e2e --skip-cpu --no-graph > gpurun_out/bench_ncu.log 2>&1
echo "ncu launches exit $?" >> gpurun_out/status.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:decode -s 1 -c 2 -o gpurun_out/prof_decode python tools/ncu_target.py decode --M 16 > gpurun_out/ncu_dec.log 2>&1
echo "ncu dec exit $?" >> gpurun_out/status.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:prefill -s 1 -c 1 -o gpurun_out/prof_prefill python tools/ncu_target.py prefill > gpurun_out/ncu_pre.log 2>&1
echo "ncu pre exit $?" >> gpurun_out/status.txt
timeout 300 ncu --set full --clock-control none --import-source on -k regex:quantize -s 1 -c 1 -o gpurun_out/prof_quant python tools/ncu_target.py quant > gpurun_out/ncu_q.log 2>&1
echo "ncu q exit $?" >> gpurun_out/status.txt
