# Round-2 final evidence: full GPU tests, smoke, bench line, plain sanitizer cases, ncu launch
# list of the headline step and ncu captures of the kernels changed in the second half.
O=gpurun_out/r02c; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest $?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench $?" >> $O/status.txt
timeout 600 python tools/sanitize_cases.py > $O/sanitize_cases_plain.log 2>&1; echo "sanitize_cases $?" >> $O/status.txt
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 1 --warmup 3 --skip-prefill --skip-quant --skip-calib --skip-7b --skip-e2e --skip-cpu --skip-gates > $O/bench_ncu.log 2>&1; echo "launches $?" >> $O/status.txt
python tools/make_profiles.py launches-only /tmp/launches.csv $O/launches.txt >> $O/status.txt 2>&1
for spec in "decode_m1_gateup decode --M 1 --N 44032 --K 8192" "decode_m1_qkv decode --M 1 --N 10240 --K 8192" "prefill_m32_gateup prefill --M 32 --N 44032 --K 8192"; do
  set -- $spec; name=$1; shift; kind=$1
  k=decode; [ $kind = prefill ] && k=prefill
  rep=$O/prof_$name
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $rep python tools/ncu_target.py "$@" --reps 3 > $O/ncu_$name.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > $rep.details.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $rep.sass.csv.gz
  gzip -f $rep.raw.csv
  [ $(stat -c %s $rep.ncu-rep) -gt 8000000 ] && rm -f $rep.ncu-rep
done
timeout 900 python tools/m_sweep.py --out $O/msweep.jsonl > $O/msweep.log 2>&1; echo "msweep $?" >> $O/status.txt
echo done >> $O/status.txt
