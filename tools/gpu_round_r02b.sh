# Round-2 (second half) evidence: full GPU tests, smoke, bench line, the sanitizer cases run plain
# (incl. the packed u4 zero-point path), ncu captures of the changed kernels (quantize; decode with u4 zeros).
O=gpurun_out/r02b; mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.limit --format=csv > $O/smi.txt 2>&1
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest $?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench $?" >> $O/status.txt
# compute-sanitizer is closed on this pool (it left GPUs needing a reset); the sanitizer cases
# still run plain, with their own result checks (u4 GEMM == fp16-Z GEMM bit for bit, etc.)
timeout 600 python tools/sanitize_cases.py > $O/sanitize_cases_plain.log 2>&1; echo "sanitize_cases $?" >> $O/status.txt
for spec in "quant quant --N 22016 --K 8192" "decode_m1_gateup_u4 decode --M 1 --N 44032 --K 8192 --zeros-u4"; do
  set -- $spec; name=$1; shift; kind=$1
  k=decode; [ $kind = quant ] && k=quantize
  rep=$O/prof_$name
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $rep python tools/ncu_target.py "$@" --reps 3 > $O/ncu_$name.log 2>&1
  ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > $rep.details.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $rep.sass.csv.gz
  gzip -f $rep.raw.csv
  [ $(stat -c %s $rep.ncu-rep) -gt 8000000 ] && rm -f $rep.ncu-rep
done
echo done >> $O/status.txt
