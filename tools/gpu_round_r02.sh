# Round-2 evidence: bench line, ncu launch list of the headline step, ncu captures, sanitizers.
# (split in parts: gpurun returns at most 64 MiB of gpurun_out/)
mkdir -p gpurun_out/r02
part=${1:-all}
if [ $part = bench ] || [ $part = all ]; then
timeout 900 python bench.py > gpurun_out/r02/bench.log 2>&1; echo "bench $?" >> gpurun_out/r02/status.txt
for t in memcheck racecheck synccheck initcheck; do
  timeout 900 compute-sanitizer --tool $t --print-limit 20 python tools/sanitize_cases.py > gpurun_out/r02/sanitize_$t.log 2>&1
  echo "$t $?" >> gpurun_out/r02/status.txt
done
fi
if [ $part = ncu ] || [ $part = all ]; then
for spec in "decode_m1_gateup decode --M 1 --N 44032 --K 8192" "decode_m16_gateup decode --M 16 --N 44032 --K 8192" "decode_m1_oproj decode --M 1 --N 8192 --K 8192" "prefill_gate prefill --M 2048 --N 22016 --K 8192" "quant quant --N 22016 --K 8192" "prefill_m32_gateup prefill --M 32 --N 44032 --K 8192"; do
  set -- $spec; name=$1; shift; kind=$1
  k=decode; [ $kind = prefill ] && k=prefill; [ $kind = quant ] && k=quantize
  rep=gpurun_out/r02/prof_$name
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:$k -s 2 -c 1 -o $rep python tools/ncu_target.py "$@" --reps 3 > gpurun_out/r02/ncu_$name.log 2>&1
  # text exports travel back; reports above 8 MB (source-embedded decode captures) do not
  ncu -i $rep.ncu-rep --page raw --csv > $rep.raw.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page details --csv > $rep.details.csv 2>/dev/null
  ncu -i $rep.ncu-rep --page source --csv --print-source sass 2>/dev/null | gzip > $rep.sass.csv.gz
  [ $(stat -c %s $rep.ncu-rep) -gt 8000000 ] && rm -f $rep.ncu-rep
done
du -sh gpurun_out/r02/* >> gpurun_out/r02/status.txt
fi
if [ $part = launches ] || [ $part = all ]; then
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/launches.csv python bench.py --steps 1 --warmup 3 --skip-prefill --skip-quant --skip-calib --skip-7b --skip-e2e --skip-cpu --skip-gates > gpurun_out/r02/bench_ncu.log 2>&1; echo "launches $?" >> gpurun_out/r02/status.txt
ls -la /tmp/launches.csv >> gpurun_out/r02/status.txt
python tools/make_profiles.py launches-only /tmp/launches.csv gpurun_out/r02/launches.txt >> gpurun_out/r02/status.txt 2>&1
gzip -c /tmp/launches.csv > gpurun_out/r02/launches.csv.gz
fi
