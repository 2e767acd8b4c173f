# final numbers: bench line + C5 sweep with the final kernels
O=gpurun_out/r02d; mkdir -p $O
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench $?" >> $O/status.txt
timeout 900 python tools/m_sweep.py --out $O/msweep.jsonl > $O/msweep.log 2>&1; echo "msweep $?" >> $O/status.txt
