# last check of the round: every GPU test, smoke, the bench line
O=gpurun_out/final; mkdir -p $O
timeout 1500 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest $?" >> $O/status.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke $?" >> $O/status.txt
timeout 900 python bench.py > $O/bench.log 2>&1; echo "bench $?" >> $O/status.txt
