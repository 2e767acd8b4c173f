# quick GPU check: selected tests (pytest -k expression in $1), then optional extra command in $2
mkdir -p gpurun_out/quick
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" > gpurun_out/quick/pytest.log 2>&1; echo "pytest exit $?" > gpurun_out/quick/status.txt
if [ -n "$2" ]; then bash -c "$2" > gpurun_out/quick/extra.log 2>&1; echo "extra exit $?" >> gpurun_out/quick/status.txt; fi
