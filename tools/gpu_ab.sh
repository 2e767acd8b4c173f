set -x
V=paper_2312_03788_b200/_lib/variants
SQ_LIB=$PWD/$V/libsq_sleep.so timeout 600 python -m pytest tests -m gpu -x -q -k "decode or p13 or zero or auto or chain" 2>&1 | tail -2
timeout 600 python tools/ab_decode.py $V/libsq_sk.so:3=1 $V/libsq_sleep.so:3=1 $V/libsq_rb.so:3=2 $V/libsq_sleep2.so:3=2 2>&1 | tail -8
