set -x
V=paper_2312_03788_b200/_lib/variants
timeout 900 python -m pytest tests -m gpu -x -q -k "prefill or p13 or zero or auto" 2>&1 | tail -2
SQ_LIB=$PWD/$V/libsq_pair.so timeout 900 python -m pytest tests -m gpu -x -q -k "prefill_parity or p13" 2>&1 | tail -2
timeout 600 python tools/ab_decode.py --prefill $V/libsq_pbase.so $V/libsq_pcs.so $V/libsq_pel.so $V/libsq_pair.so 2>&1 | tail -4
timeout 900 python tools/ab_decode.py --prefill --ms=17,64,128 $V/libsq_pcs.so $V/libsq_pel.so 2>&1 | tail -12
