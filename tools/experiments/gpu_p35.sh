for v in e4b2 e4b1 e4b3 e8b1 e8b2 e6b2 e4b2; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_retrieve.py 2>&1 | tail -1 | sed "s/^/v=$v /"; done
