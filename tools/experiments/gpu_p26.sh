for v in "" pr4 pr2; do PG_LIB_VARIANT=$v timeout 300 python tools/experiments/exp_c3_overlap.py 2>&1 | sed "s/^/v=$v /"; done
