for v in "" w8 w16 w32 w64 "" w16 w32; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep -E "program:" | sed "s/^/v=$v /"; done
