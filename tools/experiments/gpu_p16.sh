for v in "" red2 red4 poll50 poll200 stg4 ep8 "" ; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep -E "program:" | sed "s/^/v=$v /"; done
