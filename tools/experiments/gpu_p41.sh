for v in "" st5 cs16 cs64 st5s4 ""; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep -E "program:" | sed "s/^/v=$v /"; done
