for e in 0 8 0 8; do PG_PROG_EXP=$e timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program:" | sed "s/^/exp=$e /"; done
