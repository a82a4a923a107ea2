for e in 0 1 2 3 0; do PG_PROG_EXP=$e timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program:" | sed "s/^/exp=$e /"; done
