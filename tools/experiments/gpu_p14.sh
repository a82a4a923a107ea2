for e in 0 7; do echo "== exp=$e"; PG_PROG_EXP=$e PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9; done
