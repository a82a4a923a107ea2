# union program: upper bounds of the epilogue costs (PG_PROG_EXP knobs; results wrong by design)
for e in 0 1 2 3 4 7 0; do PG_PROG_EXP=$e timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program:" | sed "s/^/exp=$e /"; done
