timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert" | head -4
for e in 0 0 0; do PG_PROG_EXP=$e timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep -E "program:|rel" | sed "s/^/exp=$e /"; done
PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9
