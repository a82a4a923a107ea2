timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert" | head -4
for v in "" own0 "" own0; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep -E "program:|rel" | sed "s/^/v=$v /"; done
PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9
