export PG_PROG_MODE=${PG_PROG_MODE:-3}
for i in 1 2 3 4; do timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert|^FAILED" | head -6; done
PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -11
timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program:"
