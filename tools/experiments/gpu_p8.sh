for m in 1 0; do
export PG_PROG_REDADD=$m
echo "== redadd $m"
timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert|^FAILED" | head -6
PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9
timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program"
done
