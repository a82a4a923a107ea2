for m in 0 1 2 3; do
  echo "== mode $m"
  PG_PROG_MODE=$m timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert|^FAILED" | head -6
  PG_PROG_MODE=$m PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -10
  PG_PROG_MODE=$m timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program:"
done
