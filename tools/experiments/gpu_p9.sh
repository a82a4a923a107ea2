for v in "" s5b4 s4b4; do
echo "== variant '$v'"
PG_LIB_VARIANT=${v} timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed" | head -2
PG_LIB_VARIANT=${v} PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9 | head -4
PG_LIB_VARIANT=${v} timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program:"
done
