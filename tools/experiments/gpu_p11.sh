timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert" | head -4
for m in auto 1 0 auto; do echo "== split $m"; if [ $m = auto ]; then unset PG_PROG_SPLIT; else export PG_PROG_SPLIT=$m; fi
timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep -E "program:"; done
unset PG_PROG_SPLIT; PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9
