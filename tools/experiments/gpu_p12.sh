timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert" | head -4
timeout 200 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -1
for t in 1 0 1 0; do PG_PROG_TMA_OUT=$t timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep "program:" | sed "s/^/tma=$t /"; done
PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9
