timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert" | head -4
for c in 1 2; do echo "== chains $c"; EXP_CHAINS=$c timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep -E "program|rel"; done
EXP_CHAINS=2 PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -9
