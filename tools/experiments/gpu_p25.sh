timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefill_routed.py -x -q 2>&1 | tail -2
for v in 3 1 3 1; do PG_SCORE_V2=$v timeout 300 python tools/experiments/exp_route2.py 2>&1 | tail -1 | sed "s/^/score v$v /"; done
