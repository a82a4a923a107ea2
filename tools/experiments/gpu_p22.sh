timeout 600 python -m pytest tests/test_gpu_prefill_routed.py tests/test_gpu_prefill.py -x -q 2>&1 | tail -2
for v in "" wp0 "" wp0; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prefill.py 2>&1 | grep "prefill P" | sed "s/^/v=$v /"; done
