for v in "" eskip; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_gemm.py 2>&1 | sed "s/^/v=$v /"; done
for v in "" eskip; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prefill.py 2>&1 | sed "s/^/v=$v /"; done
