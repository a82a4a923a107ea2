timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_routed.py tests/test_gpu_parity.py -x -q 2>&1 | tail -1
for v in "" w32 "" w32; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prefill.py 2>&1 | head -1 | sed "s/^/v=$v /"; done
for v in "" w32; do PG_LIB_VARIANT=$v EXP_SHAPES="32768,4096,832;32768,11008,1216;32768,832,4096;8192,8192,8192" timeout 200 python tools/experiments/exp_gemm.py 2>&1 | sed "s/^/v=$v /"; done
