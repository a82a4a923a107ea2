export EXP_SHAPES="2048,4096,832;32768,4096,832;32768,832,4096;8192,8192,8192"
for v in head w4 ""; do echo "== lib '$v'"; PG_LIB_VARIANT=$v timeout 300 python tools/experiments/exp_gemm.py 2>&1 | tail -4; PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prefill.py 2>&1 | head -1; done
timeout 600 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_routed.py -q -x 2>&1 | tail -1
