timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | tail -1
for v in "" fl0 "" fl0; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_prog.py 32 2>&1 | grep -E "program:" | sed "s/^/v=$v /"; done
