#!/bin/bash
# union-path check: parity tests, then per-layer timing new (weights-on-M) vs round-1 path
O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_prefill.py -x -q -k "union" > $O/union_pytest.log 2>&1; echo "rc=$?" >> $O/union_pytest.log
tail -15 $O/union_pytest.log
for wm in 1 0; do
  echo "== PG_UNION_WM=$wm"; PG_UNION_WM=$wm timeout 120 python tools/experiments/exp_union.py 2>&1 | tail -9
done
