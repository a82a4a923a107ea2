timeout 600 python -m pytest tests/test_gpu_prefill_routed.py -x -q 2>&1 | tail -2
for v in "" g4; do PG_LIB_VARIANT=$v timeout 300 python tools/experiments/exp_c3.py 2>&1 | head -1 | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print('$v', json.dumps(d['modes'])[:330], d['route_ms'])"; done
