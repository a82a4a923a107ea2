PG_POOLV=0 timeout 200 python tools/experiments/exp_pool.py 2>&1 | sed "s/^/old /"
timeout 200 python tools/experiments/exp_pool.py 2>&1 | sed "s/^/new /"
python -c "
import numpy as np
for n in (4096, 11008):
    a=np.load(f'/tmp/pool_{n}_0.npy'); b=np.load(f'/tmp/pool_{n}_d.npy'); print(n, 'bit-identical', np.array_equal(a.view(np.int64), b.view(np.int64)))"
timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_prefill_routed.py -x -q 2>&1 | tail -2
timeout 300 python tools/experiments/exp_route2.py 2>&1 | tail -1
PG_POOLV=0 timeout 300 python tools/experiments/exp_route2.py 2>&1 | tail -1
