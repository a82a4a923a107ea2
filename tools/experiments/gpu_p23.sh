PG_POOLV=0 timeout 200 python tools/experiments/exp_pool.py 2>&1 | sed "s/^/old /"
for v in "" v4b16 v8b16 v4b32k32 v8b16k32; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_pool.py 2>&1 | sed "s/^/v=$v /"; done
python -c "
import numpy as np
for n in (4096, 11008):
    a=np.load(f'/tmp/pool_{n}_0.npy'); b=np.load(f'/tmp/pool_{n}_d.npy'); print(n, 'bit-identical', np.array_equal(a.view(np.int64), b.view(np.int64)))"
