for v in "" p2b64 p2b256 p2b512 p2a32 p2a32b256; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_pool.py 2>&1 | grep "n=4096" | sed "s/^/v=$v /"; done
