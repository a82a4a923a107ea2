for v in "" rp "" rp; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_chain_steps.py 2>&1 | grep -E "independent|chain 1/" | sed "s/^/v=$v /"; done
