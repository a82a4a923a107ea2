for t in 1 0 1 0; do PG_CHAIN_THROTTLE_LAST=$t timeout 200 python tools/experiments/exp_chain_steps.py 2>&1 | grep "independent" | sed "s/^/last=$t /"; done
PG_CHAIN_THROTTLE_LAST=0 timeout 200 python tools/experiments/exp_chain_timeline.py | tail -8
