for t in 1 0 1 0; do PG_CHAIN_L2PF=$t timeout 200 python tools/experiments/exp_chain_steps.py 2>&1 | grep "independent" | sed "s/^/l2pf=$t /"; done
PG_CHAIN_L2PF=1 timeout 200 python tools/experiments/exp_chain_timeline.py | tail -6
