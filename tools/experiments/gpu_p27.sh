timeout 600 python -m pytest tests/test_gpu_parity.py tests/test_gpu_peer.py -x -q 2>&1 | tail -1
for v in "" s4 s7; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_chain_steps.py 2>&1 | grep -E "independent" | sed "s/^/v=$v /"; done
PG_CHAIN_DYN=0 timeout 200 python tools/experiments/exp_chain_steps.py 2>&1 | grep -E "independent" | sed "s/^/dyn=0 /"
for v in "" s4; do PG_LIB_VARIANT=$v timeout 200 python tools/experiments/exp_c5b.py 2>&1 | grep fused | sed "s/^/v=$v /"; done
PG_CHAIN_DYN=0 timeout 200 python tools/experiments/exp_c5b.py 2>&1 | grep fused | sed "s/^/dyn=0 /"
