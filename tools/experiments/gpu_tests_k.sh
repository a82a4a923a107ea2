# gpu tests subset: bash tools/experiments/gpu_tests_k.sh "<pytest -k expr>"
O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "$1" 2>&1 | tail -15
