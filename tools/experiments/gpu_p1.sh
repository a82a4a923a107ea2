O=gpurun_out; mkdir -p $O
timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q > $O/p1_test.log 2>&1; echo "rc=$?" >> $O/p1_test.log
tail -30 $O/p1_test.log
timeout 200 python tools/experiments/exp_prog.py 4 2>&1 | tail -8
timeout 300 python tools/experiments/exp_prog.py 32 2>&1 | tail -8
