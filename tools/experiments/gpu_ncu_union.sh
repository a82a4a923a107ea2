#!/bin/bash
# ncu of the union kernels (q shape, T=256): launch list + one full capture of each stage
O=gpurun_out; mkdir -p $O
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_union_wm -c 8 --csv \
  --log-file $O/wm_launches.csv python tools/experiments/exp_union_dbg.py > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_union_wm -s 2 -c 2 \
  -o $O/wm_full -f python tools/experiments/exp_union_dbg.py > $O/wm_ncu.log 2>&1
tail -3 $O/wm_ncu.log
