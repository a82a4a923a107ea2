#!/bin/bash
# ncu --set full of one phase kernel of the grouped config-4 layer (skip S union kernels)
O=gpurun_out; mkdir -p $O
S=${1:-1}
PG_UNION_WM=1 EXP_REPS=1 timeout 600 ncu --set full --clock-control none --import-source on -k regex:k_union_wm -s $S -c 1 \
  -o $O/phase_full_$S -f python tools/experiments/exp_union.py > $O/phase_full_$S.log 2>&1
tail -2 $O/phase_full_$S.log
