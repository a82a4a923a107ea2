#!/bin/bash
# per-kernel device times of one grouped config-4 layer (8 GEMM phases), both union paths
O=gpurun_out; mkdir -p $O
for wm in 1 0; do
  PG_UNION_WM=$wm EXP_REPS=1 timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_union_wm|k_umma|k_splitk" --csv \
    --log-file $O/phase_wm$wm.csv python tools/experiments/exp_union.py > /dev/null 2>&1
done
