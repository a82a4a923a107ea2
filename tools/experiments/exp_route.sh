O=gpurun_out; mkdir -p $O
timeout 900 python -m pytest tests -m gpu -x -q -k "route or score or select or provider or pool" 2>&1 | tail -3 > $O/er.txt
timeout 300 python tools/experiments/exp_route.py >> $O/er.txt 2>&1
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"k_mean|k_score|k_route|k_hnorm" -c 8 python tools/experiments/exp_route.py > $O/er_ncu.txt 2>&1
cat $O/er.txt; grep -E "^\s+(void )?pg::|^\s+k_|gpu__time" $O/er_ncu.txt | sed 's/(.*//' | paste - - | awk '{print $1, $2, $NF}'
