# prefill evidence: bench line (decode + config-3 prefill), ncu launch list and full capture of the grouped tcgen05 GEMM
O=gpurun_out; mkdir -p $O
TAG=${1:-r1b}
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err
P=16 T=2048 timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_umma -c 28 --csv --log-file $O/${TAG}_prefill_launches.csv python tools/experiments/exp_prefill.py > /dev/null 2>&1
P=16 T=2048 timeout 600 ncu --set full --import-source on --clock-control none -k regex:k_umma -s 4 -c 1 -o $O/${TAG}_umma -f python tools/experiments/exp_prefill.py > $O/${TAG}_umma.log 2>&1
head -c 2500 $O/${TAG}_bench.json; tail -2 $O/${TAG}_bench.err
