#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench, ncu launch list + full capture.
# usage: gpurun --timeout 1800 -- 'bash tools/gpu_round.sh TAG [kernel-regex]'
TAG=${1:-r1}
KRE=${2:-k_chain}
O=gpurun_out
mkdir -p $O
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?" >> $O/${TAG}_bench.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -k regex:$KRE -c 64 --csv \
  --log-file $O/${TAG}_launches.csv python bench.py --steps 64 --warmup 3 --prefill 0 --decode-batch 0 --cpu-steps 0 > $O/${TAG}_ncu1.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$KRE -s 20 -c 1 \
  -o $O/${TAG}_full -f python bench.py --steps 64 --warmup 3 --prefill 0 --decode-batch 0 --cpu-steps 0 > $O/${TAG}_ncu2.log 2>&1
tail -3 $O/${TAG}_pytest.log; tail -2 $O/${TAG}_smoke.log; cat $O/${TAG}_bench.json | head -c 3000
