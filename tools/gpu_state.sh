#!/bin/bash
# One gpurun call: GPU tests, smoke, default bench (JSON line) + the reference arm.
O=gpurun_out; mkdir -p $O; TAG=${1:-s}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv > $O/${TAG}_smi.txt 2>&1
timeout 1200 python -m pytest tests -m gpu -x -q > $O/${TAG}_pytest.log 2>&1; echo "pytest rc=$?" >> $O/${TAG}_pytest.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/${TAG}_smoke.log 2>&1; echo "smoke rc=$?" >> $O/${TAG}_smoke.log
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?" >> $O/${TAG}_bench.err
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/${TAG}_ref.json 2> $O/${TAG}_ref.err; echo "ref rc=$?" >> $O/${TAG}_ref.err
tail -3 $O/${TAG}_pytest.log; tail -2 $O/${TAG}_smoke.log; tail -2 $O/${TAG}_bench.err; head -c 2500 $O/${TAG}_bench.json; cat $O/${TAG}_ref.json
