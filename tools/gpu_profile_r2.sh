#!/bin/bash
# Round-2 evidence: bench line, ncu launch list + one full capture of the config-4 step kernel (k_union_prog)
O=gpurun_out; mkdir -p $O; TAG=${1:-r2b}
for i in 1 2; do timeout 400 python -m pytest tests/test_gpu_prefill.py tests/test_gpu_prefill_routed.py tests/test_gpu_union_prog.py -q 2>&1 | grep -E "^E  .*(assert|Error)|FAILED|passed|failed" | head -8; done
timeout 900 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:k_union_prog -c 4 --csv \
  --log-file $O/${TAG}_launches.csv env PG_PROG_COOP=0 python bench.py --steps 2 --warmup 3 --secondary 0 --cpu 0 > $O/${TAG}_ncu1.log 2>&1; echo "ncu1 rc=$?"
timeout 1200 ncu --set full --clock-control none --import-source on -k regex:k_union_prog -s 3 -c 1 \
  -o $O/${TAG}_prog -f env PG_PROG_COOP=0 python bench.py --steps 2 --warmup 3 --secondary 0 --cpu 0 > $O/${TAG}_ncu2.log 2>&1; echo "ncu2 rc=$?"
ls -la $O/${TAG}_*
