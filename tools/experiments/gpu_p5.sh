timeout 300 python -m pytest tests/test_gpu_union_prog.py -x -q 2>&1 | grep -E "passed|failed|^E  .*assert|^FAILED" | head -6
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" 2>&1 | tail -2
PG_PROG_DBG=1 timeout 200 python tools/experiments/exp_prog.py 2 2>&1 | tail -10
timeout 600 python bench.py --secondary 0 --cpu 0 > gpurun_out/p5_bench.json 2> gpurun_out/p5_bench.err; tail -2 gpurun_out/p5_bench.err
python - <<'PY'
import json; d=json.load(open("gpurun_out/p5_bench.json"))
print("value", d["value"], "ms", d["ms_per_step"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], d["roofline"]["dominant_launch"], d["launches_per_step"], d["clocks"])
PY
