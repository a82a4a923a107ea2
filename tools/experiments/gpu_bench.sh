O=gpurun_out; mkdir -p $O
TAG=${1:-rb}
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py > $O/${TAG}_bench.json 2> $O/${TAG}_bench.err; echo "bench rc=$?"
python - <<PY
import json; d=json.load(open("$O/${TAG}_bench.json"))
print("value", d["value"], "e2e", d["e2e"]["value"], "frac", d["roofline"]["frac"], "us", d["ms_per_step"]*1e3)
print("prefill", {k: d["prefill"][k] for k in ("tokens_per_s","gemm_tokens_per_s","ms_per_layer","route_ms")}, d["prefill"]["roofline"]["frac"])
print("cpu", d.get("cpu_baseline"), "clocks", d["clocks"])
PY
