"""Config-3 arm alone (route + pack + grouped GEMMs, packed vs gathered B^T rows)."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

d = bench.config3_arm(None, 0, 1, 0)
print(json.dumps({k: d[k] for k in ("tokens_per_s", "gemm_tokens_per_s", "ms_per_layer", "route_ms", "pack_ms", "mode", "modes")}))
print(json.dumps(d["roofline"]), json.dumps(d["baselines"]))
