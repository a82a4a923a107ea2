python - <<'PY'
import sys, json, argparse
sys.argv = ["bench.py"]
import bench
args = argparse.Namespace(scaling="weak", layers=32, steps=5, warmup=3)
import torch; torch.cuda.set_device(0)
print(json.dumps(bench.config5_arm(args, 0, 1, 0), indent=1))
PY
