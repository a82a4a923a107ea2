"""Config-5 arm alone (13B layer, expert-sharded, world 1): prints its JSON object."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402

print(json.dumps(bench.config5_arm(None, 0, 1, 0)))
