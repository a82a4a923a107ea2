"""Per-CTA k_chain timeline for the config-2 MLP step (PG_CHAIN_DBG=1).
Prints median / max over CTAs of each stamp relative to the earliest start."""
import ctypes as C
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
os.environ["PG_CHAIN_DBG"] = "1"
import paper_2605_08568_b200 as pg  # noqa: E402
from paper_2605_08568_b200 import _lib  # noqa: E402

D, F = 4096, 11008
K = pg.single_layer_k(F, D, 0.6)
r = pg.store_rank(K, D)
pats = pg.make_patterns(17171, 1, [(r, K)] * 3)[0]
gg = torch.Generator(device="cuda").manual_seed(1)
aggs = []
for i, (m, n) in enumerate(((F, D), (F, D), (D, F))):
    bt = (torch.randn((r, n), generator=gg, device="cuda") / n ** 0.5).to(torch.bfloat16)
    a = (torch.randn((m, r), generator=gg, device="cuda") / m ** 0.5).to(torch.bfloat16)
    aggs.append(pg.aggregate_layout(pg.FactorizedLayer.from_device(bt, a, K), [pats[i]], 0.9))
x = torch.randn(D, device="cuda").to(torch.bfloat16)
y = torch.empty(D, device="cuda")
for _ in range(20):
    pg.mlp_forward(*aggs, 0, x, out=y)
torch.cuda.synchronize()
buf = (C.c_uint64 * (1024 * 16))()
_lib.call("pg_chain_debug_dump", buf, 1024 * 16)
a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16).astype(np.int64)
a = a[a[:, 0] > 0]
t0 = a[:, 0].min()
names = {0: "start", 6: "x staged", 1: "ph0 start", 2: "ph0 s1 done", 4: "ph0 z staged", 5: "ph0 s2 done",
         7: "ph1 start", 14: "ph1 s1 data", 8: "ph1 s1 done", 10: "ph1 z staged", 11: "ph1 s2 done",
         12: "producer done", 13: "end", 15: "ph1 s2 data"}
print(f"CTAs {a.shape[0]}")
for k in (0, 6, 1, 2, 4, 5, 7, 14, 8, 10, 15, 11, 12, 13):
    v = a[:, k]
    v = (v[v > 0] - t0) / 1e3
    if v.size:
        print(f"{k:2d} {names[k]:16s} med {np.median(v):7.2f}  min {v.min():7.2f}  max {v.max():7.2f}")
