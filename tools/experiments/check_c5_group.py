"""Config-5 prefill grouping check: prefill_batched over [q, k, v] (x replicated)
equals per-linear aggregated_forward_batched (bit-for-bit expected: same GEMM
kernels and tiles per job)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(3)
T, n, m = 256, 5120, 5120
K = pg.single_layer_k(m, n, 0.4)
r = pg.store_rank(K, n)
pats = pg.make_patterns(5151, 1, [(r, K)] * 3)[0]
aggs = []
for i in range(3):
    bt = (torch.randn(r, n, device=dev, generator=g) / n ** 0.5).to(torch.bfloat16)
    a = (torch.randn(m, r, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
    aggs.append(pg.aggregate_layout(pg.FactorizedLayer.from_device(bt, a, K), [pats[i]], 0.9))
x = torch.randn(T, n, device=dev, generator=g).to(torch.bfloat16)
ys = [pg.aggregated_forward_batched(a, [0], [0, T], x, out_dtype=torch.float32) for a in aggs]
yg = pg.prefill_batched(aggs, [0, T, 2 * T, 3 * T], x.repeat(3, 1), out_dtype=torch.float32)
for i in range(3):
    d = (yg[i * T:(i + 1) * T] - ys[i]).abs().max().item() / ys[i].abs().max().item()
    print(f"linear {i}: max rel diff grouped vs single {d:.3e}", flush=True)
    assert d <= 1e-2
print("group check ok")
