"""Device pack (K3 for routed prefill batches): 16 prompts' selected experts of each
config-3 linear, timed per linear with reused buffers; bytes moved vs HBM."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

P = 16
LIN = {"q": (4096, 4096), "up": (11008, 4096), "down": (4096, 11008)}
g = torch.Generator(device="cuda").manual_seed(0)
tot_ms = tot_b = 0.0
for nm, (m, n) in LIN.items():
    K = pg.single_layer_k(m, n, 0.6)
    r = pg.store_rank(K, min(m, n))
    bt = (torch.randn((r, n), generator=g, device="cuda")).to(torch.bfloat16)
    a = (torch.randn((m, r), generator=g, device="cuda")).to(torch.bfloat16)
    L = pg.FactorizedLayer.from_device(bt, a, K)
    sel = torch.stack([torch.sort(torch.randperm(r, generator=torch.Generator().manual_seed(p))[:K]).values
                       for p in range(P)]).to(torch.int32).cuda()
    pk = pg.pack_selected(L, sel)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(10):
        pg.pack_selected(L, sel, into=pk)
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 10
    kp = (K + 7) // 8 * 8
    b = P * K * n * 2 + m * r * 2 + P * kp * (n + m) * 2
    tot_ms += ms * (4 if nm == "q" else (2 if nm == "up" else 1))
    tot_b += b * (4 if nm == "q" else (2 if nm == "up" else 1))
    print(f"{nm:5s} {ms * 1e3:8.1f} us  {b / 1e6:8.1f} MB  {b / (ms * 1e-3) / 1e9:7.0f} GB/s")
print(f"layer (4 q-type, 2 up-type, 1 down): {tot_ms:.3f} ms, {tot_b / 1e9:.2f} GB, {tot_b / (tot_ms * 1e-3) / 1e9:.0f} GB/s")
