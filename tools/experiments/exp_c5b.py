"""13B MLP block decode (config-5 shapes, world 1, ratio 0.4): per-linear
aggregated_forward launches vs the fused mlp_forward chain, CUDA graphs of 8 tokens."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
shapes = {"up": (13824, 5120), "gate": (13824, 5120), "down": (5120, 13824)}
dims = {nm: (pg.store_rank(pg.single_layer_k(m, n, 0.4), n), pg.single_layer_k(m, n, 0.4)) for nm, (m, n) in shapes.items()}
pats = pg.make_patterns(5151, 1, [dims[nm] for nm in shapes])[0]
aggs = {}
for j, (nm, (m, n)) in enumerate(shapes.items()):
    r, K = dims[nm]
    bt = (torch.randn(r, n, device=dev, generator=g) / n ** 0.5).to(torch.bfloat16)
    a = (torch.randn(m, r, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
    L = pg.FactorizedLayer.from_device(bt, a, K)
    aggs[nm] = pg.aggregate_layout(L, [pats[j]], 0.9)
xd = torch.randn(5120, device=dev).to(torch.bfloat16)
act = torch.empty(13824, device=dev, dtype=torch.bfloat16)
y = torch.empty(5120, device=dev, dtype=torch.bfloat16)
yl = {nm: torch.empty(m, device=dev, dtype=torch.bfloat16) for nm, (m, n) in shapes.items()}
xf = torch.randn(13824, device=dev).to(torch.bfloat16)
st = torch.cuda.Stream()
nbytes = sum(dims[nm][1] * (m + n) * 2 for nm, (m, n) in shapes.items())


def per_linear():
    for nm, (m, n) in shapes.items():
        pg.aggregated_forward(aggs[nm], 0, xf if n == 13824 else xd, out_dtype=torch.bfloat16, out=yl[nm])


def fused():
    pg.mlp_forward(aggs["up"], aggs["gate"], aggs["down"], 0, xd, out=y, act=act)


def timeit(fn, G=8, windows=20):
    with torch.cuda.stream(st):
        fn()
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for _ in range(G):
            fn()
    with torch.cuda.stream(st):
        for _ in range(3):
            gr.replay()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(windows + 1)]
        ev[0].record(st)
        for i in range(windows):
            gr.replay()
            ev[i + 1].record(st)
    st.synchronize()
    return float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(windows)])) / G * 1e3


for name, fn in (("per-linear", per_linear), ("fused mlp_forward", fused)):
    try:
        us = timeit(fn)
        print(f"{name:20s} {us:7.2f} us/token  {nbytes / us / 1e3:7.1f} GB/s  frac {nbytes / us / 1e3 / 6538:.3f}", flush=True)
    except Exception as e:  # noqa: BLE001
        print(name, "failed:", e)
