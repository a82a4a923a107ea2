"""Config-2 MLP block decode step (one launch per block, 4 weight replicas, 64-step
graph, median of 20 windows) and the single-linear up / down launches; the env
switches of the decode chain (PG_CHAIN_*) select the variant."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

D, F, G, R = 4096, 11008, 64, 4
K = pg.single_layer_k(F, D, 0.6)
r = pg.store_rank(K, D)
pats = pg.make_patterns(17171, 1, [(r, K)] * 3)[0]
blocks = []
for j in range(R):
    gg = torch.Generator(device="cuda").manual_seed(100 + j)
    b = []
    for i, (m, n) in enumerate(((F, D), (F, D), (D, F))):
        bt = (torch.randn((r, n), generator=gg, device="cuda") / n ** 0.5).to(torch.bfloat16)
        sig = 1.0 / (1.0 + torch.arange(r, device="cuda", dtype=torch.float32) / 64.0)
        a = (torch.randn((m, r), generator=gg, device="cuda") * sig / m ** 0.5 * 8).to(torch.bfloat16)
        L = pg.FactorizedLayer.from_device(bt, a, K)
        b.append(pg.aggregate_layout(L, [pats[i]], 0.9))
    blocks.append(tuple(b))
xs = torch.randn((G, D), device="cuda").to(torch.bfloat16)
ys = torch.empty((G, D), device="cuda", dtype=torch.bfloat16)
acts = (torch.randn((G, F), device="cuda") * 0.1).to(torch.bfloat16)
ups = torch.empty((G, F), device="cuda")
st = torch.cuda.Stream()


def mlp():
    for i in range(G):
        u, g, d = blocks[i % R]
        pg.mlp_forward(u, g, d, 0, xs[i], out=ys[i], act=acts[i], out_dtype=torch.bfloat16)


def up():
    for i in range(G):
        pg.aggregated_forward(blocks[i % R][0], 0, xs[i], out=ups[i])


def down():
    for i in range(G):
        pg.aggregated_forward(blocks[i % R][2], 0, acts[i], out=ys[i])


def timeit(fn, windows=20):
    with torch.cuda.stream(st):
        fn()
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
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


tag = " ".join(f"{k}={v}" for k, v in sorted(os.environ.items()) if k.startswith("PG_CHAIN"))
bl = K * (F + D) * 2
res = {nm: timeit(fn) for nm, fn in (("mlp", mlp), ("up", up), ("down", down))}
print(f"[{tag}] mlp {res['mlp']:.2f} us ({3 * bl / res['mlp'] / 1e3 / 6538:.3f})  up {res['up']:.2f}  down {res['down']:.2f}",
      flush=True)
