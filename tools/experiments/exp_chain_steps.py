"""Config-2 MLP block decode: one launch per block (independent x per step, the
round-1 bench) vs chains of blocks (x_{s+1} = y_s) with up to 8 blocks per launch."""
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
acts = torch.empty((G, F), device="cuda", dtype=torch.bfloat16)
st = torch.cuda.Stream()


def indep():
    for i in range(G):
        u, g, d = blocks[i % R]
        pg.mlp_forward(u, g, d, 0, xs[i], out=ys[i], act=acts[i], out_dtype=torch.bfloat16)


def chained(per):
    chain = [blocks[i % R] for i in range(G)]
    for s0 in range(0, G, per):
        pg.mlp_forward_chain(chain[s0:s0 + per], xs[0] if s0 == 0 else ys[s0 - 1],
                             outs=[ys[i] for i in range(s0, s0 + per)], acts=[acts[i] for i in range(s0, s0 + per)])


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


bytes_step = 3 * K * (F + D) * 2
for name, fn in [("independent (1 launch/block)", indep)] + [(f"chain {p}/launch", (lambda p=p: chained(p))) for p in (1, 2, 4, 8)]:
    us = timeit(fn)
    print(f"{name:32s} {us:6.2f} us/block  {bytes_step / us / 1e3:7.1f} GB/s  frac {bytes_step / us / 1e3 / 6538:.3f}", flush=True)
print("y finite:", bool(torch.isfinite(ys.float()).all()), float(ys.float().abs().max()))
