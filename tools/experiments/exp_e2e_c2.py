"""Config-2 e2e step I/O: copy kernels (pg_copy_io before/after the k_chain launch)
vs zero-copy (k_chain reads x from / writes y to pinned host memory)."""
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
        a = (torch.randn((m, r), generator=gg, device="cuda") / m ** 0.5).to(torch.bfloat16)
        b.append(pg.aggregate_layout(pg.FactorizedLayer.from_device(bt, a, K), [pats[i]], 0.9))
    blocks.append(b)
xs = torch.randn((G, D), device="cuda").to(torch.bfloat16)
y = torch.empty((G, D), device="cuda")
act = torch.empty((G, F), device="cuda", dtype=torch.bfloat16)
x_host = xs.cpu().pin_memory()
y_host = torch.empty((G, D), dtype=torch.float32).pin_memory()
st = torch.cuda.Stream()


def copies():
    for i in range(G):
        u, g, d = blocks[i % R]
        pg.copy_io(xs[i], x_host[i])
        pg.mlp_forward(u, g, d, 0, xs[i], out=y[i], act=act[i])
        pg.copy_io(y_host[i], y[i])


def zero_copy():
    for i in range(G):
        u, g, d = blocks[i % R]
        pg.mlp_forward(u, g, d, 0, x_host[i], out=y_host[i], act=act[i])


def device_only():
    for i in range(G):
        u, g, d = blocks[i % R]
        pg.mlp_forward(u, g, d, 0, xs[i], out=y[i], act=act[i])


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


for name, fn in (("device only", device_only), ("copy kernels", copies), ("zero-copy", zero_copy)):
    print(f"{name:14s} {timeit(fn):6.2f} us/step", flush=True)
zero_copy()
torch.cuda.synchronize()
ref = y_host.clone()
copies()
torch.cuda.synchronize()
print("zero-copy == copies:", torch.equal(ref, y_host))
