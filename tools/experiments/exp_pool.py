"""mean_pool (bf16 token-major, 16 prompts x 2048 tokens) at n = 4096 and 11008:
us per call (CUDA graph of 10 calls) and GB/s; checks the result equals PG_POOL8=0's."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

P, T = 16, 2048
offs = [i * T for i in range(P + 1)]
st = torch.cuda.Stream()
for n in (4096, 11008):
    g = torch.Generator(device="cuda").manual_seed(n)
    X = torch.randn(P * T, n, device="cuda", generator=g).to(torch.bfloat16)
    with torch.cuda.stream(st):
        h = pg.mean_pool(X, layout="token", offsets=offs)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=st):
            for _ in range(10):
                pg.mean_pool(X, layout="token", offsets=offs)
        gr.replay()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(11)]
        ev[0].record(st)
        for i in range(10):
            gr.replay()
            ev[i + 1].record(st)
    st.synchronize()
    us = float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(10)])) / 10 * 1e3
    print(f"n={n}: {us:7.1f} us  {X.numel() * 2 / us / 1e3:7.1f} GB/s  h[0,:2]={h[0, :2].tolist()}", flush=True)
    np.save(f"/tmp/pool_{n}_{os.environ.get('PG_POOLV', 'd')}.npy", h.cpu().numpy())
