"""retrieve (N=1024 x d=4096 f64, config 2) device time: CUDA graph of 20 pg_retrieve calls."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402
from paper_2605_08568_b200 import _lib  # noqa: E402

N, D = 1024, 4096
g = torch.Generator(device="cuda").manual_seed(3)
emb = torch.randn((N, D), generator=g, device="cuda", dtype=torch.float64)
emb /= emb.norm(dim=1, keepdim=True)
cache = pg.PatternCache(D, N, 0.8)
cache.load([pg.CacheEntry(pg.PromptEmbedding(e), {}) for e in emb.cpu().numpy()])
q = emb[7] + 0.3 / D ** 0.5 * torch.randn(D, generator=g, device="cuda", dtype=torch.float64)
q /= q.norm()
entry = torch.empty(1, dtype=torch.int32, device="cuda")
hit = torch.empty(1, dtype=torch.int32, device="cuda")
st = torch.cuda.Stream()


def one():
    _lib.call("pg_retrieve", cache.handle, q.data_ptr(), 0, None, entry.data_ptr(), hit.data_ptr(), st.cuda_stream)


with torch.cuda.stream(st):
    one()
st.synchronize()
assert entry.item() == 7 and hit.item() == 1, (entry.item(), hit.item())
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=st):
    for _ in range(20):
        one()
with torch.cuda.stream(st):
    gr.replay()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(10):
        gr.replay()
    e1.record(st)
st.synchronize()
us = e0.elapsed_time(e1) / 200 * 1e3
print(f"retrieve {us:.2f} us per call (graph), scan floor {8 * N * D / 6538e3:.2f} us, frac {8 * N * D / (us * 1e-6) / 1e9 / 6538:.3f}")
