"""13B q/k/v/o decode (config-5 shapes, world 1, ratio 0.4): the fused q/k/v
module launch and the o launch timed alone (R weight replicas rotated so the
working set exceeds L2), CUDA graphs of 8 launches, median of 20 windows."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(5)
R = int(os.environ.get("EXP_R", "8"))
# EXP_SHAPE="m n ratio": other shapes (e.g. "4096 4096 0.6" for 7B q/k/v, "11008 4096 0.6" for up/gate)
m, n, ratio = (5120, 5120, 0.4) if not os.environ.get("EXP_SHAPE") else \
    (int(os.environ["EXP_SHAPE"].split()[0]), int(os.environ["EXP_SHAPE"].split()[1]),
     float(os.environ["EXP_SHAPE"].split()[2]))
K = pg.single_layer_k(m, n, ratio)
r = pg.store_rank(K, n)
pats = pg.make_patterns(5151, 1, [(r, K)] * 4)[0]
reps = []
for j in range(R):
    aggs = []
    for i in range(4):
        bt = (torch.randn(r, n, device=dev, generator=g) / n ** 0.5).to(torch.bfloat16)
        a = (torch.randn(m, r, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
        aggs.append(pg.aggregate_layout(pg.FactorizedLayer.from_device(bt, a, K), [pats[i]], 0.9))
    reps.append(aggs)
xd = torch.randn(n, device=dev).to(torch.bfloat16)
ys = [torch.empty(m, device=dev) for _ in range(4)]
st = torch.cuda.Stream()
lin_bytes = K * (m + n) * 2


def qkv(i):
    pg.module_forward(reps[i % R][:3], 0, xd, out_dtype=torch.float32, outs=ys[:3])


def o(i):
    pg.aggregated_forward(reps[i % R][3], 0, xd, out_dtype=torch.float32, out=ys[3])


def token(i):
    qkv(i)
    o(i)


def timeit(fn, G=8, windows=20):
    with torch.cuda.stream(st):
        for i in range(G):
            fn(i)
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        for i in range(G):
            fn(i)
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
def mod2(i):
    pg.module_forward(reps[i % R][:2], 0, xd, out_dtype=torch.float32, outs=ys[:2])


for name, fn, nb in (("qkv module", qkv, 3 * lin_bytes), ("2-lin module", mod2, 2 * lin_bytes), ("o", o, lin_bytes),
                     ("qkv + o", token, 4 * lin_bytes)):
    if os.environ.get("EXP_ONLY") and name != os.environ["EXP_ONLY"]:
        continue
    us = timeit(fn)
    print(f"[{tag} {m}x{n}] {name:12s} {us:7.2f} us  {nb / us / 1e3:7.1f} GB/s  frac {nb / us / 1e3 / 6538:.3f}", flush=True)

if os.environ.get("PG_CHAIN_DBG"):  # per-CTA stamps of the last launch (o): us from the earliest CTA start
    import ctypes as C
    from paper_2605_08568_b200 import _lib
    with torch.cuda.stream(st):
        o(0)
    st.synchronize()
    buf = (C.c_uint64 * (1024 * 16))()
    _lib.call("pg_chain_debug_dump", buf, 1024 * 16)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16)[:148].astype(np.int64)
    t0 = a[:, 0].min()
    for k in range(16):
        col = a[:, k]
        if (col > 0).all():
            print(f"stamp {k:2d} min {(col.min() - t0) / 1e3:7.2f} med {(np.median(col) - t0) / 1e3:7.2f} "
                  f"max {(col.max() - t0) / 1e3:7.2f} us")
