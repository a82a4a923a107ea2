"""Config-3 pack + GEMMs: sequential vs the pack of linear L+1 on a side stream
overlapping the GEMMs of linear L (events; selections routed once)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2605_08568_b200 as pg  # noqa: E402

P, T = 16, 2048
dev = torch.device("cuda", 0)
g = torch.Generator(device=dev).manual_seed(7)
X = torch.randn(P * T, bench.D_MODEL, device=dev, generator=g).to(torch.bfloat16)
X2 = torch.randn(P * T, bench.D_FF, device=dev, generator=g).to(torch.bfloat16)
offs = [i * T for i in range(P + 1)]
layers, sels, outs = {}, {}, {}
for nm, (m, n) in bench.LIN.items():
    r, K = bench.dims(m, n)
    bt = (torch.randn((r, n), generator=g, device=dev) / n ** 0.5).to(torch.bfloat16)
    a = (torch.randn((m, r), generator=g, device=dev) / m ** 0.5).to(torch.bfloat16)
    layers[nm] = (pg.FactorizedLayer.from_device(bt, a, K), K)
    sels[nm] = torch.stack([torch.randperm(r, device=dev)[:K].sort().values for _ in range(P)]).to(torch.int32)
    outs[nm] = torch.empty(P * T, m, device=dev, dtype=torch.bfloat16)
src = {nm: (X2 if nm == "down" else X) for nm in bench.LIN}
bufs = {}
ps = torch.cuda.Stream(device=dev)


def seq():
    for nm in bench.LIN:
        bufs[nm] = pg.pack_selected(layers[nm][0], sels[nm], into=bufs.get(nm))
    for nm in bench.LIN:
        pg.prefill_packed(bufs[nm], offs, src[nm], out_dtype=torch.bfloat16, out=outs[nm])


def overlap():
    cur = torch.cuda.current_stream(dev)
    ps.wait_stream(cur)  # the previous pass's GEMMs are done with the buffers
    evs = {}
    with torch.cuda.stream(ps):
        for nm in bench.LIN:
            bufs[nm] = pg.pack_selected(layers[nm][0], sels[nm], into=bufs.get(nm))
            evs[nm] = torch.cuda.Event()
            evs[nm].record(ps)
    for nm in bench.LIN:
        cur.wait_event(evs[nm])
        pg.prefill_packed(bufs[nm], offs, src[nm], out_dtype=torch.bfloat16, out=outs[nm])


def timeit(fn, reps=5):
    for _ in range(2):
        fn()
    torch.cuda.synchronize()
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
    ev[0].record()
    for i in range(reps):
        fn()
        ev[i + 1].record()
    torch.cuda.synchronize()
    return float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]))


ref = None
for name, fn in (("sequential", seq), ("overlapped", overlap), ("sequential", seq), ("overlapped", overlap)):
    ms = timeit(fn)
    y = outs["down"].clone()
    if ref is None:
        ref = y
    print(f"{name:12s} pack + GEMMs {ms:.3f} ms/layer  same={bool(torch.equal(y, ref))}", flush=True)
