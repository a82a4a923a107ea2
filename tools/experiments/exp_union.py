"""Config-4 layer step through the union-masked path: 7 linears of a LLaMA-7B
decoder layer, 256 decode tokens from 256 prompts with their own selections
(reference pattern generator), weights read once per layer.  Prints us per
layer, HBM GB/s on the stored bytes and TFLOP/s on the masked-union flops."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402
from oracle import pyoracle  # noqa: E402

SH = {"q": (4096, 4096), "k": (4096, 4096), "v": (4096, 4096), "o": (4096, 4096),
      "up": (11008, 4096), "gate": (11008, 4096), "down": (4096, 11008)}
if os.environ.get("EXP_ONLY"):
    SH = {k: v for k, v in SH.items() if k in os.environ["EXP_ONLY"].split(",")}


def main():
    P = T = int(os.environ.get("EXP_T", "256"))
    dev = torch.device("cuda")
    lays, batches, xs = {}, {}, {}
    dims = [(pg.store_rank(pg.single_layer_k(m, n, 0.6), n), pg.single_layer_k(m, n, 0.6)) for m, n in SH.values()]
    pats = pyoracle.make_patterns(17171, P, dims)
    for li, (nm, (m, n)) in enumerate(SH.items()):
        r, K = dims[li]
        bt = (torch.randn(r, n, device=dev) / n ** 0.5).to(torch.bfloat16)
        a = (torch.randn(m, r, device=dev) / m ** 0.5).to(torch.bfloat16)
        lays[nm] = pg.FactorizedLayer.from_device(bt, a, K, layer_id=nm)
        batches[nm] = pg.SelectionBatch(lays[nm], [pg.RankSelection(p[li]) for p in pats])
        xs[nm] = torch.randn(T, n, device=dev).to(torch.bfloat16)
    tp = torch.arange(T, device=dev, dtype=torch.int32) % P
    ys = {nm: torch.empty(T, m, device=dev, dtype=torch.bfloat16) for nm, (m, n) in SH.items()}

    def layer():
        if os.environ.get("EXP_GROUP", "1") == "1" and not os.environ.get("EXP_ONLY"):
            for grp in (("q", "k", "v"), ("o",), ("up", "gate"), ("down",)):
                pg.module_forward_union([lays[g] for g in grp], [batches[g] for g in grp], tp, xs[grp[0]],
                                        out_dtype=torch.bfloat16, outs=[ys[g] for g in grp])
            return
        for nm in SH:
            pg.masked_forward_union(lays[nm], batches[nm], tp, xs[nm], out_dtype=torch.bfloat16, out=ys[nm])

    reps = int(os.environ.get("EXP_REPS", "20"))

    def graph_us(fn):  # device time of fn replayed as a CUDA graph (no host launch cost)
        st = torch.cuda.Stream()
        with torch.cuda.stream(st):
            for _ in range(3):
                fn()
        st.synchronize()
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=st):
            fn()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(st):
            g.replay()
            e0.record(st)
            for _ in range(reps):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / reps * 1e3

    us = graph_us(layer)
    byt = sum(dims[i][0] * (m + n) * 2 for i, (m, n) in enumerate(SH.values()))
    fl = 2 * T * sum(dims[i][0] * (m + n) for i, (m, n) in enumerate(SH.values()))
    print(f"T={T} P={P}: {us:.1f} us/layer  {byt / us / 1e3:.0f} GB/s  {fl / us / 1e6:.0f} TFLOP/s  "
          f"-> {T / (32 * us * 1e-6):.0f} tok/s for a 32-layer stack")
    for nm in SH:  # per linear
        t = graph_us(lambda: pg.masked_forward_union(lays[nm], batches[nm], tp, xs[nm], out_dtype=torch.bfloat16,
                                                     out=ys[nm]))
        print(f"  {nm:5s} {t:7.1f} us")


if __name__ == "__main__":
    main()
