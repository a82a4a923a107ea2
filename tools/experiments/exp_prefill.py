"""Config-3 prefill experiment: one LLaMA-7B decoder layer's 7 rank-expert
linears, 16 prompts x 2048 tokens, each prompt with its own expert subset,
bf16, grouped tcgen05 GEMMs.  Prints ms, tokens/s and TFLOP/s."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

D, FF, RATIO = 4096, 11008, 0.6
P, T = int(os.environ.get("P", 16)), int(os.environ.get("T", 2048))
dev = torch.device("cuda", 0)
lin = {"q": (D, D), "k": (D, D), "v": (D, D), "o": (D, D), "up": (FF, D), "gate": (FF, D), "down": (D, FF)}
g = torch.Generator(device=dev).manual_seed(0)
aggs, flops = {}, 0
for name, (m, n) in lin.items():
    K = pg.single_layer_k(m, n, RATIO); r = pg.store_rank(K, min(m, n))
    bt = (torch.randn((r, n), generator=g, device=dev) / n ** 0.5).to(torch.bfloat16)
    a = (torch.randn((m, r), generator=g, device=dev) / m ** 0.5).to(torch.bfloat16)
    L = pg.FactorizedLayer.from_device(bt, a, K)
    pats = pg.make_patterns(17 + len(aggs), P, [(r, K)])
    aggs[name] = ([pg.aggregate_layout(L, [p[0]], 0.9) for p in pats], L)
    flops += 2 * P * T * K * (m + n)
offs = [i * T for i in range(P + 1)]
X = torch.randn(P * T, D, device=dev).to(torch.bfloat16)
X2 = torch.randn(P * T, FF, device=dev).to(torch.bfloat16)
outs = {nm: torch.empty(P * T, m, device=dev, dtype=torch.bfloat16) for nm, (m, n) in lin.items()}


def step():
    for nm, (m, n) in lin.items():
        pg.prefill_batched(aggs[nm][0], offs, X2 if nm == "down" else X, out_dtype=torch.bfloat16, out=outs[nm])


for _ in range(2):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
reps = 5
e0.record()
for _ in range(reps):
    step()
e1.record()
torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / reps
print(f"prefill P={P} T={T}: {ms:.3f} ms/layer, {P * T / ms * 1e3:.0f} tokens/s, "
      f"{flops / ms / 1e9:.0f} TFLOP/s ({flops / 1e12:.3f} TFLOP)")
# per-linear breakdown
for nm, (m, n) in lin.items():
    e0.record()
    for _ in range(reps):
        pg.prefill_batched(aggs[nm][0], offs, X2 if nm == "down" else X, out_dtype=torch.bfloat16, out=outs[nm])
    e1.record()
    torch.cuda.synchronize()
    K = pg.single_layer_k(m, n, RATIO)
    f = 2 * P * T * K * (m + n)
    t = e0.elapsed_time(e1) / reps
    print(f"  {nm:5s} {t:7.3f} ms  {f / t / 1e9:6.0f} TFLOP/s")
