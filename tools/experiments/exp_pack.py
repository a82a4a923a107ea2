"""Device pack timing (config-3 shapes): pack_selected for the 7 linears of a layer, 16 prompts."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402
LIN = {"q": (4096, 4096), "k": (4096, 4096), "v": (4096, 4096), "o": (4096, 4096),
       "up": (11008, 4096), "gate": (11008, 4096), "down": (4096, 11008)}
P = 16
lay, sels, byt = {}, {}, 0
for nm, (m, n) in LIN.items():
    K = pg.single_layer_k(m, n, 0.6); r = pg.store_rank(K, min(m, n))
    bt = torch.randn(r, n, device="cuda").to(torch.bfloat16); a = torch.randn(m, r, device="cuda").to(torch.bfloat16)
    lay[nm] = pg.FactorizedLayer.from_device(bt, a, K)
    sels[nm] = torch.stack([torch.sort(torch.randperm(r, device="cuda")[:K])[0] for _ in range(P)]).to(torch.int32)
    byt += P * ((K + 7) // 8 * 8) * (m + n) * 2
for _ in range(2):
    packs = {nm: pg.pack_selected(lay[nm], sels[nm]) for nm in LIN}
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    packs = {nm: pg.pack_selected(lay[nm], sels[nm]) for nm in LIN}
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"pack per layer {ms:.3f} ms, written {byt/1e9:.2f} GB -> {byt/ms/1e6:.0f} GB/s")
