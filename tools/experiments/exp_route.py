"""Config-3 routing experiment: 7 routers (q,k,v,o,gate,up,down) x 16 prompts
x 2048 tokens, token-major bf16 activations, exact selection on device."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

D, FF, RATIO = 4096, 11008, 0.6
P, T = int(os.environ.get("P", 16)), int(os.environ.get("T", 2048))
dev = torch.device("cuda", 0)
lin = {"q": (D, D), "k": (D, D), "v": (D, D), "o": (D, D), "up": (FF, D), "gate": (FF, D), "down": (D, FF)}
g = torch.Generator(device=dev).manual_seed(7)
X = torch.randn(P * T, D, device=dev, generator=g).to(torch.bfloat16)
X2 = torch.randn(P * T, FF, device=dev, generator=g).to(torch.bfloat16)
offs = [i * T for i in range(P + 1)]
routers, Ks = {}, {}
for nm, (m, n) in lin.items():
    K = pg.single_layer_k(m, n, RATIO)
    r = pg.store_rank(K, min(m, n))
    routers[nm] = pg.RouterParams(torch.randn((r, n), generator=g, device=dev, dtype=torch.float64))
    Ks[nm] = K


def step():
    for nm in lin:
        pg.route_select(routers[nm], X2 if nm == "down" else X, Ks[nm], layout="token", offsets=offs)


for _ in range(2):
    step()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5):
    step()
e1.record()
torch.cuda.synchronize()
print(f"routing P={P} T={T}: {e0.elapsed_time(e1) / 5:.3f} ms per layer (7 routers)")
