"""Config-3 routing as the bench runs it (3 pooled inputs, 7 routers, 16 prompts
x 2048 tokens): eager wall time per routing pass, and (under ncu) the kernels."""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402

D, FF, RATIO, P, T = 4096, 11008, 0.6, 16, 2048
dev = torch.device("cuda", 0)
lin = {"q": (D, D), "k": (D, D), "v": (D, D), "o": (D, D), "up": (FF, D), "gate": (FF, D), "down": (D, FF)}
g = torch.Generator(device=dev).manual_seed(7)
X = torch.randn(P * T, D, device=dev, generator=g).to(torch.bfloat16)
X2 = torch.randn(P * T, FF, device=dev, generator=g).to(torch.bfloat16)
Xo = torch.randn(P * T, D, device=dev, generator=g).to(torch.bfloat16)
offs = [i * T for i in range(P + 1)]
routers, Ks = {}, {}
for nm, (m, n) in lin.items():
    K = pg.single_layer_k(m, n, RATIO)
    routers[nm] = pg.RouterParams(torch.randn((pg.store_rank(K, min(m, n)), n), generator=g, device=dev,
                                              dtype=torch.float64))
    Ks[nm] = K
src = {"q": X, "k": X, "v": X, "up": X, "gate": X, "o": Xo, "down": X2}


def route_all():
    pooled = {id(x): pg.mean_pool(x, layout="token", offsets=offs) for x in (X, Xo, X2)}
    return {nm: pg.route_select_pooled(routers[nm], pooled[id(src[nm])], Ks[nm]) for nm in lin}


for _ in range(3):
    route_all()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
t0 = time.perf_counter()
e0.record()
for _ in range(5):
    route_all()
e1.record()
torch.cuda.synchronize()
print(f"routing: {e0.elapsed_time(e1) / 5:.3f} ms (events), host {(time.perf_counter() - t0) / 5 * 1e3:.3f} ms")
