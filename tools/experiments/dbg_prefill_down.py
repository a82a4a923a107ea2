"""Debug: config-3 down-shape prefill error vs f64/fp32 references."""
import os, sys
import numpy as np, torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg
m, n = int(os.environ.get("M", 4096)), int(os.environ.get("N", 11008)); P, T = 4, 2048
K = pg.single_layer_k(m, n, 0.6); r = pg.store_rank(K, min(m, n))
rng = np.random.default_rng(m + n)
sig = 1.0 / (1.0 + np.arange(r) / 64.0)
A = rng.standard_normal((m, r)) * sig / np.sqrt(m); B = rng.standard_normal((n, r)) / np.sqrt(n)
theta = rng.standard_normal((r, n))
L = pg.FactorizedLayer(A, B, K, dtype="bf16"); router = pg.RouterParams(theta)
X = torch.randn(P * T, n, device="cuda")
X += torch.randn(P, 1, n, device="cuda").repeat_interleave(T, 0).reshape(P * T, n) * 0.5
X = X.to(torch.bfloat16); offs = [p * T for p in range(P + 1)]
sel = pg.route_select_pooled(router, pg.mean_pool(X, layout="token", offsets=offs), K)
sels = sel.cpu().numpy()
aggs = [pg.aggregate_layout(L, [pg.RankSelection(s)], 0.9) for s in sels.astype(np.uint32)]
y1 = pg.prefill_batched(aggs, offs, X, out_dtype=torch.float32)
y2 = pg.prefill_packed(pg.pack_selected(L, sel), offs, X, out_dtype=torch.float32)
Ab = torch.from_numpy(A).to(torch.bfloat16).double().cuda(); Bb = torch.from_numpy(B).to(torch.bfloat16).double().cuda()
for p in range(P):
    s = torch.from_numpy(sels[p].astype(np.int64)).cuda()
    xp = X[p * T:(p + 1) * T].double()
    z64 = xp @ Bb[:, s]
    zb = z64.to(torch.bfloat16).double()
    ref = zb @ Ab[:, s].t()
    ref_nor = z64 @ Ab[:, s].t()
    d = ref.abs().max().item()
    for nm, y in (("batched", y1), ("packed", y2)):
        e = (y[p * T:(p + 1) * T].double() - ref).abs()
        i = int(e.argmax()); t, c = divmod(i, m)
        print(f"p{p} {nm}: rel {e.max().item()/d:.2e} at tok {t} col {c}; vs unrounded-z ref {((y[p*T:(p+1)*T].double()-ref_nor).abs().max().item()/d):.2e}; |z| max {z64.abs().max().item():.2f}")
    print(f"   bf16-rounding effect alone {(ref - ref_nor).abs().max().item()/d:.2e}")
