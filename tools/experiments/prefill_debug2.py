import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg

m, n, r, K = 1000, 4096, 1664, 832
A = np.random.default_rng(1).standard_normal((m, r)) / np.sqrt(m)
B = np.random.default_rng(2).standard_normal((n, r)) / np.sqrt(n)
sel = np.sort(np.random.default_rng(3).choice(r, K, replace=False)).astype(np.uint32)
L = pg.FactorizedLayer(A, B, K, dtype="bf16")
Ab = torch.from_numpy(np.ascontiguousarray(A[:, sel])).to(torch.bfloat16).cuda()
Bb = torch.from_numpy(np.ascontiguousarray(B[:, sel])).to(torch.bfloat16).cuda()
g = pg.aggregate_layout(L, [pg.RankSelection(sel)], 0.9)
for T in (16, 200):
    x = torch.randn(T, n, device="cuda").to(torch.bfloat16)
    ref = ((x.float() @ Bb.float()).to(torch.bfloat16).float() @ Ab.float().t())
    for name, y in (("masked", pg.masked_forward(L, pg.RankSelection(sel), x, layout="token")),
                    ("agg", pg.aggregated_forward(g, 0, x, layout="token"))):
        err = (y - ref).abs()
        print(T, name, "rel", (err.max() / ref.abs().max()).item())
        colblk = [round((err[:, c:c + 256].max() / ref.abs().max()).item(), 4) for c in range(0, m, 256)]
        rowblk = [round((err[r0:r0 + 128].max() / ref.abs().max()).item(), 4) for r0 in range(0, T, 128)]
        print("   per 256-col block:", colblk, " per 128-row block:", rowblk)
        ratio = (y / ref)[:4, :6]
        print("   y/ref sample:", [[round(v, 3) for v in row] for row in ratio.tolist()])
