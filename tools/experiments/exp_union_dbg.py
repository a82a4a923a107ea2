"""Debug: which union path runs, and per-linear device time (q shape, T=256)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402
from oracle import pyoracle  # noqa: E402
m, n = int(os.environ.get("M", 4096)), int(os.environ.get("N", 4096))
K = pg.single_layer_k(m, n, 0.6); r = pg.store_rank(K, min(m, n)); T = 256
pats = pyoracle.make_patterns(17171, T, [(r, K)])
bt = (torch.randn(r, n, device="cuda") / n ** 0.5).to(torch.bfloat16)
a = (torch.randn(m, r, device="cuda") / m ** 0.5).to(torch.bfloat16)
L = pg.FactorizedLayer.from_device(bt, a, K)
b = pg.SelectionBatch(L, [pg.RankSelection(p[0]) for p in pats])
x = torch.randn(T, n, device="cuda").to(torch.bfloat16)
tp = torch.arange(T, device="cuda", dtype=torch.int32)
y = torch.empty(T, m, device="cuda", dtype=torch.bfloat16)
n0 = pg.launch_count()
pg.masked_forward_union(L, b, tp, x, out_dtype=torch.bfloat16, out=y)
torch.cuda.synchronize()
print("launches", pg.launch_count() - n0)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
for _ in range(3):
    pg.masked_forward_union(L, b, tp, x, out_dtype=torch.bfloat16, out=y)
e0.record()
for _ in range(20):
    pg.masked_forward_union(L, b, tp, x, out_dtype=torch.bfloat16, out=y)
e1.record(); torch.cuda.synchronize()
us = e0.elapsed_time(e1) / 20 * 1e3
print(f"m={m} n={n} r={r}: {us:.1f} us/linear (eager), {r*(m+n)*2/us/1e3:.0f} GB/s")
if os.environ.get("PG_WM_DBG"):
    import ctypes as C, numpy as np
    from paper_2605_08568_b200 import _lib
    pg.masked_forward_union(L, b, tp, x, out_dtype=torch.bfloat16, out=y)  # stage 1 + stage 2; stamps: stage 2
    torch.cuda.synchronize()
    buf = (C.c_uint64 * (1024 * 16))()
    _lib.call("pg_chain_debug_dump", buf, 1024 * 16)
    a = np.array(buf, dtype=np.float64).reshape(1024, 16)[:148]
    t0 = a[:, 0].min()
    rel = (a - t0) / 1e3
    rel[a == 0] = np.nan
    names = ["start", "prod_wait_done", "prod_issued", "epi_done", "flags_ok", "-", "reduce_done", "exit", "epi_first_acc", "partial_stored", "flag_set", "bulk_in", "-", "reduced", "-"]
    for k, nm in enumerate(names):
        col = rel[:, k]
        print(f"{nm:15s} min {np.nanmin(col) if np.isfinite(col).any() else float('nan'):7.2f}  "
              f"med {np.nanmedian(col) if np.isfinite(col).any() else float('nan'):7.2f}  "
              f"max {np.nanmax(col) if np.isfinite(col).any() else float('nan'):7.2f} us")
