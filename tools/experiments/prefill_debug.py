import os, sys
import numpy as np
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg
from paper_2605_08568_b200 import _lib

torch.manual_seed(0)
m, n, r, K, T = 1000, 4096, 1664, 832, 200
A = np.random.default_rng(1).standard_normal((m, r)) / np.sqrt(m)
B = np.random.default_rng(2).standard_normal((n, r)) / np.sqrt(n)
sel = np.sort(np.random.default_rng(3).choice(r, K, replace=False)).astype(np.uint32)
x = torch.randn(T, n, device="cuda").to(torch.bfloat16)
L = pg.FactorizedLayer(A, B, K, dtype="bf16")
Ab = torch.from_numpy(A[:, sel]).to(torch.bfloat16).cuda()
Bb = torch.from_numpy(B[:, sel]).to(torch.bfloat16).cuda()
z_ref = (x.float() @ Bb.float())
# step 1 via the primitive: Z = x . (B_S^T)^T
bt = Bb.t().contiguous()   # [K, n]
z = torch.empty(T, K, device="cuda", dtype=torch.bfloat16)
_lib.call("pg_gemm_bf16", x.data_ptr(), n, bt.data_ptr(), n, z.data_ptr(), K, T, K, n, 1, torch.cuda.current_stream().cuda_stream)
print("Z via primitive rel:", ((z.float() - z_ref).abs().max() / z_ref.abs().max()).item())
y_ref = z.float() @ Ab.float().t()
y = torch.empty(T, m, device="cuda")
_lib.call("pg_gemm_bf16", z.data_ptr(), K, Ab.data_ptr(), K, y.data_ptr(), m, T, m, K, 0, torch.cuda.current_stream().cuda_stream)
print("Y via primitive rel:", ((y - y_ref).abs().max() / y_ref.abs().max()).item())
y2 = pg.masked_forward(L, pg.RankSelection(sel), x, layout="token")
print("masked_forward rel:", ((y2 - y_ref).abs().max() / y_ref.abs().max()).item())
for T2 in (8, 9, 16, 64):
    xs = x[:T2].contiguous()
    y3 = pg.masked_forward(L, pg.RankSelection(sel), xs, layout="token")
    ref3 = (xs.float() @ Bb.float()) @ Ab.float().t()
    print(f"T={T2} masked_forward rel vs f32-z ref:", ((y3 - ref3).abs().max() / ref3.abs().max()).item())
print("z finite:", torch.isfinite(z.float()).all().item(), "z absmax", z.float().abs().max().item(), "Ab absmax", Ab.float().abs().max().item())
zr = torch.randn(T, K, device="cuda").to(torch.bfloat16)
for name, aa in (("randn z, Ab", zr), ("our z clone", z.clone())):
    yy = torch.empty(T, m, device="cuda")
    _lib.call("pg_gemm_bf16", aa.data_ptr(), K, Ab.data_ptr(), K, yy.data_ptr(), m, T, m, K, 0, torch.cuda.current_stream().cuda_stream)
    rr = aa.float() @ Ab.float().t()
    print(name, ((yy - rr).abs().max() / rr.abs().max()).item())
Ar = torch.randn(m, K, device="cuda").to(torch.bfloat16)
yy = torch.empty(T, m, device="cuda")
_lib.call("pg_gemm_bf16", zr.data_ptr(), K, Ar.data_ptr(), K, yy.data_ptr(), m, T, m, K, 0, torch.cuda.current_stream().cuda_stream)
rr = zr.float() @ Ar.float().t()
print("randn z, randn A", ((yy - rr).abs().max() / rr.abs().max()).item())
print("Ab contiguous", Ab.is_contiguous(), Ab.stride(), Ab.data_ptr() % 1024)
