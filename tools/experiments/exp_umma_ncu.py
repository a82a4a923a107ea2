"""One 8192^3 tcgen05 GEMM (for ncu)."""
import os, sys
import torch
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_08568_b200 import _lib  # noqa: E402
M = int(os.environ.get("GM", 8192)); N = int(os.environ.get("GN", 8192)); K = int(os.environ.get("GK", 8192))
a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
st = torch.cuda.current_stream().cuda_stream
for _ in range(3):
    _lib.call("pg_gemm_bf16", a.data_ptr(), K, b.data_ptr(), K, c.data_ptr(), N, M, N, K, 1, st)
torch.cuda.synchronize()
