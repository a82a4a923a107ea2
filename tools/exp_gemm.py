"""tcgen05 GEMM (pg_gemm_bf16) vs torch.matmul timing at prefill shapes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2605_08568_b200 import _lib  # noqa: E402


def bench(fn, reps=20):
    for _ in range(3):
        fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for (M, N, K) in [(2048, 832, 4096), (2048, 4096, 832), (2048, 11008, 1200), (2048, 1200, 11008),
                  (8192, 8192, 8192), (32768, 832, 4096), (32768, 4096, 832)]:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    st = torch.cuda.current_stream().cuda_stream
    t_ours = bench(lambda: _lib.call("pg_gemm_bf16", a.data_ptr(), K, b.data_ptr(), K, c.data_ptr(), N, M, N, K, 1, st))
    t_cub = bench(lambda: torch.matmul(a, b.t(), out=c))
    f = 2 * M * N * K
    print(f"M={M:6d} N={N:6d} K={K:6d}: ours {t_ours * 1e3:8.1f} us {f / t_ours / 1e9:6.0f} TF/s | "
          f"cuBLAS {t_cub * 1e3:8.1f} us {f / t_cub / 1e9:6.0f} TF/s", flush=True)
