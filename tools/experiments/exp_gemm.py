"""tcgen05 GEMM (pg_gemm_bf16) vs torch.matmul timing at prefill shapes."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_08568_b200 import _lib  # noqa: E402


def bench(fn, reps=20):
    """Device time per call: 10 calls captured in a CUDA graph, replayed."""
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
    st.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=st):
        for _ in range(10):
            fn()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        g.replay()
        e0.record(st)
        for _ in range(reps):
            g.replay()
        e1.record(st)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 10


SHAPES = [(2048, 832, 4096), (2048, 4096, 832), (2048, 11008, 1200), (2048, 1200, 11008),
          (8192, 8192, 8192), (32768, 832, 4096), (32768, 4096, 832)]
if os.environ.get("EXP_SHAPES"):  # "M,N,K;M,N,K"
    SHAPES = [tuple(int(v) for v in t.split(",")) for t in os.environ["EXP_SHAPES"].split(";")]
for (M, N, K) in SHAPES:
    a = torch.randn(M, K, device="cuda").to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda").to(torch.bfloat16)
    c = torch.empty(M, N, device="cuda", dtype=torch.bfloat16)
    t_ours = bench(lambda: _lib.call("pg_gemm_bf16", a.data_ptr(), K, b.data_ptr(), K, c.data_ptr(), N, M, N, K, 1,
                                     torch.cuda.current_stream().cuda_stream))
    t_cub = bench(lambda: torch.matmul(a, b.t(), out=c))
    f = 2 * M * N * K
    print(f"M={M:6d} N={N:6d} K={K:6d}: ours {t_ours * 1e3:8.1f} us {f / t_ours / 1e9:6.0f} TF/s | "
          f"cuBLAS {t_cub * 1e3:8.1f} us {f / t_cub / 1e9:6.0f} TF/s", flush=True)
