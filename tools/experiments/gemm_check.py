"""tcgen05 GEMM mechanics sweep vs torch (debug aid)."""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2605_08568_b200 import _lib  # noqa: E402


def run(M, N, K, pattern="randn"):
    g = torch.Generator(device="cuda").manual_seed(M * 7 + N * 3 + K)
    if pattern == "randn":
        a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
        b = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    else:  # identity-ish probes
        a = torch.zeros(M, K, device="cuda", dtype=torch.bfloat16)
        b = torch.zeros(N, K, device="cuda", dtype=torch.bfloat16)
        for i in range(min(M, K)):
            a[i, i] = 1
        for j in range(min(N, K)):
            b[j, j] = float(j % 7 + 1)
    c = torch.zeros(M, N, device="cuda", dtype=torch.float32)
    _lib.call("pg_gemm_bf16", a.data_ptr(), K, b.data_ptr(), K, c.data_ptr(), N, M, N, K, 0,
              torch.cuda.current_stream().cuda_stream)
    ref = a.float() @ b.float().t()
    torch.cuda.synchronize()
    err = (c - ref).abs().max().item() / max(ref.abs().max().item(), 1e-30)
    return err, c, ref


if __name__ == "__main__":
    shapes = [(128, 16, 16), (128, 256, 64), (200, 1000, 832), (128, 128, 1024), (128, 256, 4096), (200, 832, 4096),
              (16, 832, 4096), (128, 128, 512), (128, 128, 320), (128, 128, 256), (1024, 1216, 4096)]
    for (M, N, K) in shapes:
        for pat in ("randn",):
            err, c, ref = run(M, N, K, pat)
            print(f"M={M} N={N} K={K} {pat}: rel err {err:.3e}")
            if err > 1e-2 and pat == "eye":
                bad = ((c - ref).abs() > 1e-3).nonzero()[:8].tolist()
                print("   first bad (row, col):", bad, "c:", [round(c[i, j].item(), 3) for i, j in bad[:4]],
                      "ref:", [round(ref[i, j].item(), 3) for i, j in bad[:4]])
