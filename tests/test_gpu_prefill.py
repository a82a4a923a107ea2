"""K5: bf16 prefill on the tensor cores (tcgen05 + TMEM + TMA grouped GEMM).

Two bars:
  * GEMM mechanics vs a plain PyTorch fp32 reference of the SAME two GEMMs
    (z rounded to bf16 between them, as the kernel does): max|d|/max|ref| <= 2e-3
    (accumulation order only);
  * end to end vs the f64 oracle on the same bf16-rounded A, B, X:
    <= 8e-3 (TOLBF_PREFILL).
Shapes cover ragged M (tokens), N not a multiple of the 256 tile (m=1000,
K=832 -> 4 x 208), multi-pattern arenas (packing + masks) and grouped prompts.
"""
import os
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_08568_b200 as m
    return m


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def layer_data(port, m, n, r, seed):
    sig = 1.0 / (1.0 + np.arange(r) / 64.0)
    A = port.gaussian(seed, (m, r)) * sig / np.sqrt(m)
    B = port.gaussian(seed + 1, (n, r)) / np.sqrt(n)
    return A, B


def torch_ref(A, B, sel, x_tok):
    """fp32 reference of the kernel's math: z = bf16(x B_S), y = z A_S^T (token-major)."""
    Ab = torch.from_numpy(A[:, sel]).to(torch.bfloat16).float().cuda()
    Bb = torch.from_numpy(B[:, sel]).to(torch.bfloat16).float().cuda()
    xb = x_tok.float()
    z = (xb @ Bb).to(torch.bfloat16).float()
    return (z @ Ab.t()).double().cpu().numpy()


@pytest.mark.parametrize("m,n,r,K,T", [(1000, 4096, 1664, 832, 200), (4096, 4096, 1638, 819, 128),
                                       (512, 1024, 384, 150, 37), (11008, 4096, 2388, 1194, 256)])
def test_prefill_masked_forward(pg, port, m, n, r, K, T):
    A, B = layer_data(port, m, n, r, 7 + m)
    sel = port.select_topk(port.gaussian(8 + m, (r,)), K)
    x = port.gaussian(9 + m, (T, n))
    L = pg.FactorizedLayer(A, B, K, dtype="bf16")
    xt = torch.from_numpy(x).cuda().to(torch.bfloat16)
    n0 = pg.launch_count()
    y = pg.masked_forward(L, pg.RankSelection(sel), xt, layout="token")
    assert pg.launch_count() > n0
    assert rel(y.cpu().numpy(), torch_ref(A, B, sel, xt)) <= 2e-3
    bfr = lambda a: torch.from_numpy(np.asarray(a)).to(torch.bfloat16).double().numpy()  # noqa: E731
    ref = port.masked_forward(bfr(A), bfr(B), sel, bfr(x).T).T
    assert rel(y.cpu().numpy(), ref) <= 8e-3
    # feature-major activations (the reference's Mat layout) through the same kernel
    yf = pg.masked_forward(L, pg.RankSelection(sel), xt.t().contiguous())
    assert torch.equal(yf.t().contiguous(), y)


def test_prefill_grouped_heterogeneous_prompts(pg, port):
    """config-3 style: several prompts, each with its own expert subset, in one
    grouped launch per stage; equals the per-prompt path bit for bit."""
    m, n, r, K = 2048, 1024, 768, 384
    A, B = layer_data(port, m, n, r, 3)
    from oracle import pyoracle
    pats = [p[0] for p in pyoracle.make_patterns(17171, 6, [(r, K)])]
    L = pg.FactorizedLayer(A, B, K, dtype="bf16")
    g = pg.aggregate_layout(L, [pg.RankSelection(p) for p in pats], 0.9)  # multi-pattern arena: masks + 2 runs
    lens = [128, 300, 17, 64, 256, 9]
    pids = [0, 3, 5, 1, 2, 4]
    offs = np.concatenate([[0], np.cumsum(lens)])
    X = torch.from_numpy(port.gaussian(4, (offs[-1], n))).cuda().to(torch.bfloat16)
    Y = pg.aggregated_forward_batched(g, pids, offs, X)
    for q, pid in enumerate(pids):
        xq = X[offs[q]:offs[q + 1]].contiguous()
        yq = pg.aggregated_forward(g, pid, xq, layout="token")
        assert torch.equal(Y[offs[q]:offs[q + 1]], yq)
        assert rel(yq.cpu().numpy(), torch_ref(A, B, pats[pid].astype(np.int64), xq)) <= 2e-3


@pytest.mark.parametrize("M,N,K", [(128, 16, 16), (200, 1000, 832), (200, 832, 4096), (16, 832, 4096),
                                   (1024, 1216, 4096), (300, 11008, 1216), (2048, 4096, 832)])
def test_gemm_primitive_vs_torch(pg, M, N, K):
    """pg_gemm_bf16 (the K5 building block) vs torch fp32 matmul of the same bf16
    operands; covers ragged M, tiles narrower than 32-column chunks (N=832 ->
    4 x 208) and long K loops around the 4-stage ring."""
    from paper_2605_08568_b200 import _lib
    g = torch.Generator(device="cuda").manual_seed(M + N + K)
    a = torch.randn(M, K, device="cuda", generator=g).to(torch.bfloat16)
    b = torch.randn(N, K, device="cuda", generator=g).to(torch.bfloat16)
    for out_bf16 in (0, 1):
        c = torch.full((M, N), float("nan"), device="cuda",
                       dtype=torch.bfloat16 if out_bf16 else torch.float32)
        _lib.call("pg_gemm_bf16", a.data_ptr(), K, b.data_ptr(), K, c.data_ptr(), N, M, N, K, out_bf16,
                  torch.cuda.current_stream().cuda_stream)
        ref = a.float() @ b.float().t()
        err = ((c.float() - ref).abs().max() / ref.abs().max()).item()
        assert err <= (8e-3 if out_bf16 else 1e-5), err


def _union_ref(A, B, masks, pid, X):
    """fp32 reference of the union-masked kernel: z = bf16(mask * (x B)), y = z A^T."""
    Ab = torch.from_numpy(A).to(torch.bfloat16).float().cuda()
    Bb = torch.from_numpy(B).to(torch.bfloat16).float().cuda()
    M = torch.from_numpy(masks[pid]).float().cuda()
    z = ((X.float() @ Bb) * M).to(torch.bfloat16).float()
    return (z @ Ab.t()).double().cpu().numpy()


@pytest.mark.parametrize("m,n,r,K,P,T", [(1000, 1024, 768, 384, 6, 300), (4096, 4096, 1638, 819, 256, 256),
                                         (11008, 4096, 2388, 1194, 64, 256), (384, 512, 300, 150, 3, 5),
                                         (4096, 11008, 2388, 1194, 32, 256)])  # last: long K, split-K path
def test_union_masked_batch(pg, port, m, n, r, K, P, T):
    """config 4: a heterogeneous decode batch (every token with its prompt's
    selection) through one pass over the weights equals masked_forward per
    token: vs the fp32 reference of the same math (<= 2e-3), vs the f64 oracle
    per prompt (<= 8e-3), and bit-identical to single-prompt union calls."""
    from oracle import pyoracle
    A, B = layer_data(port, m, n, r, 11 + m)
    pats = [p[0] for p in pyoracle.make_patterns(17171, P, [(r, K)])]
    L = pg.FactorizedLayer(A, B, K, dtype="bf16")
    batch = pg.SelectionBatch(L, [pg.RankSelection(p) for p in pats])
    rng = np.random.default_rng(T + P)
    pid = rng.integers(0, P, T)
    X = torch.from_numpy(port.gaussian(12 + m, (T, n))).cuda().to(torch.bfloat16)
    n0 = pg.launch_count()
    Y = pg.masked_forward_union(L, batch, pid, X)
    assert pg.launch_count() >= n0 + 2
    masks = np.zeros((P, r), np.float32)
    for p, s in enumerate(pats):
        masks[p, s] = 1.0
    assert rel(Y.cpu().numpy(), _union_ref(A, B, masks, pid, X)) <= 2e-3
    bfr = lambda a: torch.from_numpy(np.asarray(a)).to(torch.bfloat16).double().numpy()  # noqa: E731
    Ab, Bb = bfr(A), bfr(B)
    Xd = X.double().cpu().numpy()
    for p in sorted(set(pid.tolist()))[:3]:
        rows = np.nonzero(pid == p)[0]
        ref = port.masked_forward(Ab, Bb, pats[p], Xd[rows].T).T
        assert rel(Y[rows].cpu().numpy(), ref) <= 8e-3
    # deterministic (split-K partials are summed in slice order), and a row's
    # result does not depend on its batch-mates beyond accumulation order
    assert torch.equal(pg.masked_forward_union(L, batch, pid, X), Y)
    one = pg.masked_forward_union(L, batch, pid[:1], X[:1].contiguous())
    assert rel(one.cpu().numpy(), Y[:1].cpu().numpy()) <= 2e-3
    with pytest.raises(IndexError):
        pg.masked_forward_union(L, batch, [P], X[:1].contiguous())


def test_module_forward_union_grouped_equals_single(pg, port):
    """q/k/v-style linears sharing x through one grouped launch per stage give
    the single-linear union results (the stream-K split of a grouped launch
    differs from a single linear's, so f32 partials are summed in another
    order: equal within one bf16 rounding), deterministically."""
    from oracle import pyoracle
    shapes = [(512, 1024, 384, 192), (256, 1024, 384, 192), (768, 1024, 320, 160)]
    P, T = 16, 96
    pats = pyoracle.make_patterns(4242, P, [(r, K) for _, _, r, K in shapes])
    Ls, Bs = [], []
    for li, (m, n, r, K) in enumerate(shapes):
        A, B = layer_data(port, m, n, r, 31 + li)
        L = pg.FactorizedLayer(A, B, K, dtype="bf16")
        Ls.append(L)
        Bs.append(pg.SelectionBatch(L, [pg.RankSelection(p[li]) for p in pats]))
    pid = np.random.default_rng(3).integers(0, P, T)
    X = torch.from_numpy(port.gaussian(33, (T, 1024))).cuda().to(torch.bfloat16)
    ys = pg.module_forward_union(Ls, Bs, pid, X)
    ys2 = pg.module_forward_union(Ls, Bs, pid, X)
    for L, b, y, y2 in zip(Ls, Bs, ys, ys2):
        assert torch.equal(y, y2)
        one = pg.masked_forward_union(L, b, pid, X).float()
        assert ((y.float() - one).abs().max() / one.abs().max()).item() <= 8e-3


def test_union_masked_batch_f32_out_and_long_batch(pg, port):
    """f32 output and a long heterogeneous batch (T = 1024: several M tiles of
    CTA pairs) through the union path, vs the fp32 reference of the same math."""
    from oracle import pyoracle
    m, n, r, K, P, T = 2048, 1024, 640, 320, 40, 1024
    A, B = layer_data(port, m, n, r, 77)
    pats = [p[0] for p in pyoracle.make_patterns(9090, P, [(r, K)])]
    L = pg.FactorizedLayer(A, B, K, dtype="bf16")
    batch = pg.SelectionBatch(L, [pg.RankSelection(p) for p in pats])
    pid = np.random.default_rng(11).integers(0, P, T)
    X = torch.from_numpy(port.gaussian(78, (T, n))).cuda().to(torch.bfloat16)
    Y = pg.masked_forward_union(L, batch, torch.from_numpy(pid.astype(np.int32)).cuda(), X, out_dtype=torch.float32)
    assert Y.dtype == torch.float32 and Y.shape == (T, m)
    masks = np.zeros((P, r), np.float32)
    for p, s in enumerate(pats):
        masks[p, s] = 1.0
    assert rel(Y.cpu().numpy(), _union_ref(A, B, masks, pid, X)) <= 2e-3
    Yb = pg.masked_forward_union(L, batch, pid, X)  # bf16 output: the same values rounded
    assert rel(Yb.float().cpu().numpy(), Y.cpu().numpy()) <= 1e-2


def test_union_weights_on_m_forced():
    """The weights-on-M union kernel (union_wm.cu) on every union shape above,
    forced for all GEMMs (PG_UNION_WM_MINKB=0; by default it only takes the
    long-K / many-tile GEMMs): the union parity tests re-run in a subprocess."""
    import subprocess
    import sys
    env = dict(os.environ, PG_UNION_WM_MINKB="0")
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", __file__, "-k", "union and not forced"],
                       env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
