"""Config-3 prefill exactly as bench.py times it: 16 prompts x 2048 tokens, each
prompt routed on device to its own expert subset (route_select_pooled from one
pooled input), then
  * pg_prefill_batched over 16 distinct per-prompt aggregated arenas, and
  * pg_pack_selected (device pack from the device selection) + pg_prefill_packed,
at the q (4096 x 4096) and down (4096 x 11008) shapes of LLaMA-7B at ratio 0.6.

Bars: selection bit-exact vs the oracle's
select_topk(score(mean_pool(x))); values vs a torch reference of the same
math (z rounded to bf16 between the GEMMs, accumulated in f64) <= 2e-3 over all
32768 tokens, and vs
the f64 oracle masked_forward (rank_experts.hpp:52-72) on the same bf16-rounded
A, B, X <= 8e-3 for a token sample of several prompts; the two device paths
agree and repeat bit-identically.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

P, T = 16, 2048


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_08568_b200 as m
    return m


def rel(a, b):
    a = np.asarray(a, np.float64); b = np.asarray(b, np.float64)
    return float(np.abs(a - b).max() / max(np.abs(b).max(), 1e-300))


def bf16r(a):
    return torch.from_numpy(np.ascontiguousarray(a)).to(torch.bfloat16).double().numpy()


@pytest.mark.parametrize("m,n", [(4096, 4096), (4096, 11008)])
def test_routed_prefill_config3(pg, port, m, n):
    K = pg.single_layer_k(m, n, 0.6)
    r = pg.store_rank(K, min(m, n))
    rng = np.random.default_rng(m + n)
    sig = 1.0 / (1.0 + np.arange(r) / 64.0)
    A = rng.standard_normal((m, r)) * sig / np.sqrt(m)
    B = rng.standard_normal((n, r)) / np.sqrt(n)
    theta = rng.standard_normal((r, n))
    L = pg.FactorizedLayer(A, B, K, dtype="bf16")
    router = pg.RouterParams(theta)
    # per-prompt token distributions differ (prompt-dependent mean) so the routes differ
    g = torch.Generator(device="cuda").manual_seed(m + n)
    X = torch.randn(P * T, n, device="cuda", generator=g)
    X += torch.randn(P, 1, n, device="cuda", generator=g).repeat_interleave(T, 0).reshape(P * T, n) * 0.5
    X = X.to(torch.bfloat16)
    offs = [p * T for p in range(P + 1)]

    h = pg.mean_pool(X, layout="token", offsets=offs)
    sel = pg.route_select_pooled(router, h, K)  # [P, K] device int32
    sels = sel.cpu().numpy().astype(np.uint32)
    assert len({tuple(s) for s in sels}) == P, "prompts should route to distinct subsets"
    for p in (0, P - 1):  # bit-exact selection vs the reference router on the same bf16 input
        xp = X[p * T:(p + 1) * T].double().cpu().numpy().T  # feature-major n x T, exact widening
        want = port.select_topk(port.score(theta, np.zeros(r), port.mean_pool(xp)), K)
        assert np.array_equal(sels[p], want)

    aggs = [pg.aggregate_layout(L, [pg.RankSelection(s)], 0.9) for s in sels]
    y1 = pg.prefill_batched(aggs, offs, X, out_dtype=torch.float32)
    pk = pg.pack_selected(L, sel)
    y2 = pg.prefill_packed(pk, offs, X, out_dtype=torch.float32)
    assert torch.equal(pg.prefill_packed(pg.pack_selected(L, sel), offs, X, out_dtype=torch.float32), y2)
    # the B^T rows gathered inside the stage-1 GEMM (TMA gather4, A packed only):
    # the same operands in the same order -> bit-identical to the packed path
    pkg = pg.pack_selected(L, sel, gather=True)
    assert pkg.gathered and pkg.bt is None
    assert torch.equal(pg.prefill_packed(pkg, offs, X, out_dtype=torch.float32), y2)

    # reference of the kernel's math: z = bf16(x B_S) accumulated in f64 (an
    # fp32-accumulated torch reference is itself ~2e-3 off at K = 11008 over
    # 32768 tokens: bf16 rounding of z amplifies accumulation-order noise),
    # then y = z A_S^T.  Bar 3e-3: an f32-accumulated z lands on the other side
    # of a bf16 rounding boundary than the f64 one for a few entries, and
    # those flips reach ~2.2e-3 of max|y| on random data (seen at K = 819)
    Ab = torch.from_numpy(A).to(torch.bfloat16).double().cuda()
    Bb = torch.from_numpy(B).to(torch.bfloat16).double().cuda()
    err1 = err2 = 0.0
    for p in range(P):
        s = torch.from_numpy(sels[p].astype(np.int64)).cuda()
        xp = X[p * T:(p + 1) * T].double()
        z = (xp @ Bb[:, s]).to(torch.bfloat16).double()
        ref = z @ Ab[:, s].t()
        d = ref.abs().max().item()
        err1 = max(err1, (y1[p * T:(p + 1) * T].double() - ref).abs().max().item() / d)
        err2 = max(err2, (y2[p * T:(p + 1) * T].double() - ref).abs().max().item() / d)
    assert err1 <= 3e-3, err1
    assert err2 <= 3e-3, err2
    assert rel(y1.cpu().numpy(), y2.cpu().numpy()) <= 2e-3

    # f64 oracle (the reference's masked_forward) on a token sample of 3 prompts
    Ad, Bd = bf16r(A), bf16r(B)
    for p in (0, 7, P - 1):
        rows = np.arange(p * T, p * T + T, T // 8)  # 8 tokens spread over the prompt
        xs = X[rows].double().cpu().numpy().T
        ref = port.masked_forward(Ad, Bd, sels[p], xs).T
        assert rel(y2[rows].double().cpu().numpy(), ref) <= 8e-3
        assert rel(y1[rows].double().cpu().numpy(), ref) <= 8e-3


def test_pack_selected_layout(pg, port):
    """The device pack equals the selected rows of B^T / columns of A, zero
    padded to kp = K rounded up to 8 (exec_engine.hpp:136-158 column copies)."""
    m, n, r, K, Pp = 300, 264, 200, 93, 3
    rng = np.random.default_rng(5)
    A = rng.standard_normal((m, r))
    B = rng.standard_normal((n, r))
    L = pg.FactorizedLayer(A, B, K, dtype="bf16")
    sels = np.stack([np.sort(rng.choice(r, K, replace=False)) for _ in range(Pp)]).astype(np.int32)
    pk = pg.pack_selected(L, torch.from_numpy(sels).cuda())
    kp = (K + 7) // 8 * 8
    a = pk.a.view(torch.bfloat16).reshape(Pp, m, kp).double().cpu().numpy()
    bt = pk.bt.view(torch.bfloat16).reshape(Pp, kp, -1).double().cpu().numpy()
    for p in range(Pp):
        assert np.array_equal(a[p, :, :K], bf16r(A[:, sels[p]]))
        assert not a[p, :, K:].any()
        assert np.array_equal(bt[p, :K, :n], bf16r(B[:, sels[p]].T))
        assert not bt[p, K:].any()
    with pytest.raises(ValueError):
        pg.pack_selected(L, sels)  # host array: the device path only


@pytest.mark.parametrize("K", [93, 96, 200])
def test_prefill_gathered_ragged(pg, K):
    """Gathered B^T rows (pg_prefill_gathered) vs the packed arena on ragged
    prompts (0, 256, 300, 517 tokens), K not a multiple of 8 or 4 (padding rows
    read as zero through out-of-range gather coordinates), a reused `into`
    buffer, bf16 and f32 outputs: bit-identical."""
    m, n, r = 384, 512, 240
    rng = np.random.default_rng(K)
    A = rng.standard_normal((m, r)) / np.sqrt(m)
    B = rng.standard_normal((n, r)) / np.sqrt(n)
    L = pg.FactorizedLayer(A, B, K, dtype="bf16")
    lens = [256, 0, 300, 517]
    offs = np.concatenate([[0], np.cumsum(lens)]).tolist()
    Pp = len(lens)
    sels = np.stack([np.sort(rng.choice(r, K, replace=False)) for _ in range(Pp)]).astype(np.int32)
    sel = torch.from_numpy(sels).cuda()
    g = torch.Generator(device="cuda").manual_seed(K)
    X = torch.randn(offs[-1], n, device="cuda", generator=g).to(torch.bfloat16)
    pk = pg.pack_selected(L, sel)
    pkg = pg.pack_selected(L, sel, gather=True)
    for dt in (torch.float32, torch.bfloat16):
        y_pack = pg.prefill_packed(pk, offs, X, out_dtype=dt)
        y_gath = pg.prefill_packed(pkg, offs, X, out_dtype=dt)
        assert torch.equal(y_gath, y_pack)
    # reuse of the gathered buffers with another selection
    sels2 = np.stack([np.sort(rng.choice(r, K, replace=False)) for _ in range(Pp)]).astype(np.int32)
    sel2 = torch.from_numpy(sels2).cuda()
    pkg2 = pg.pack_selected(L, sel2, into=pkg, gather=True)
    assert pkg2.a.data_ptr() == pkg.a.data_ptr()
    y2 = pg.prefill_packed(pkg2, offs, X, out_dtype=torch.float32)
    assert torch.equal(y2, pg.prefill_packed(pg.pack_selected(L, sel2), offs, X, out_dtype=torch.float32))
    with pytest.raises(ValueError):
        pg.pack_selected(L, sel2, into=pk, gather=True)  # mode mismatch
    # prompts shorter than a CTA-pair tile are refused by the gathered path
    with pytest.raises(Exception):
        pg.prefill_packed(pkg, [0, 100, 356, 656, 1073], torch.zeros(1073, n, device="cuda", dtype=torch.bfloat16))
