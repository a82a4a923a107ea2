"""Expert-sharded decode with the all-reduce fused into the kernel over peer
memory (dist.PeerReduceLinear / pg_agg_forward_peer).  Only one GPU is
reachable here, so the ranks are virtual: one process, one stream per rank,
each rank's kernel on 148/world SMs so all ranks' kernels are co-resident and
exchange through each other's receive buffers exactly as over NVLink."""
import numpy as np
import pytest
import torch

pytestmark = [pytest.mark.gpu, pytest.mark.timeout(300)]


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_08568_b200 as m
    return m


@pytest.mark.parametrize("world,m,n,r,K", [(2, 1024, 512, 384, 192), (4, 4096, 1024, 768, 320)])
def test_peer_reduce_fused_allreduce(pg, port, world, m, n, r, K):
    from paper_2605_08568_b200.dist import PeerReduceLinear
    sig = 1.0 / (1.0 + np.arange(r) / 64.0)
    A = port.gaussian(50 + world, (m, r)) * sig / np.sqrt(m)
    B = port.gaussian(51 + world, (n, r)) / np.sqrt(n)
    sel = np.sort(np.random.default_rng(world).choice(r, K, replace=False)).astype(np.uint32)
    ranks = PeerReduceLinear.local_group(A, B, world, dtype="bf16", grid=148 // world)
    streams = [torch.cuda.Stream() for _ in ranks]
    for rk in ranks:
        rk.prepare(sel)
    torch.cuda.synchronize()
    bfr = lambda a: torch.from_numpy(np.asarray(a)).to(torch.bfloat16).double().numpy()  # noqa: E731
    for step in range(4):  # repeated launches: the receive buffers alternate by tag parity
        x = torch.from_numpy(port.gaussian(60 + step, (n,))).cuda().to(torch.bfloat16)
        torch.cuda.synchronize()
        outs = []
        for rk, st in zip(ranks, streams):
            with torch.cuda.stream(st):
                outs.append(rk.forward(sel, x, stream=st))
        torch.cuda.synchronize()
        for o in outs[1:]:
            assert torch.equal(o, outs[0])  # every rank holds the same, rank-ordered sum
        ref = port.masked_forward(bfr(A), bfr(B), sel, x.double().cpu().numpy()[:, None])[:, 0]
        y = outs[0].double().cpu().numpy()
        assert np.abs(y - ref).max() / np.abs(ref).max() <= 1e-4
