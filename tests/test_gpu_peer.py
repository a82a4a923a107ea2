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


def _ipc_worker(rank, world, init, q):
    import ctypes as C
    import torch.distributed as dist
    torch.cuda.set_device(0)
    dist.init_process_group("gloo", init_method=init, rank=rank, world_size=world)
    from paper_2605_08568_b200.dist import PeerReduceLinear
    rng = np.random.default_rng(7)
    A = rng.standard_normal((256, 96)) / 16.0
    B = rng.standard_normal((128, 96)) / 11.0
    pr = PeerReduceLinear(A, B, world, rank, dtype="bf16", group=dist.group.WORLD)
    assert pr.peer_ptrs[rank] == pr.recv.data_ptr() and len(pr._opened) == world - 1
    # every rank writes its id into its right neighbour's receive buffer through
    # the IPC-opened pointer, then reads its own buffer
    cudart = C.CDLL("/usr/local/cuda/lib64/libcudart.so")
    src = torch.full((16,), 1000 + rank, dtype=torch.int64, device="cuda")
    torch.cuda.synchronize()
    dst = (rank + 1) % world
    rc = cudart.cudaMemcpy(C.c_void_p(pr.peer_ptrs[dst]), C.c_void_p(src.data_ptr()), C.c_size_t(16 * 8), 3)
    torch.cuda.synchronize()
    dist.barrier()
    got = pr.recv[:16].cpu().tolist()
    pr.close()
    dist.barrier()
    dist.destroy_process_group()
    q.put((rank, rc, got))


def test_peer_ipc_exchange_two_processes(tmp_path):
    """PeerReduceLinear._exchange across real processes: receive-buffer IPC
    handles all-gathered over a gloo group, opened with pg_ipc_open_handle, and
    written through by the neighbour rank (two processes on the one reachable
    GPU; the fused kernel itself runs in the virtual-rank test above)."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    world = 2
    init = f"file://{tmp_path}/rdzv"
    procs = [ctx.Process(target=_ipc_worker, args=(r, world, init, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, rc, got in res:
        assert rc == 0
        assert got == [1000 + (rank - 1) % world] * 16


@pytest.mark.parametrize("world,d,ff,dtype", [(1, 512, 1376, "bf16"), (2, 512, 1376, "bf16"), (4, 1024, 2752, "bf16"),
                                              (2, 512, 1376, "f32")])
def test_peer_mlp_block_fused_allreduce(pg, port, world, d, ff, dtype):
    """Expert-sharded MLP block in one launch per rank (pg_mlp_forward_peer):
    up/gate partials reduced over the ranks into act mid-launch, then down's
    partials; every rank ends with the same y, within the single-GPU MLP
    tolerance of the f64 oracle composition on the same rounded inputs."""
    from oracle import pyoracle
    from paper_2605_08568_b200.dist import PeerReduceMLP
    from tests.test_gpu_parity import _silu, bf16_round, make_layer_data
    K = pg.single_layer_k(ff, d, 0.6)
    r = pg.store_rank(K, d)
    pats = pyoracle.make_patterns(17171 + world, 2, [(r, K)] * 3)
    data = {nm: make_layer_data(port, *(shp + (r, 70 + i))) for i, (nm, shp) in
            enumerate([("up", (ff, d)), ("gate", (ff, d)), ("down", (d, ff))])}
    ranks = PeerReduceMLP.local_group(data["up"], data["gate"], data["down"], world, dtype=dtype, grid=148 // world)
    streams = [torch.cuda.Stream() for _ in ranks]
    tdt = torch.bfloat16 if dtype == "bf16" else torch.float32
    rnd = bf16_round if dtype == "bf16" else (lambda a: np.asarray(a, np.float32).astype(np.float64))
    for step in range(4):  # repeated launches, alternating patterns: tag parity and per-selection packs
        sels = [np.asarray(s, dtype=np.uint32) for s in pats[step % 2]]
        for rk in ranks:
            rk.prepare(sels)
        x = port.gaussian(80 + step, (d, 1))
        xd = torch.from_numpy(x[:, 0]).cuda().to(tdt)
        torch.cuda.synchronize()
        outs, acts = [], []
        for rk, st in zip(ranks, streams):
            with torch.cuda.stream(st):
                a = torch.empty(ff, dtype=tdt, device="cuda")
                outs.append(rk.forward(sels, xd, act=a, stream=st))
                acts.append(a)
        torch.cuda.synchronize()
        for o, a in zip(outs[1:], acts[1:]):
            assert torch.equal(o, outs[0]) and torch.equal(a, acts[0])
        xr = rnd(x)
        u = port.masked_forward(rnd(data["up"][0]), rnd(data["up"][1]), sels[0], xr)
        g = port.masked_forward(rnd(data["gate"][0]), rnd(data["gate"][1]), sels[1], xr)
        act = rnd(_silu(g) * u)
        ref = port.masked_forward(rnd(data["down"][0]), rnd(data["down"][1]), sels[2], act)[:, 0]
        y = outs[0].double().cpu().numpy()
        assert np.abs(y - ref).max() / np.abs(ref).max() <= (2e-3 if dtype == "bf16" else 1e-5), step
