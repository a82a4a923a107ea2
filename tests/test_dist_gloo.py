"""Multi-process (world_size 2, gloo, CPU) tests of the multi-GPU host logic:
data-parallel prompt partitioning, pattern affinity, the expert-sharded
all-reduce protocol and max-over-ranks timing.  Per-rank
compute is the oracle (C restatement of rank_experts.hpp:52-72) standing in
for the GPU kernels; the collective and sharding code is the product's."""
import os
import socket
import sys

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)

from paper_2605_08568_b200 import dist as pgd  # noqa: E402


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, fn, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        q.put((rank, fn(rank, world)))
    except Exception as e:  # surface the failure to the parent
        q.put((rank, repr(e)))
    finally:
        dist.destroy_process_group()


def _run(fn, world=2):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, fn, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = dict(q.get(timeout=120) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
    return out


# ---- per-rank bodies (module level: picklable for spawn)
def _body_partitions(rank, world):
    mine = list(pgd.partition_prompts(37, world, rank))
    pats = [3, 1, 3, 2, 2, 3, 0, 1, 3, 9]
    aff = pgd.partition_by_pattern(pats, world)
    gathered = [None] * world
    dist.all_gather_object(gathered, (mine, aff))
    return gathered


def _body_sharded(rank, world):
    from oracle import pyoracle
    o = pyoracle.Oracle("port")
    m, n, r, K, T = 96, 80, 64, 29, 3
    A = o.gaussian(1, (m, r))
    B = o.gaussian(2, (n, r))
    x = o.gaussian(3, (n, T))
    sel = pyoracle.make_patterns(5, 1, [(r, K)])[0][0]
    shard = pgd.shard_layer(A, B, world, rank)

    def fwd(sh, local_ids, xt):
        y = o.masked_forward(sh.A, sh.B, np.asarray(local_ids, dtype=np.uint32), xt.numpy())
        return torch.from_numpy(np.ascontiguousarray(y))

    y = pgd.sharded_forward(shard, sel, torch.from_numpy(x), fwd)
    full = o.masked_forward(A, B, np.asarray(sel, dtype=np.uint32), x)
    rel = float(np.abs(y.numpy() - full).max() / np.abs(full).max())
    t = pgd.max_over_ranks(1.5 + rank)
    return rel, t, pgd.shard_selection(sel, world, rank).tolist(), [int(v) for v in sel]


def _body_sharded_mlp(rank, world):
    """The expert-sharded MLP block's algebra (PeerReduceMLP / pg_mlp_forward_peer):
    up and gate partials summed over the ranks BEFORE the nonlinearity, every
    rank forming the same act, then down's partials summed."""
    from oracle import pyoracle
    o = pyoracle.Oracle("port")
    d, ff, r, K = 48, 112, 40, 17
    fac = {nm: (o.gaussian(10 + i, (m, r)), o.gaussian(20 + i, (n, r)))
           for i, (nm, m, n) in enumerate((("up", ff, d), ("gate", ff, d), ("down", d, ff)))}
    sels = pyoracle.make_patterns(7, 1, [(r, K)] * 3)[0]
    x = o.gaussian(30, (d, 1))

    def fwd(sh, local_ids, xt):
        y = o.masked_forward(sh.A, sh.B, np.asarray(local_ids, dtype=np.uint32), xt.numpy())
        return torch.from_numpy(np.ascontiguousarray(y))

    sh = {nm: pgd.shard_layer(A, B, world, rank) for nm, (A, B) in fac.items()}
    u = pgd.sharded_forward(sh["up"], sels[0], torch.from_numpy(x), fwd).numpy()
    g = pgd.sharded_forward(sh["gate"], sels[1], torch.from_numpy(x), fwd).numpy()
    act = g / (1.0 + np.exp(-g)) * u
    y = pgd.sharded_forward(sh["down"], sels[2], torch.from_numpy(act), fwd).numpy()
    mf = lambda nm, s, v: o.masked_forward(fac[nm][0], fac[nm][1], np.asarray(s, dtype=np.uint32), v)  # noqa: E731
    gu, gg = mf("up", sels[0], x), mf("gate", sels[1], x)
    full = mf("down", sels[2], gg / (1.0 + np.exp(-gg)) * gu)
    gathered = [None] * world
    dist.all_gather_object(gathered, act.tobytes())
    return float(np.abs(y - full).max() / np.abs(full).max()), len(set(gathered))


def test_expert_sharded_mlp_block_matches_single_process():
    out = _run(_body_sharded_mlp)
    for rank in (0, 1):
        rel, distinct_acts = out[rank]
        assert rel <= 1e-12, rel
        assert distinct_acts == 1  # every rank holds the same act for its down shard


def test_partitions_cover_and_agree():
    out = _run(_body_partitions)
    g0, g1 = out[0], out[1]
    assert g0 == g1  # every rank sees the same assignment
    ranges = [g0[r][0] for r in range(2)]
    assert sorted(sum(ranges, [])) == list(range(37))
    assert abs(len(ranges[0]) - len(ranges[1])) <= 1
    aff = g0[0][1]
    assert sorted(sum(aff, [])) == list(range(10))
    pats = [3, 1, 3, 2, 2, 3, 0, 1, 3, 9]
    for p in set(pats):  # a pattern's prompts never straddle ranks
        owners = {r for r in range(2) for i in aff[r] if pats[i] == p}
        assert len(owners) == 1
    assert abs(len(aff[0]) - len(aff[1])) <= 2


def test_expert_sharded_allreduce_matches_single_process():
    out = _run(_body_sharded)
    for rank in (0, 1):
        rel, t, mine, sel = out[rank]
        assert rel <= 1e-12, rel  # fp64: reduction order only
        assert t == 2.5  # max over ranks
    s0, s1 = out[0][2], out[1][2]
    assert not set(s0) & set(s1)
    assert sorted(s0 + s1) == sorted(out[0][3])
    assert all(e % 2 == 0 for e in s0) and all(e % 2 == 1 for e in s1)


def test_partition_helpers_single_process():
    assert list(pgd.partition_prompts(5, 1, 0)) == [0, 1, 2, 3, 4]
    with pytest.raises(ValueError):
        pgd.partition_prompts(5, 2, 2)
    sh = pgd.shard_layer(np.arange(12.0).reshape(2, 6), np.arange(18.0).reshape(3, 6), 3, 1)
    assert sh.A.shape == (2, 2) and sh.A[0].tolist() == [1.0, 4.0]
    assert sh.local_ids([1, 4]).tolist() == [0, 1]
    with pytest.raises(ValueError):
        sh.local_ids([2])
    assert pgd.max_over_ranks(3.0) == 3.0


@pytest.mark.parametrize("scaling", ["weak", "strong"])
def test_bench_gpus_2_spawns_ranks(scaling):
    """`bench.py --gpus 2` re-executes itself under torch.distributed.run (one
    process per GPU); the dry run exercises that launch path on CPU: 2 ranks in
    a gloo group, the prompt partition (strong: 256 global prompts split by
    pattern affinity, weak: 256 per rank) and the max-over-ranks reduction."""
    import json
    import subprocess
    import sys
    env = dict(os.environ, MASTER_PORT="29631")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--gpus", "2", "--dry-run", "--scaling",
                        scaling], capture_output=True, text=True, timeout=300, env=env)
    assert r.returncode == 0, r.stderr[-2000:]
    line = json.loads([ln for ln in r.stdout.splitlines() if ln.startswith("{")][-1])
    assert line["n_gpus"] == 2 and line["max_over_ranks"] == 2.0
    if scaling == "strong":
        assert line["prompts_per_rank"] == [128, 128] and line["prompts_covered"] == 256
    else:
        assert line["prompts_per_rank"] == [256, 256] and line["global_tokens"] == 512
