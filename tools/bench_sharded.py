"""Expert-sharded mode (BASELINE config 5 shapes: LLaMA-13B up-projection
13824 x 5120 at ratio 0.4, K=2241, r_store=4482), one process per GPU:
experts e mod G live on rank e; each rank computes its partial through the
rank-expert kernels and one NCCL all-reduce sums the partials.  Mixed work:
a T=256 prefill chunk and T=1 decode steps with the prompt's frozen selection.
Device time, max over ranks.  Weights are random (seeded); the all-reduced
output is checked against a single-rank reference computation on rank 0.

    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port 29600 tools/bench_sharded.py
"""
import json
import os
import sys

import numpy as np
import torch
import torch.distributed as dist

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2605_08568_b200 as pg  # noqa: E402
from paper_2605_08568_b200 import dist as pgd  # noqa: E402


def main():
    rank, world = int(os.environ.get("RANK", 0)), int(os.environ.get("WORLD_SIZE", 1))
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", 0)))
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", int(os.environ.get("LOCAL_RANK", 0))))
    m, n = 13824, 5120
    K = pg.single_layer_k(m, n, 0.4)
    r = pg.store_rank(K, n)
    rng = np.random.default_rng(5)
    sig = 1.0 / (1.0 + np.arange(r) / 64.0)
    A = rng.standard_normal((m, r)) * (sig / np.sqrt(m))
    B = rng.standard_normal((n, r)) / np.sqrt(n)
    sel = pg.RankSelection(np.sort(rng.choice(r, K, replace=False)).astype(np.uint32))
    lin = pgd.ShardedLinear(A, B, world, rank, dtype="bf16")
    xp = torch.from_numpy(rng.standard_normal((n, 256))).cuda().to(torch.bfloat16)
    xd = torch.from_numpy(rng.standard_normal((n, 1))).cuda().to(torch.bfloat16)

    def step():
        lin.forward(sel, xp)           # prefill chunk
        for _ in range(8):
            lin.forward(sel, xd)       # decode steps reusing S

    for _ in range(3):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 10
    e0.record()
    for _ in range(reps):
        step()
    e1.record()
    torch.cuda.synchronize()
    ms = pgd.max_over_ranks(e0.elapsed_time(e1) / reps, device=torch.device("cuda"))
    y = lin.forward(sel, xd).double().cpu().numpy()
    full = pg.FactorizedLayer(A, B, K, dtype="bf16")
    yr = pg.masked_forward(full, sel, xd, out_dtype=torch.float32).double().cpu().numpy()
    if rank == 0:
        rel = float(np.abs(y - yr).max() / np.abs(yr).max())
        print(json.dumps({"workload": "config5 shapes: 13824x5120 ratio 0.4 expert-sharded (e mod G)",
                          "world": world, "ms_per_step": ms, "step": "1 x T=256 prefill + 8 x T=1 decode",
                          "tokens_per_s": (256 + 8) / (ms * 1e-3), "rel_vs_single_gpu": rel,
                          "per_rank_weight_bytes": int((lin.shard.A.shape[1]) * (m + n) * 2)}))
    # decode steps with the all-reduce fused into the kernel over peer memory
    if world > 1:
        fused = pgd.PeerReduceLinear(A, B, world, rank, dtype="bf16", group=dist.group.WORLD)
    else:
        fused = pgd.PeerReduceLinear.local_group(A, B, 1, dtype="bf16")[0]
    fused.prepare(sel)
    for _ in range(3):
        fused.forward(sel, xd)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    e0.record()
    for _ in range(reps * 8):
        fused.forward(sel, xd)
    e1.record()
    torch.cuda.synchronize()
    fus_us = pgd.max_over_ranks(e0.elapsed_time(e1) / (reps * 8) * 1e3, device=torch.device("cuda"))
    yf = fused.forward(sel, xd).double().cpu().numpy()
    if rank == 0:
        relf = float(np.abs(yf - yr[:, 0]).max() / np.abs(yr).max())
        print(json.dumps({"fused_peer_decode_us_per_token": fus_us, "rel_vs_single_gpu": relf}))
    fused.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
