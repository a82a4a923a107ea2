#!/usr/bin/env python
"""Benchmark: PARSE rank-expert hot path on B200 (BASELINE.json metric
"prefill & decode tokens/s, LLaMA-7B SVD@0.6 rank-expert layers, 1-8 B200").

Default workload = BASELINE.json configs[1] ("config2"): LLaMA-7B MLP block
(gate/up 4096->11008, down 11008->4096) at ratio 0.6 (K=1194, r_store=2388),
bf16 storage, f32 accumulation, decode batch 1, the expert subset S taken from
a pattern-cache hit (N=1024 x d=4096 fp64 cache) and reused across every decode
step.  One step = one decode token through the block: up, gate (rank-expert
linears over the packed S arena), silu(gate)*up, down.

  value  -- device-resident tokens/s, whole job (sum over ranks), CUDA-graph
            replay of the step chain, inputs already in HBM; 4 MLP-block weight
            replicas rotated per step (433 MB packed > 126 MB L2).
  e2e    -- the same steps through the public API with the per-step input
            copied H2D from pinned host memory and the result read back D2H
            inside the timed region.
  roofline -- the dominant rank-expert linear forward (up-projection: stage-1
            GEMV + stage-2 GEMV kernels), algorithmic bytes K(m+n)*2 + x + y per
            launch / CUDA-event time, vs MEASURED_PEAKS.json hbm_gbs.
  cpu_baseline -- the reference's own CPU path (oracle/_ref: aggregate_layout +
            aggregated_forward<float>, exec_engine.hpp:113,194) on this host's
            cores, bounded sample.

--impl reference runs only the reference CPU arm (rank 0) and prints its line.
"""
from __future__ import annotations

import argparse
import json
import os
import subprocess
import sys
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "prefill & decode tokens/s, LLaMA-7B SVD@0.6 rank-expert layers, 1–8 B200"
D_MODEL, D_FF, RATIO = 4096, 11008, 0.6
N_CACHE, MIN_SIM, PSI = 1024, 0.80, 0.9
REPLICAS = 4


def shapes():
    from paper_2605_08568_b200 import single_layer_k, store_rank
    out = {}
    for name, (m, n) in {"up": (D_FF, D_MODEL), "gate": (D_FF, D_MODEL), "down": (D_MODEL, D_FF)}.items():
        K = single_layer_k(m, n, RATIO)
        out[name] = (m, n, K, store_rank(K, min(m, n)))
    return out


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled during the timed region."""

    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
         "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
         "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index, self.rows, self.proc = index, [], None

    def __enter__(self):
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--id={self.index}", f"--query-gpu={self.Q}",
                                          "--format=csv,noheader,nounits", "-lms", "100"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.25)
            self.proc.terminate()
            try:
                self.proc.wait(timeout=2)
            except subprocess.TimeoutExpired:
                self.proc.kill()

    def summary(self):
        sm = [float(r[1]) for r in self.rows if len(r) > 8 and r[1].replace(".", "").isdigit()]
        mx = [float(r[2]) for r in self.rows if len(r) > 8 and r[2].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows if len(r) > 8 for i in range(4) if r[5 + i] == "Active"})
        return {"sm_mhz": float(np.median(sm)) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(sm)}


# ----------------------------------------------------------------- reference CPU arm

def reference_arm(steps: int, warmup: int, threads: int | None = None, target_s: float = 0.0):
    """The reference's own served path on host cores: ExecEngine<float>'s
    aggregated_forward over the hit pattern's layout, one decode token = the
    three MLP linears at T=1.  `threads` independent decode streams."""
    from oracle import pyoracle
    kind = "reference" if pyoracle.available("reference") else "port"
    o = pyoracle.Oracle(kind)
    threads = threads or os.cpu_count() or 1
    sh = shapes()
    rng = np.random.default_rng(0)
    aggs = {}
    for name, (m, n, K, r) in sh.items():
        sig = 1.0 / (1.0 + np.arange(r) / 64.0)
        A = rng.standard_normal((m, r)) * (sig / np.sqrt(m))
        B = rng.standard_normal((n, r)) / np.sqrt(n)
        pat = pyoracle.make_patterns(17171, 1, [(r, K)])[0][0]
        aggs[name] = o.aggregate_layout(A, B, [pat], PSI, elem=4)
        del A, B
    xs = [rng.standard_normal((D_MODEL, 1)).astype(np.float32) for _ in range(threads)]

    def token(i):
        x = xs[i]
        u = aggs["up"].forward(0, x)
        g = aggs["gate"].forward(0, x)
        act = (g / (1.0 + np.exp(-g)) * u).astype(np.float32)
        aggs["down"].forward(0, act)

    def run(nsteps):
        ths = [threading.Thread(target=lambda i=i: [token(i) for _ in range(nsteps)]) for i in range(threads)]
        t0 = time.perf_counter()
        for t in ths:
            t.start()
        for t in ths:
            t.join()
        return time.perf_counter() - t0

    run(warmup)
    wall = run(steps)
    toks = steps * threads
    return {"value": toks / wall, "unit": "tokens/s", "cores": threads, "kind": kind,
            "sample": f"{threads} threads x {steps} decode tokens (3 MLP linears, T=1, aggregated_forward<float>)",
            "ms_per_step": wall / steps * 1e3}


# ----------------------------------------------------------------- GPU arm

def build_block(pg, torch, sh, dev, seed):
    """Random-init rank-expert MLP block in the device layout (B^T expert-major,
    A [m, r_store]); A columns scaled by sigma_e = 1/(1+e/64)."""
    g = torch.Generator(device=dev).manual_seed(seed)
    layers = {}
    for name, (m, n, K, r) in sh.items():
        bt = (torch.randn((r, n), generator=g, device=dev) / n ** 0.5).to(torch.bfloat16)
        sig = 1.0 / (1.0 + torch.arange(r, device=dev, dtype=torch.float32) / 64.0)
        a = (torch.randn((m, r), generator=g, device=dev) * sig / m ** 0.5).to(torch.bfloat16)
        layers[name] = pg.FactorizedLayer.from_device(bt, a, K, layer_id=name)
        layers[name]._raw = (bt, a, K)  # for the native fixed-rank SVD baseline
    return layers


def gpu_arm(args, rank, world, local_rank):
    import torch
    import paper_2605_08568_b200 as pg

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    sh = shapes()
    hbm_peak, _, peak_kind = peaks()

    # ---- pattern cache: N entries, each with a SelectionMap for the 3 linears
    pats = pg.make_patterns(17171 + rank, N_CACHE, [(sh[k][3], sh[k][2]) for k in ("up", "gate", "down")])
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    emb = torch.randn((N_CACHE, D_MODEL), generator=gen, device=dev, dtype=torch.float64)
    emb /= emb.norm(dim=1, keepdim=True)
    cache = pg.PatternCache(D_MODEL, N_CACHE, MIN_SIM)
    cache.load([pg.CacheEntry(pg.PromptEmbedding(e), {"up": p[0], "gate": p[1], "down": p[2]})
                for e, p in zip(emb.cpu().numpy(), pats)])
    q = emb[7] + 0.3 / D_MODEL ** 0.5 * torch.randn(D_MODEL, generator=gen, device=dev, dtype=torch.float64)
    q /= q.norm()

    blocks = [build_block(pg, torch, sh, dev, 100 * rank + j) for j in range(REPLICAS)]
    torch.cuda.synchronize()

    # ---- prompt-level work (once per prompt): retrieve -> pack the hit's experts
    t0 = time.perf_counter()
    res = pg.retrieve(cache, q)
    assert res.hit and res.entry == 7, (res.entry, res.similarity)
    aggs = [{k: pg.aggregate_layout(b[k], [res.pattern[k]], PSI) for k in b} for b in blocks]
    torch.cuda.synchronize()
    setup_ms = (time.perf_counter() - t0) * 1e3
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ev0.record()
    for _ in range(10):
        pg.retrieve_device(cache, q)
    ev1.record()
    torch.cuda.synchronize()
    retrieve_us = ev0.elapsed_time(ev1) / 10 * 1e3

    # ---- per-step buffers
    G = 64  # steps per captured graph
    xs = torch.randn((G, D_MODEL), generator=gen, device=dev).to(torch.bfloat16)
    up = torch.empty((G, D_FF), device=dev)
    gt = torch.empty((G, D_FF), device=dev)
    act = torch.empty((G, D_FF), device=dev, dtype=torch.bfloat16)
    y = torch.empty((G, D_MODEL), device=dev)
    x_host = torch.empty((G, D_MODEL), dtype=torch.bfloat16).pin_memory()
    x_host.copy_(xs.cpu())
    y_host = torch.empty((G, D_MODEL), dtype=torch.float32).pin_memory()

    def step(i, host_io, fused=True):
        a = aggs[i % REPLICAS]
        if host_io == "zc":  # zero-copy: the MLP kernel reads x from / writes y to pinned host memory itself
            pg.mlp_forward(a["up"], a["gate"], a["down"], 0, x_host[i], out=y_host[i], act=act[i])
            return
        if host_io:  # per-token input H2D from pinned memory, as a PDL-chained kernel
            pg.copy_io(xs[i], x_host[i])
        if fused:  # K6: whole MLP block in one kernel (up/gate fused B side, silu epilogue, down)
            pg.mlp_forward(a["up"], a["gate"], a["down"], 0, xs[i], out=y[i], act=act[i])
        else:      # aggregated-only: one chain kernel per linear + silu kernel
            pg.aggregated_forward(a["up"], 0, xs[i], out=up[i])
            pg.aggregated_forward(a["gate"], 0, xs[i], out=gt[i])
            pg.silu_mul(gt[i], up[i], out=act[i])
            pg.aggregated_forward(a["down"], 0, act[i], out=y[i])
        if host_io:  # result D2H into pinned memory
            pg.copy_io(y_host[i], y[i])

    stream = torch.cuda.Stream(device=dev)
    graphs = {}
    for key in ((False, True), (True, True), (False, False), ("zc", True)):
        host_io, fused = key
        with torch.cuda.stream(stream):
            for i in range(G):  # warm (kernel attributes, pools) outside capture
                step(i, host_io, fused)
        stream.synchronize()
        g = torch.cuda.CUDAGraph()
        n0 = pg.launch_count()
        with torch.cuda.graph(g, stream=stream):
            for i in range(G):
                step(i, host_io, fused)
        graphs[key] = (g, pg.launch_count() - n0)
    torch.cuda.synchronize()

    def timed(host_io, steps, fused=True):
        g, _ = graphs[(host_io, fused)]
        reps = max(1, steps // G)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            for _ in range(max(1, args.warmup // G + 1)):
                g.replay()
        stream.synchronize()
        if world > 1:
            torch.distributed.barrier()
        torch.cuda.synchronize()
        with torch.cuda.stream(stream):
            s0.record(stream)
            for _ in range(reps):
                g.replay()
            s1.record(stream)
        torch.cuda.synchronize()
        if world > 1:
            torch.distributed.barrier()
        ms = s0.elapsed_time(s1)
        if world > 1:
            t = torch.tensor([ms], device=dev, dtype=torch.float64)
            torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
            ms = float(t.item())
        return ms, reps * G

    # ---- baselines in the same run: native fixed-rank SVD, i.e.
    # the static prefix A[:, :K] (B[:, :K]^T x) through cuBLAS (torch.matmul),
    # and the dense layer W x, both bf16, same replicas, same graph recipe
    def cublas_graph(mats):
        xb = torch.randn((G, D_MODEL), generator=gen, device=dev).to(torch.bfloat16)

        def one(i):
            w = mats[i % REPLICAS]
            if len(w) == 6:  # fixed-rank SVD: B_K^T x then A_K z per linear
                bu, au, bg, ag, bd, ad = w
                u = au @ (bu @ xb[i])
                gg = ag @ (bg @ xb[i])
                return ad @ (bd @ (torch.nn.functional.silu(gg) * u))
            wu, wg, wd = w
            return wd @ (torch.nn.functional.silu(wg @ xb[i]) * (wu @ xb[i]))

        with torch.cuda.stream(stream):
            for i in range(G):
                one(i)
        stream.synchronize()
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr, stream=stream):
            for i in range(G):
                one(i)
        s0, s1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(stream):
            gr.replay()
            s0.record(stream)
            for _ in range(8):
                gr.replay()
            s1.record(stream)
        torch.cuda.synchronize()
        return 8 * G / (s0.elapsed_time(s1) * 1e-3) * world

    svd = []
    for b in blocks:
        w = []
        for nm in ("up", "gate", "down"):
            bt, a, K_ = b[nm]._raw
            w += [bt[:K_].contiguous(), a[:, :K_].contiguous()]
        svd.append(tuple(w))
    svd_tok_s = cublas_graph(svd)
    del svd
    dense = [tuple(torch.randn(shp, generator=gen, device=dev).to(torch.bfloat16) / 64
                   for shp in ((D_FF, D_MODEL), (D_FF, D_MODEL), (D_MODEL, D_FF))) for _ in range(REPLICAS)]
    dense_tok_s = cublas_graph(dense)
    del dense
    torch.cuda.empty_cache()

    with ClockSampler(local_rank) as clk:
        ms, nsteps = timed(False, args.steps)
    ms_e2e, nsteps_e2e = timed(True, args.steps)
    ms_unf, nsteps_unf = timed(False, args.steps, fused=False)
    ms_zc, nsteps_zc = timed("zc", args.steps)
    # e2e = the faster of the two host-I/O recipes (both move the same bytes
    # between pinned host memory and the GPU inside the timed region)
    e2e_kind = "zero-copy (kernel reads x / writes y in pinned host memory)"
    if ms_e2e < ms_zc:
        e2e_kind = "pg_copy_io kernels (H2D x, D2H y) chained by PDL"
    ms_e2e_best, nsteps_e2e_best = (ms_zc, nsteps_zc) if ms_zc <= ms_e2e else (ms_e2e, nsteps_e2e)
    launches_per_step = graphs[(False, True)][1] / G

    # ---- roofline: the dominant (only) kernel of the step is k_chain<bf16>, the
    # fused MLP block; one launch per step, timed by CUDA events on its stream
    # over the timed region.  Algorithmic bytes = sum_l K_l (m_l + n_l) * 2 (the
    # selected experts' U and V rows) + x, act (write+read) and y.
    traffic = None  # dram read+write bytes per launch of k_chain from the committed ncu --set full capture
    tp = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp):
        traffic = json.load(open(tp)).get("k_chain<bf16>")
    lin_bytes = {k: K_ * (m_ + n_) * 2 for k, (m_, n_, K_, _) in sh.items()}
    step_bytes = sum(lin_bytes.values()) + D_MODEL * 2 + D_FF * 2 * 2 + D_MODEL * 4
    step_us = ms / nsteps * 1e3
    achieved = step_bytes / (step_us * 1e-6) / 1e9
    tok_s = nsteps / (ms * 1e-3) * world
    out = {
        "metric": METRIC, "value": tok_s, "unit": "tokens/s", "n_gpus": world, "steps": nsteps,
        "warmup": args.warmup, "ms_per_step": ms / nsteps, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "bf16", "data": "synthetic (random-init rank-expert factors, seeded)",
        "config": {"workload": "config2: LLaMA-7B MLP block (gate/up 4096->11008, down 11008->4096) ratio 0.6 "
                               "K=1194 r_store=2388, decode batch 1, S from a pattern-cache hit reused across steps",
                   "cache": f"N={N_CACHE} x d={D_MODEL} f64, min_similarity {MIN_SIM}, hit entry {res.entry}",
                   "l2": f"{REPLICAS} MLP-block weight replicas rotated per step "
                         f"({REPLICAS * step_bytes / 1e6:.0f} MB packed > 126 MB L2)",
                   "parallelism": f"dp{world} (independent decode streams per GPU)",
                   "psi": PSI, "graph": f"CUDA graph of {G} steps replayed"},
        "e2e": {"value": nsteps_e2e_best / (ms_e2e_best * 1e-3) * world, "unit": "tokens/s",
                "h2d_bytes_per_step": D_MODEL * 2, "d2h_bytes_per_step": D_MODEL * 4, "io": e2e_kind},
        "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                     "frac": achieved / hbm_peak, "traffic": traffic,
                     "kernel": "k_chain<bf16> (fused MLP block: up+gate stage 1, grid barrier, stage 2 + "
                               "silu epilogue, down stage 1/2; 1 launch per step)",
                     "alg_bytes_per_launch": step_bytes, "avg_us": step_us, "peak_kind": peak_kind},
        "variants": {"aggregated_fused_tok_s": tok_s,
                     "aggregated_only_tok_s": nsteps_unf / (ms_unf * 1e-3) * world,
                     "e2e_copy_io_tok_s": nsteps_e2e / (ms_e2e * 1e-3) * world,
                     "e2e_zero_copy_tok_s": nsteps_zc / (ms_zc * 1e-3) * world,
                     "launches_per_step": {"fused": launches_per_step,
                                           "unfused": graphs[(False, False)][1] / G}},
        "gpu_launches": int(launches_per_step * nsteps),
        "clocks": clk.summary(),
        "prefill_setup": {"retrieve_us": retrieve_us, "retrieve_plus_pack_ms_host": setup_ms},
        "baselines": {"native_fixed_rank_svd_cublas_tok_s": svd_tok_s, "dense_cublas_tok_s": dense_tok_s,
                      "note": "static prefix A[:, :K](B[:, :K]^T x) and dense W x, bf16 torch.matmul, "
                              "same replicas, CUDA graph of 64 steps"},
    }
    if args.prefill:
        del blocks, aggs
        torch.cuda.empty_cache()
        out["prefill"] = prefill_arm(pg, torch, dev, world)
        torch.cuda.empty_cache()
    if args.decode_batch:
        out["decode_batch"] = decode_batch_arm(pg, torch, dev, world, hbm_peak)
    return out


def decode_batch_arm(pg, torch, dev, world, hbm_peak, P=256, layers=32, distinct=4):
    """BASELINE config 4 (per GPU, data-parallel): a 32-layer LLaMA-7B-shaped
    stack of rank-expert linears decoding 256 prompts x 1 token, each prompt
    with its own selection per linear (the reference's pattern generator).
    Union-masked: every linear reads its stored experts once for the whole
    batch (two tcgen05 GEMMs, the per-token mask in the first's epilogue).
    `distinct` layer weight sets (each 324 MB > L2) are cycled through the 32
    layers; attention and norms are outside the path."""
    lin = {"q": (D_MODEL, D_MODEL), "k": (D_MODEL, D_MODEL), "v": (D_MODEL, D_MODEL), "o": (D_MODEL, D_MODEL),
           "up": (D_FF, D_MODEL), "gate": (D_FF, D_MODEL), "down": (D_MODEL, D_FF)}
    dims = [(pg.store_rank(pg.single_layer_k(m, n, RATIO), n), pg.single_layer_k(m, n, RATIO)) for m, n in lin.values()]
    pats = pg.make_patterns(17171, P, dims)  # the reference's generator (pg_make_patterns, same bits)
    g = torch.Generator(device=dev).manual_seed(11)
    stack = []
    for _ in range(distinct):
        lay = {}
        for li, (nm, (m, n)) in enumerate(lin.items()):
            r, K = dims[li]
            bt = (torch.randn(r, n, device=dev, generator=g) / n ** 0.5).to(torch.bfloat16)
            a = (torch.randn(m, r, device=dev, generator=g) / m ** 0.5).to(torch.bfloat16)
            L = pg.FactorizedLayer.from_device(bt, a, K, layer_id=nm)
            lay[nm] = (L, pg.SelectionBatch(L, [p[li] for p in pats]))
        stack.append(lay)
    X = {n: torch.randn(P, n, device=dev, generator=g).to(torch.bfloat16) for n in (D_MODEL, D_FF)}
    tp = torch.arange(P, device=dev, dtype=torch.int32)  # prompt q -> its own selection q

    Yl = {nm: torch.empty(P, m, device=dev, dtype=torch.bfloat16) for nm, (m, n) in lin.items()}
    groups = (("q", "k", "v"), ("o",), ("up", "gate"), ("down",))  # linears sharing an input: one launch per stage

    def step():
        for li in range(layers):
            lay = stack[li % distinct]
            for grp in groups:
                pg.module_forward_union([lay[g][0] for g in grp], [lay[g][1] for g in grp], tp, X[lin[grp[0]][1]],
                                        out_dtype=torch.bfloat16, outs=[Yl[g] for g in grp])

    st = torch.cuda.Stream(device=dev)
    with torch.cuda.stream(st):
        step()
    st.synchronize()
    gr = torch.cuda.CUDAGraph()
    n0 = pg.launch_count()
    with torch.cuda.graph(gr, stream=st):
        step()
    launches = pg.launch_count() - n0
    reps = 5
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if world > 1:
        torch.distributed.barrier()
    with torch.cuda.stream(st):
        gr.replay()
        e0.record(st)
        for _ in range(reps):
            gr.replay()
        e1.record(st)
    torch.cuda.synchronize()
    ms = max_over_ranks_ms(torch, e0.elapsed_time(e1) / reps, dev, world)
    byt = layers * sum(dims[i][0] * (m + n) * 2 for i, (m, n) in enumerate(lin.values()))
    fl = layers * 2 * P * sum(dims[i][0] * (m + n) for i, (m, n) in enumerate(lin.values()))
    return {"workload": f"config4: {layers}-layer LLaMA-7B-shaped stack, {P} prompts x 1 decode token, "
                        f"{P} heterogeneous selections per linear (reference generator, seed 17171), "
                        f"union-masked tcgen05 GEMMs (q/k/v and up/gate grouped per stage); {distinct} distinct layer "
                        f"weight sets cycled (each > L2)",
            "tokens_per_s": P / (ms * 1e-3) * world, "ms_per_step": ms, "launches_per_step": launches,
            "roofline": {"bound": "hbm", "achieved": byt / (ms * 1e-3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                         "frac": byt / (ms * 1e-3) / 1e9 / hbm_peak, "bytes_per_step": byt,
                         "tensor_tflops": fl / (ms * 1e-3) / 1e12}}


def max_over_ranks_ms(torch, ms, dev, world):
    """Device time of a secondary arm: the slowest rank's (like the headline)."""
    if world <= 1:
        return ms
    t = torch.tensor([ms], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def prefill_arm(pg, torch, dev, world, P=16, T=2048):
    """BASELINE config 3: one LLaMA-7B decoder layer's 7 rank-expert linears,
    16 prompts x 2048 tokens, each prompt routed on device to its own expert
    subset (bit-exact router), packed once, then grouped tcgen05 GEMMs.
    Timed: routing (7 routers, 16 prompts) + the 7 prefill linears."""
    lin = {"q": (D_MODEL, D_MODEL), "k": (D_MODEL, D_MODEL), "v": (D_MODEL, D_MODEL), "o": (D_MODEL, D_MODEL),
           "up": (D_FF, D_MODEL), "gate": (D_FF, D_MODEL), "down": (D_MODEL, D_FF)}
    g = torch.Generator(device=dev).manual_seed(7)
    X = torch.randn(P * T, D_MODEL, device=dev, generator=g).to(torch.bfloat16)
    X2 = torch.randn(P * T, D_FF, device=dev, generator=g).to(torch.bfloat16)
    offs = [i * T for i in range(P + 1)]
    layers, routers, outs, flops = {}, {}, {}, 0
    for nm, (m, n) in lin.items():
        K = pg.single_layer_k(m, n, RATIO)
        r = pg.store_rank(K, min(m, n))
        bt = (torch.randn((r, n), generator=g, device=dev) / n ** 0.5).to(torch.bfloat16)
        a = (torch.randn((m, r), generator=g, device=dev) / m ** 0.5).to(torch.bfloat16)
        layers[nm] = (pg.FactorizedLayer.from_device(bt, a, K), K)
        routers[nm] = pg.RouterParams(torch.randn((r, n), generator=g, device=dev, dtype=torch.float64))
        outs[nm] = torch.empty(P * T, m, device=dev, dtype=torch.bfloat16)
        flops += 2 * P * T * K * (m + n)
    # routing (timed separately): select_topk(score(mean_pool(x_p))) per prompt.
    # Linears sharing an input pool it once (toy_lm.hpp:220-249: q/k/v and
    # up/gate read hn, o the attention output, down act), then every router
    # scores its own pooled input.
    Xo = torch.randn(P * T, D_MODEL, device=dev, generator=g).to(torch.bfloat16)
    src = {"q": X, "k": X, "v": X, "up": X, "gate": X, "o": Xo, "down": X2}
    sels = {}
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def route_all():
        pooled = {id(x): pg.mean_pool(x, layout="token", offsets=offs) for x in (X, Xo, X2)}
        for nm in lin:
            sels[nm] = pg.route_select_pooled(routers[nm], pooled[id(src[nm])], layers[nm][1])

    for _ in range(3):  # warm: scratch pools, kernel attributes
        route_all()
    torch.cuda.synchronize()
    route_reps = 5
    if world > 1:
        torch.distributed.barrier()
    e0.record()
    for _ in range(route_reps):
        route_all()
    e1.record()
    torch.cuda.synchronize()
    route_ms = max_over_ranks_ms(torch, e0.elapsed_time(e1) / route_reps, dev, world)
    # pack each prompt's experts once (serving: after routing / a cache hit)
    t0 = time.perf_counter()
    aggs = {nm: [pg.aggregate_layout(layers[nm][0], [pg.RankSelection(sels[nm][p].cpu().numpy())], PSI)
                 for p in range(P)] for nm in lin}
    torch.cuda.synchronize()
    pack_ms = (time.perf_counter() - t0) * 1e3

    def layer_step():
        for nm in lin:
            pg.prefill_batched(aggs[nm], offs, src[nm], out_dtype=torch.bfloat16, out=outs[nm])

    for _ in range(2):
        layer_step()
    torch.cuda.synchronize()
    reps = 5
    if world > 1:
        torch.distributed.barrier()
    e0.record()
    for _ in range(reps):
        layer_step()
    e1.record()
    torch.cuda.synchronize()
    ms = max_over_ranks_ms(torch, e0.elapsed_time(e1) / reps, dev, world)
    _, tflops_peak, peak_kind = peaks()
    achieved = flops / (ms * 1e-3) / 1e12
    return {"workload": "config3: LLaMA-7B decoder layer (q,k,v,o,gate,up,down) ratio 0.6, 16 prompts x 2048 "
                        "tokens, per-prompt expert subsets routed on device, bf16 (z rounded to bf16 between stages)",
            "tokens_per_s": P * T / ((ms + route_ms) * 1e-3) * world,
            "gemm_tokens_per_s": P * T / (ms * 1e-3) * world,
            "ms_per_layer": ms, "route_ms": route_ms, "pack_ms_host": pack_ms,
            "roofline": {"bound": "tensor", "achieved": achieved, "peak": tflops_peak, "unit": "TFLOP/s",
                         "frac": achieved / tflops_peak, "flops_per_layer": flops, "peak_kind": peak_kind,
                         "kernel": "k_umma_grouped (tcgen05.mma kind::f16, TMA, TMEM; 2 grouped launches per linear)"}}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20000)
    ap.add_argument("--warmup", type=int, default=200)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--cpu-steps", type=int, default=3)
    ap.add_argument("--prefill", type=int, default=1, help="also measure config-3 prefill (secondary)")
    ap.add_argument("--decode-batch", type=int, default=1,
                    help="also measure config-4 batched heterogeneous decode (secondary)")
    args = ap.parse_args()
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))

    if args.impl == "reference":
        if rank != 0:
            return
        st = max(1, min(args.steps, 20))
        wu = max(1, min(args.warmup, 3))  # bounded CPU sample: the whole arm stays within minutes
        ref = reference_arm(st, wu)
        line = {"metric": METRIC, "value": ref["value"], "unit": "tokens/s", "n_gpus": 0, "steps": st,
                "warmup": wu, "ms_per_step": ref["ms_per_step"],
                "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "impl": "reference",
                "config": {"workload": "config2: LLaMA-7B MLP block decode batch 1 (reference CPU "
                                       "aggregated_forward<float>, exec_engine.hpp:194)"},
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")},
                "e2e": {"value": ref["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0,
                        "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    if world > 1:
        import torch
        import torch.distributed as dist
        torch.cuda.set_device(local_rank)
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = gpu_arm(args, rank, world, local_rank)
    if rank == 0:
        if world == 1 and args.cpu_steps > 0:
            ref = reference_arm(args.cpu_steps, 1)
            out["cpu_baseline"] = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(out), flush=True)
    if world > 1:
        import torch.distributed as dist
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
