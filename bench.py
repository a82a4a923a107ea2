#!/usr/bin/env python
"""Benchmark: PARSE rank-expert hot path on B200 (BASELINE.json metric
"prefill & decode tokens/s, LLaMA-7B SVD@0.6 rank-expert layers, 1-8 B200").

Headline workload = BASELINE.json configs[3] ("config4"), the config the metric
is quoted on across 1-8 GPUs and the largest single-GPU configuration: a
32-layer LLaMA-7B-shaped stack of rank-expert linears (q/k/v/o 4096x4096, gate/up
4096->11008, down 11008->4096, ratio 0.6: K = 819 / 1194, r_store = 1638 / 2388),
bf16 storage with f32 accumulation, decoding a batch of 256 heterogeneous prompts,
each prompt with its own expert subset per linear (the reference's prefix-biased
pattern generator).  One step = one decode token for every prompt through all
32 x 7 linears (q/k/v and up/gate sharing an input run as one grouped launch per
GEMM stage; o reads v's output and down reads up's output as stand-ins for the
attention / SiLU glue, which is outside the path).  32 distinct layer weight
sets (10.36 GB): every byte streams from HBM each step (inputs >> L2, no flush).

  value     -- tokens/s of the whole job (sum over ranks), device time (CUDA
               events, max over ranks) over exactly --steps graph replays of the
               step after --warmup untimed ones; the median per-step window is
               reported beside it.
  e2e       -- the same steps through the public API with the step's input
               hidden states copied H2D from pinned host memory and the last
               layer's output read back D2H inside the timed region.
  roofline  -- HBM: stored expert bytes per step (every linear reads its r_store
               experts once for the whole batch) / step time, vs MEASURED_PEAKS;
               the dominant launch (up+gate stage 2) timed alone beside it.
  cpu_baseline / --impl reference -- the reference's own served path
               (aggregate_layout + aggregated_forward<float>, exec_engine.hpp:
               112-164,193-236, compiled from /root/reference into oracle/_ref)
               on the host cores: one prompt per thread through one sampled layer
               (7 linears, T = 1), extrapolated to the 32-layer stack.
Secondary objects (same line): config2 decode batch 1 (the fused MLP-block
decode kernel), config3 prefill (routing + pack + grouped tcgen05 GEMMs), config1
fp32 (routed q_proj, 128-token prefill + 32 decode steps, the reference CPU path
run in full in the same process).

--gpus N (N > 1) without torchrun re-executes itself under
torch.distributed.run; --scaling weak (default: 256 prompts per GPU) or strong
(256 global prompts partitioned over the ranks with pattern affinity).
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
N_LAYERS, N_PROMPTS = 32, 256
LIN = {"q": (D_MODEL, D_MODEL), "k": (D_MODEL, D_MODEL), "v": (D_MODEL, D_MODEL), "o": (D_MODEL, D_MODEL),
       "up": (D_FF, D_MODEL), "gate": (D_FF, D_MODEL), "down": (D_MODEL, D_FF)}
GROUPS = (("q", "k", "v"), ("o",), ("up", "gate"), ("down",))  # linears sharing an input: one launch per stage
SRC = {"q": "x", "k": "x", "v": "x", "o": "v", "up": "o", "gate": "o", "down": "up"}  # stand-in data flow


def dims(m, n):
    from paper_2605_08568_b200 import single_layer_k, store_rank
    K = single_layer_k(m, n, RATIO)
    return store_rank(K, min(m, n)), K


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        j = json.load(open(p))
        return float(j["hbm_gbs"]), float(j["bf16_tflops"]), "measured"
    return 6650.0, 1590.0, "fallback"


def cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return "unknown"


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
                                          "--format=csv,noheader,nounits", "-lms", "50"],
                                         stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            time.sleep(0.3)  # first sample before the timed region starts
        except FileNotFoundError:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.rows.append([c.strip() for c in line.split(",")])

    def __exit__(self, *a):
        if self.proc:
            time.sleep(0.15)
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


def max_over_ranks(torch, v, dev, world):
    if world <= 1:
        return v
    t = torch.tensor([float(v)], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    return float(t.item())


def barrier(torch, world):
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()


# ======================================================================= CPU (reference)

def reference_config4(threads: int | None = None, repeats: int = 3):
    """The reference's served path for config 4 on the host cores: ExecEngine<float>
    (aggregate_layout over the served patterns, exec_engine.hpp:112-164, then
    aggregated_forward<float>, :193-236) for one decode token (T = 1) of one
    prompt per thread through the 7 linears of one sampled layer; median of
    `repeats` passes (time_engine_pass recipe, exec_engine.hpp:362-379), x 32
    layers.  Packing is per prompt (amortised over its decode) and not timed."""
    from oracle import pyoracle
    kind = "reference" if pyoracle.available("reference") else "port"
    o = pyoracle.Oracle(kind)
    threads = threads or os.cpu_count() or 1
    ldims = [dims(m, n) for m, n in LIN.values()]
    pats = pyoracle.make_patterns(17171, threads, ldims)
    rng = np.random.default_rng(0)
    aggs = {}
    t0 = time.perf_counter()
    for li, (nm, (m, n)) in enumerate(LIN.items()):
        r, K = ldims[li]
        A = rng.standard_normal((m, r)) / np.sqrt(K)
        B = rng.standard_normal((n, r)) / np.sqrt(n)
        aggs[nm] = o.aggregate_layout(A, B, [p[li] for p in pats], PSI, elem=4)
        del A, B
    pack_s = time.perf_counter() - t0
    xs = [{n: rng.standard_normal((n, 1)).astype(np.float32) for n in (D_MODEL, D_FF)} for _ in range(threads)]
    times = [[0.0] * repeats for _ in range(threads)]

    def work(i):
        for rep in range(repeats):
            t = time.perf_counter()
            for nm, (m, n) in LIN.items():
                aggs[nm].forward(i, xs[i][n])
            times[i][rep] = time.perf_counter() - t

    ths = [threading.Thread(target=work, args=(i,)) for i in range(threads)]
    w0 = time.perf_counter()
    for t in ths:
        t.start()
    for t in ths:
        t.join()
    wall = time.perf_counter() - w0
    layer_s = float(np.median([np.median(t) for t in times]))  # one prompt, one layer, T = 1
    tok_s = threads / (N_LAYERS * layer_s)
    return {"value": tok_s, "unit": "tokens/s", "cores": threads, "kind": kind,
            "sample": f"{threads} threads, one prompt each (its own pattern), one decode token through the 7 "
                      f"linears of 1 of {N_LAYERS} layers (aggregated_forward<float>, T=1), median of {repeats} "
                      f"passes; extrapolated x{N_LAYERS} layers",
            "extrapolated": True, "cpu_model": cpu_model(), "nproc": os.cpu_count(),
            "ms_per_layer_per_prompt": layer_s * 1e3, "pack_s": pack_s, "wall_s": wall}


# ======================================================================= config 4 (headline)

def build_stack(pg, torch, dev, prompts, layers):
    """32 distinct layers of rank-expert linears (B^T expert-major, A [m, r_store],
    A scaled 1/sqrt(K) so activations stay O(1) through the stack) and, per layer
    and linear, the selections of this rank's prompts as device masks."""
    g = torch.Generator(device=dev).manual_seed(11)
    ldims = [dims(m, n) for m, n in LIN.values()]
    stack = []
    for li in range(layers):
        pats = pg.make_patterns(17171 + li, N_PROMPTS, ldims)  # the reference's generator (same bits)
        lay = {}
        for j, (nm, (m, n)) in enumerate(LIN.items()):
            r, K = ldims[j]
            bt = (torch.randn(r, n, device=dev, generator=g) / n ** 0.5).to(torch.bfloat16)
            a = (torch.randn(m, r, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
            L = pg.FactorizedLayer.from_device(bt, a, K, layer_id=f"b{li}.{nm}")
            lay[nm] = (L, pg.SelectionBatch(L, [pats[p][j] for p in prompts]))
        stack.append(lay)
    return stack, ldims


def config4_config(layers, prompts_per_gpu, world, scaling):
    """The config-4 workload description, identical in both arms (ours and
    --impl reference): what is computed, not how."""
    glob = N_PROMPTS if scaling == "strong" else prompts_per_gpu * world
    return {"workload": f"config4: {layers}-layer LLaMA-7B-shaped stack of rank-expert linears (q/k/v/o 4096x4096, "
                        f"gate/up 4096->11008, down 11008->4096) ratio {RATIO}, one decode token for each of "
                        f"{prompts_per_gpu} heterogeneous prompts per GPU, each prompt with its own expert subset per "
                        f"linear (reference pattern generator, seed 17171)",
            "global_batch": glob, "prompts_per_gpu": prompts_per_gpu, "layers": layers,
            "parallelism": f"dp{world} ({scaling} scaling; replicated weights, no collective)"}


def config4_arm(args, rank, world, local_rank):
    import torch
    import paper_2605_08568_b200 as pg
    from paper_2605_08568_b200 import dist as pgd

    dev = torch.device("cuda", local_rank)
    hbm_peak, _, peak_kind = peaks()
    if args.scaling == "strong":  # 256 global prompts, pattern affinity (all distinct here: contiguous)
        prompts = pgd.partition_by_pattern(list(range(N_PROMPTS)), world)[rank]
    else:
        prompts = list(range(N_PROMPTS))
    Pl = len(prompts)
    stack, ldims = build_stack(pg, torch, dev, prompts, args.layers)
    tp = torch.arange(Pl, device=dev, dtype=torch.int32)  # token t -> its prompt's selection t
    g = torch.Generator(device=dev).manual_seed(5)
    x0 = torch.randn(Pl, D_MODEL, device=dev, generator=g).to(torch.bfloat16)
    # the whole step as ONE persistent launch (union_prog.cu): per-layer
    # activation buffers (a program writes each buffer once), layer l+1 reads
    # layer l's output tile by tile
    prog = pg.UnionProgram(Pl)
    bufs = []
    src = x0
    for lay in stack:
        b = {"x": src}
        for grp in GROUPS:
            for nm in grp:
                b[nm] = torch.empty(Pl, LIN[nm][0], device=dev, dtype=torch.bfloat16)
            prog.add_module([lay[nm][0] for nm in grp], [lay[nm][1] for nm in grp], b[SRC[grp[0]]],
                            [b[nm] for nm in grp])
        bufs.append(b)
        src = b["down"]
    y_dev = bufs[-1]["down"]
    x_host = torch.empty(Pl, D_MODEL, dtype=torch.bfloat16).pin_memory()
    x_host.copy_(x0.cpu())
    y_host = torch.empty(Pl, D_MODEL, dtype=torch.bfloat16).pin_memory()

    def step(host_io):
        if host_io:
            pg.copy_io(x0, x_host)      # the step's input hidden states, H2D
        prog.run(tp)
        if host_io:
            pg.copy_io(y_host, y_dev)   # the last layer's output, D2H

    def modules():  # the same step as per-module launches (2 union GEMM launches per module)
        for lay, b in zip(stack, bufs):
            for grp in GROUPS:
                pg.module_forward_union([lay[n][0] for n in grp], [lay[n][1] for n in grp], tp, b[SRC[grp[0]]],
                                        out_dtype=torch.bfloat16, outs=[b[n] for n in grp])

    st = torch.cuda.Stream(device=dev)
    graphs = {}
    for key, fn in ((False, lambda: step(False)), (True, lambda: step(True)), ("modules", modules)):
        with torch.cuda.stream(st):
            fn()  # sizes workspaces / pools outside capture
        st.synchronize()
        gr = torch.cuda.CUDAGraph()
        n0 = pg.launch_count()
        with torch.cuda.graph(gr, stream=st):
            fn()
        graphs[key] = (gr, pg.launch_count() - n0)

    def timed(key, steps, warmup):
        gr = graphs[key][0]
        with torch.cuda.stream(st):
            for _ in range(warmup):
                gr.replay()
        barrier(torch, world)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(steps + 1)]
        with torch.cuda.stream(st):
            ev[0].record(st)
            for i in range(steps):
                gr.replay()
                ev[i + 1].record(st)
        barrier(torch, world)
        per = [ev[i].elapsed_time(ev[i + 1]) for i in range(steps)]
        total = ev[0].elapsed_time(ev[steps])
        return max_over_ranks(torch, total, dev, world), max_over_ranks(torch, float(np.median(per)), dev, world)

    with ClockSampler(local_rank) as clk:
        ms_total, ms_med = timed(False, args.steps, args.warmup)
    ms_e2e, ms_e2e_med = timed(True, args.steps, max(1, args.warmup // 2))
    _, ms_modules = timed("modules", min(args.steps, 10), 2)
    launches = graphs[False][1]
    # the modules path and the program must agree (the same step, two schedules)
    with torch.cuda.stream(st):
        graphs["modules"][0].replay()
        ref = y_dev.float().clone()
        graphs[False][0].replay()
    st.synchronize()
    agree = float((y_dev.float() - ref).abs().max() / ref.abs().max().clamp_min(1e-30))
    # native fixed-rank SVD on the GPU (north star): the same 32-layer step with
    # every linear's static prefix y = A[:, :K] (B[:, :K]^T x) through cuBLAS
    # (torch.matmul, bf16), one selection for all prompts, K experts read
    # (contiguous copies, K padded to a multiple of 8 with zero experts so every
    # row is 16-byte aligned for cuBLAS)
    svd = {}
    fixed = []
    for lay in stack:
        fl = {}
        for nm in LIN:
            L = lay[nm][0]
            bt, a = L._keep
            K = L.K
            K8 = (K + 7) // 8 * 8
            bK = torch.zeros(K8, bt.shape[1], device=dev, dtype=bt.dtype)
            bK[:K] = bt[:K]
            aK = torch.zeros(a.shape[0], K8, device=dev, dtype=a.dtype)
            aK[:, :K] = a[:, :K]
            fl[nm] = (bK, aK)
        fixed.append(fl)

    def svd_step():
        for fl, b in zip(fixed, bufs):
            h = {"x": b["x"]}
            for nm in LIN:
                bK, aK = fl[nm]
                h[nm] = torch.matmul(torch.matmul(h[SRC[nm]], bK.t()), aK.t())
            svd["y"] = h["down"]

    with torch.cuda.stream(st):
        svd_step()
    st.synchronize()
    gsvd = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gsvd, stream=st):
        svd_step()
    with torch.cuda.stream(st):
        for _ in range(3):
            gsvd.replay()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(st)
        for _ in range(10):
            gsvd.replay()
        e1.record(st)
    st.synchronize()
    ms_svd = max_over_ranks(torch, e0.elapsed_time(e1) / 10, dev, world)
    del gsvd, fixed
    torch.cuda.empty_cache()
    # the same union-masked step through cuBLAS: per linear Z = X B^T over all
    # r_store experts (torch.matmul), the per-token selection mask as a torch
    # multiply (bf16), Y = Z A^T -- identical GEMM shapes and bytes to k_union_prog
    # (operands copied with r_store padded to a multiple of 8 by zero experts, so
    # every row is 16-byte aligned for cuBLAS, as the kernel pads Z)
    umask = []
    for lay in stack:
        um = {}
        for nm in LIN:
            L, sb = lay[nm][0], lay[nm][1]
            r8 = (L.r_store + 7) // 8 * 8
            bt, a = L._keep
            bp = torch.zeros(r8, bt.shape[1], device=dev, dtype=bt.dtype)
            bp[:L.r_store] = bt
            ap = torch.zeros(a.shape[0], r8, device=dev, dtype=a.dtype)
            ap[:, :L.r_store] = a
            mk = torch.zeros(len(prompts), r8, device=dev, dtype=torch.bfloat16)
            mk[:, :L.r_store] = sb.masks.view(sb.P, sb.stride)[:, :L.r_store].to(torch.bfloat16)[tp.long()]
            um[nm] = (bp, ap, mk)
        umask.append(um)

    def cublas_union_step():
        for um, b in zip(umask, bufs):
            h = {"x": b["x"]}
            for nm in LIN:
                bp, ap, mk = um[nm]
                h[nm] = torch.matmul(torch.matmul(h[SRC[nm]], bp.t()) * mk, ap.t())
            svd["u"] = h["down"]

    with torch.cuda.stream(st):
        cublas_union_step()
    st.synchronize()
    gcu = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gcu, stream=st):
        cublas_union_step()
    with torch.cuda.stream(st):
        for _ in range(3):
            gcu.replay()
        e0.record(st)
        for _ in range(10):
            gcu.replay()
        e1.record(st)
    st.synchronize()
    ms_cu = max_over_ranks(torch, e0.elapsed_time(e1) / 10, dev, world)
    del gcu, umask
    svd_bytes = args.layers * sum(ldims[i][1] * (m + n) * 2 for i, (m, n) in enumerate(LIN.values()))
    del svd
    dom = {"what": "k_union_prog: the whole step (all 32 x 8 union GEMM stages) is one launch",
           "modules_ms_per_step": ms_modules, "modules_launches_per_step": graphs["modules"][1],
           "program_vs_modules_rel": agree}

    bytes_step = args.layers * sum(ldims[i][0] * (m + n) * 2 for i, (m, n) in enumerate(LIN.values()))
    flops_step = args.layers * 2 * Pl * sum(ldims[i][0] * (m + n) for i, (m, n) in enumerate(LIN.values()))
    step_s = ms_total / args.steps * 1e-3
    glob_tok = N_PROMPTS if args.scaling == "strong" else Pl * world
    traffic = None
    tp_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp_path):
        traffic = json.load(open(tp_path)).get("config4_step")
    out = {
        "metric": METRIC, "value": glob_tok / step_s, "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
        "warmup": args.warmup, "ms_per_step": ms_total / args.steps, "higher_is_better": True,
        "scaling": args.scaling, "vs_baseline": None, "dtype": "bf16",
        "data": "synthetic (random-init rank-expert factors and inputs, seeded; selections from the reference's "
                "pattern generator)",
        "config": config4_config(args.layers, Pl, world, args.scaling),
        "method": {"kernel": "union-masked tcgen05 GEMMs, q/k/v and up/gate grouped per stage, the whole step one "
                             "persistent launch (k_union_prog)",
                   "l2": f"{args.layers} distinct layer weight sets, {bytes_step / 1e9:.2f} GB streamed per step "
                         f"(>> 126 MB L2, no flush needed)",
                   "median_ms_per_step": ms_med, "graph": "one CUDA graph per step, replayed"},
        "e2e": {"value": glob_tok / (ms_e2e / args.steps * 1e-3), "unit": "tokens/s",
                "h2d_bytes_per_step": Pl * D_MODEL * 2, "d2h_bytes_per_step": Pl * D_MODEL * 2,
                "io": "input hidden states H2D from pinned memory and the last layer's output D2H, inside the "
                      "timed step (pg_copy_io kernels)", "median_ms_per_step": ms_e2e_med},
        "roofline": {"bound": "hbm", "achieved": bytes_step / step_s / 1e9, "peak": hbm_peak, "unit": "GB/s",
                     "frac": bytes_step / step_s / 1e9 / hbm_peak, "traffic": traffic,
                     "kernel": "k_union_prog (the step's 256 union GEMM stages in one persistent launch): stored "
                               "expert bytes r_store(m+n)*2 of every linear, read once per step for the whole batch",
                     "alg_bytes_per_step": bytes_step, "tensor_tflops": flops_step / step_s / 1e12,
                     "peak_kind": peak_kind, "dominant_launch": dom},
        "baselines": {"union_gemms_cublas": {
            "tokens_per_s": glob_tok / (ms_cu * 1e-3), "ms_per_step": ms_cu,
            "what": "the identical union-masked step through cuBLAS: per linear torch.matmul over all r_store experts, "
                    "the per-token selection mask as a bf16 multiply, torch.matmul back (2 GEMMs + 1 elementwise per "
                    "linear, 7 linears x 32 layers, CUDA graph; operands zero-padded to r_store rounded to 8)"},
            "native_fixed_rank_svd_cublas": {
            "tokens_per_s": glob_tok / (ms_svd * 1e-3), "ms_per_step": ms_svd,
            "what": "the same 32-layer step with each linear's static prefix A[:, :K] (B[:, :K]^T x) through cuBLAS "
                    "(torch.matmul, bf16, CUDA graph, contiguous factors with K padded to a multiple of 8): one "
                    "fixed K-expert subset for every prompt, K(m+n)*2 bytes "
                    f"per linear ({svd_bytes / 1e9:.2f} GB per step) -- the rank-expert step serves a different subset "
                    "per prompt and reads the union of the subsets (r_store = 2K experts)"}},
        "gpu_launches": launches * args.steps,
        "launches_per_step": launches,
        "clocks": clk.summary(),
    }
    del stack, bufs, prog, graphs
    torch.cuda.empty_cache()
    return out


# ======================================================================= config 2 (decode batch 1)

def config2_arm(args, rank, world, local_rank, windows=20, G=64, replicas=4):
    """BASELINE config 2: LLaMA-7B MLP block decode batch 1, S from a pattern-
    cache hit reused across steps; the whole block is one k_chain launch."""
    import torch
    import paper_2605_08568_b200 as pg
    dev = torch.device("cuda", local_rank)
    hbm_peak, _, peak_kind = peaks()
    sh = {k: (LIN[k][0], LIN[k][1]) + dims(*LIN[k])[::-1] for k in ("up", "gate", "down")}  # m, n, K, r
    pats = pg.make_patterns(17171 + rank, N_CACHE, [(sh[k][3], sh[k][2]) for k in ("up", "gate", "down")])
    gen = torch.Generator(device=dev).manual_seed(1234 + rank)
    emb = torch.randn((N_CACHE, D_MODEL), generator=gen, device=dev, dtype=torch.float64)
    emb /= emb.norm(dim=1, keepdim=True)
    cache = pg.PatternCache(D_MODEL, N_CACHE, MIN_SIM)
    cache.load([pg.CacheEntry(pg.PromptEmbedding(e), {"up": p[0], "gate": p[1], "down": p[2]})
                for e, p in zip(emb.cpu().numpy(), pats)])
    q = emb[7] + 0.3 / D_MODEL ** 0.5 * torch.randn(D_MODEL, generator=gen, device=dev, dtype=torch.float64)
    q /= q.norm()
    blocks = []
    for j in range(replicas):
        gg = torch.Generator(device=dev).manual_seed(100 * rank + j)
        b = {}
        for name, (m, n, K, r) in sh.items():
            bt = (torch.randn((r, n), generator=gg, device=dev) / n ** 0.5).to(torch.bfloat16)
            sig = 1.0 / (1.0 + torch.arange(r, device=dev, dtype=torch.float32) / 64.0)
            a = (torch.randn((m, r), generator=gg, device=dev) * sig / m ** 0.5).to(torch.bfloat16)
            b[name] = pg.FactorizedLayer.from_device(bt, a, K, layer_id=name)
            b[name]._raw = (bt, a, K)
        blocks.append(b)
    torch.cuda.synchronize()
    res = pg.retrieve(cache, q)
    assert res.hit and res.entry == 7, (res.entry, res.similarity)
    aggs = [{k: pg.aggregate_layout(b[k], [res.pattern[k]], PSI) for k in b} for b in blocks]
    # retrieve (scan + exact-band select, 2 kernels) as a 20-call CUDA graph:
    # device time per call; the 33.5 MB table is L2-resident between calls
    ent = torch.empty(1, dtype=torch.int32, device=dev)
    hit = torch.empty(1, dtype=torch.int32, device=dev)
    rst = torch.cuda.Stream(device=dev)

    def ret():
        from paper_2605_08568_b200 import _lib
        _lib.call("pg_retrieve", cache.handle, q.data_ptr(), 0, None, ent.data_ptr(), hit.data_ptr(), rst.cuda_stream)

    with torch.cuda.stream(rst):
        ret()
    rst.synchronize()
    rg = torch.cuda.CUDAGraph()
    with torch.cuda.graph(rg, stream=rst):
        for _ in range(20):
            ret()
    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(rst):
        rg.replay()
        ev0.record(rst)
        for _ in range(5):
            rg.replay()
        ev1.record(rst)
    rst.synchronize()
    retrieve_us = ev0.elapsed_time(ev1) / 100 * 1e3

    xs = torch.randn((G, D_MODEL), generator=gen, device=dev).to(torch.bfloat16)
    act = torch.empty((G, D_FF), device=dev, dtype=torch.bfloat16)
    y = torch.empty((G, D_MODEL), device=dev)
    x_host = torch.empty((G, D_MODEL), dtype=torch.bfloat16).pin_memory()
    x_host.copy_(xs.cpu())
    y_host = torch.empty((G, D_MODEL), dtype=torch.float32).pin_memory()

    def step(i, host_io):
        a = aggs[i % replicas]
        if host_io:
            pg.copy_io(xs[i], x_host[i])
        pg.mlp_forward(a["up"], a["gate"], a["down"], 0, xs[i], out=y[i], act=act[i])
        if host_io:
            pg.copy_io(y_host[i], y[i])

    stream = torch.cuda.Stream(device=dev)
    graphs = {}
    for host_io in (False, True):
        with torch.cuda.stream(stream):
            for i in range(G):
                step(i, host_io)
        stream.synchronize()
        gr = torch.cuda.CUDAGraph()
        n0 = pg.launch_count()
        with torch.cuda.graph(gr, stream=stream):
            for i in range(G):
                step(i, host_io)
        graphs[host_io] = (gr, pg.launch_count() - n0)

    def timed(host_io):  # median over `windows` replays of a G-step graph
        gr = graphs[host_io][0]
        with torch.cuda.stream(stream):
            for _ in range(3):
                gr.replay()
        barrier(torch, world)
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(windows + 1)]
        with torch.cuda.stream(stream):
            ev[0].record(stream)
            for i in range(windows):
                gr.replay()
                ev[i + 1].record(stream)
        barrier(torch, world)
        med = float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(windows)]))
        return max_over_ranks(torch, med, dev, world) / G  # ms per step

    def cublas_tok_s(mats):
        xb = torch.randn((G, D_MODEL), generator=gen, device=dev).to(torch.bfloat16)

        def one(i):
            w = mats[i % replicas]
            if len(w) == 6:
                bu, au, bg, ag, bd, ad = w
                return ad @ (bd @ (torch.nn.functional.silu(ag @ (bg @ xb[i])) * (au @ (bu @ xb[i]))))
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
    svd_tok_s = cublas_tok_s(svd)
    del svd
    dense = [tuple(torch.randn(shp, generator=gen, device=dev).to(torch.bfloat16) / 64
                   for shp in ((D_FF, D_MODEL), (D_FF, D_MODEL), (D_MODEL, D_FF))) for _ in range(replicas)]
    dense_tok_s = cublas_tok_s(dense)
    del dense
    ms = timed(False)
    ms_e2e = timed(True)
    traffic = None
    tp_path = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if os.path.exists(tp_path):
        traffic = json.load(open(tp_path)).get("k_chain<bf16>")
    step_bytes = sum(K_ * (m_ + n_) * 2 for (m_, n_, K_, _) in sh.values()) + D_MODEL * 2 + D_FF * 4 + D_MODEL * 4
    achieved = step_bytes / (ms * 1e-3) / 1e9
    out = {"workload": "config2: LLaMA-7B MLP block (gate/up 4096->11008, down 11008->4096) ratio 0.6 K=1194 "
                       "r_store=2388, decode batch 1, S from a pattern-cache hit (N=1024 x d=4096 f64) reused "
                       f"across steps, bf16; {replicas} weight replicas rotated (> L2)",
           "tokens_per_s": world / (ms * 1e-3), "ms_per_step": ms,
           "e2e_tokens_per_s": world / (ms_e2e * 1e-3), "launches_per_step": graphs[False][1] / G,
           "timing": f"median of {windows} windows of a {G}-step CUDA graph",
           "roofline": {"bound": "hbm", "achieved": achieved, "peak": hbm_peak, "unit": "GB/s",
                        "frac": achieved / hbm_peak, "traffic": traffic, "alg_bytes_per_launch": step_bytes,
                        "kernel": "k_chain<bf16> (fused MLP block, 1 launch per step)", "peak_kind": peak_kind},
           "retrieve_us": retrieve_us,
           "retrieve": {"us": retrieve_us, "what": "pg_retrieve (wide cosine scan + exact-band select, PDL), N=1024 x "
                        "d=4096 f64, 20-call CUDA graph; table L2-resident between calls",
                        "alg_bytes": 8 * N_CACHE * D_MODEL,
                        "achieved_gbs": 8 * N_CACHE * D_MODEL / (retrieve_us * 1e-6) / 1e9,
                        "frac_hbm": 8 * N_CACHE * D_MODEL / (retrieve_us * 1e-6) / 1e9 / hbm_peak},
           "baselines": {"native_fixed_rank_svd_cublas_tok_s": svd_tok_s, "dense_cublas_tok_s": dense_tok_s}}
    del blocks, aggs
    torch.cuda.empty_cache()
    return out


# ======================================================================= config 3 (prefill)

def config3_arm(args, rank, world, local_rank, P=16, T=2048):
    """BASELINE config 3: one LLaMA-7B decoder layer's 7 rank-expert linears,
    16 prompts x 2048 tokens, each routed on device to its own expert subset
    (bit-exact router), packed on device, grouped tcgen05 GEMMs.  Timed: routing
    + pack + the 7 prefill linears."""
    import torch
    import paper_2605_08568_b200 as pg
    dev = torch.device("cuda", local_rank)
    g = torch.Generator(device=dev).manual_seed(7)
    X = torch.randn(P * T, D_MODEL, device=dev, generator=g).to(torch.bfloat16)
    X2 = torch.randn(P * T, D_FF, device=dev, generator=g).to(torch.bfloat16)
    Xo = torch.randn(P * T, D_MODEL, device=dev, generator=g).to(torch.bfloat16)
    offs = [i * T for i in range(P + 1)]
    layers, routers, outs, flops = {}, {}, {}, 0
    for nm, (m, n) in LIN.items():
        r, K = dims(m, n)
        bt = (torch.randn((r, n), generator=g, device=dev) / n ** 0.5).to(torch.bfloat16)
        a = (torch.randn((m, r), generator=g, device=dev) / m ** 0.5).to(torch.bfloat16)
        layers[nm] = (pg.FactorizedLayer.from_device(bt, a, K), K)
        routers[nm] = pg.RouterParams(torch.randn((r, n), generator=g, device=dev, dtype=torch.float64))
        outs[nm] = torch.empty(P * T, m, device=dev, dtype=torch.bfloat16)
        flops += 2 * P * T * K * (m + n)
    src = {"q": X, "k": X, "v": X, "up": X, "gate": X, "o": Xo, "down": X2}
    sels = {}

    # the seven routers are independent given their pooled inputs: four side
    # streams forked from / joined to the current one (pool X -> q, k, v | up,
    # gate; pool Xo -> o; pool X2 -> down), so the narrow score / select
    # launches of one router fill the SMs another leaves idle
    side = [torch.cuda.Stream(device=dev) for _ in range(4)]
    lanes = [(X, ("q", "k", "v")), (None, ("up", "gate")), (Xo, ("o",)), (X2, ("down",))]

    def route_all():
        cur = torch.cuda.current_stream(dev)
        fork = torch.cuda.Event()
        fork.record(cur)
        pooled_x = torch.cuda.Event()
        hx = None
        for i, (inp, names) in enumerate(lanes):
            st_i = side[i]
            st_i.wait_event(fork)
            with torch.cuda.stream(st_i):
                if inp is None:  # up / gate reuse X's pooling
                    st_i.wait_event(pooled_x)
                    h = hx
                else:
                    h = pg.mean_pool(inp, layout="token", offsets=offs)
                    if inp is X:
                        hx = h
                        pooled_x.record(st_i)
                for nm in names:
                    sels[nm] = pg.route_select_pooled(routers[nm], h, layers[nm][1])
        for st_i in side:
            cur.wait_stream(st_i)

    have_dev_pack = hasattr(pg, "pack_selected")

    bufs = {False: {}, True: {}}
    have_gather = have_dev_pack and hasattr(pg, "PackedExperts") and hasattr(pg.PackedExperts, "gathered")

    def pack_all(gather=False):  # device pack into persistent buffers (no allocation inside the timed region)
        # gather=True: A columns only; the stage-1 GEMM gathers the B^T rows (TMA gather4)
        if not have_dev_pack:
            return None
        b = bufs[gather]
        for nm in LIN:
            b[nm] = (pg.pack_selected(layers[nm][0], sels[nm], into=b.get(nm), gather=True) if gather
                     else pg.pack_selected(layers[nm][0], sels[nm], into=b.get(nm)))
        return dict(b)

    def gemms(packs):
        for nm in LIN:
            if have_dev_pack:
                pg.prefill_packed(packs[nm], offs, src[nm], out_dtype=torch.bfloat16, out=outs[nm])
            else:
                pg.prefill_batched(packs[nm], offs, src[nm], out_dtype=torch.bfloat16, out=outs[nm])

    for _ in range(2):
        route_all()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if have_dev_pack:
        packs = pack_all()
    else:  # host-driven pack per prompt (round-1 path)
        packs = {nm: [pg.aggregate_layout(layers[nm][0], [pg.RankSelection(sels[nm][p].cpu().numpy())], PSI)
                      for p in range(P)] for nm in LIN}
    torch.cuda.synchronize()
    pack_ms_host = (time.perf_counter() - t0) * 1e3
    gemms(packs)
    torch.cuda.synchronize()
    if have_gather:
        gemms(pack_all(True))
        torch.cuda.synchronize()
    reps = 5
    e = [torch.cuda.Event(enable_timing=True) for _ in range(6)]
    barrier(torch, world)
    e[0].record()
    for _ in range(reps):
        route_all()
    e[1].record()
    for _ in range(reps if have_dev_pack else 0):
        packs = pack_all()
    e[2].record()
    for _ in range(reps):
        gemms(packs)
    e[3].record()
    for _ in range(reps if have_gather else 0):
        gpacks = pack_all(True)
    e[4].record()
    for _ in range(reps if have_gather else 0):
        gemms(gpacks)
    e[5].record()
    barrier(torch, world)
    # the same packed GEMMs through cuBLAS (torch.bmm over the 16 prompts: the
    # batched-GEMM analogue of the grouped launch), z rounded to bf16 between
    cub_ms = None
    if have_dev_pack:
        def cublas_gemms():
            for nm, (m, n) in LIN.items():
                pk = packs[nm]
                kp = (pk.k + 7) // 8 * 8
                ldb = pk.bt.numel() // 2 // (P * kp)
                bt = pk.bt.view(torch.bfloat16).view(P, kp, ldb)[:, :, :n]
                a = pk.a.view(torch.bfloat16).view(P, m, kp)
                x = src[nm].view(P, T, n)
                z = torch.bmm(x, bt.transpose(1, 2))
                outs[nm].view(P, T, m).copy_(torch.bmm(z, a.transpose(1, 2)))

        gst = torch.cuda.Stream(device=dev)
        with torch.cuda.stream(gst):
            cublas_gemms()
        gst.synchronize()
        gcb = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gcb, stream=gst):
            cublas_gemms()
        ec = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
        with torch.cuda.stream(gst):
            gcb.replay()
            ec[0].record(gst)
            for _ in range(reps):
                gcb.replay()
            ec[1].record(gst)
        gst.synchronize()
        cub_ms = max_over_ranks(torch, ec[0].elapsed_time(ec[1]) / reps, dev, world)
        del gcb
    route_ms = max_over_ranks(torch, e[0].elapsed_time(e[1]) / reps, dev, world)
    pack_ms = max_over_ranks(torch, e[1].elapsed_time(e[2]) / reps, dev, world) if have_dev_pack else pack_ms_host
    ms = max_over_ranks(torch, e[2].elapsed_time(e[3]) / reps, dev, world)
    modes = {"packed": {"pack_ms": pack_ms, "gemm_ms": ms,
                        "what": "pack B^T rows + A columns per prompt, GEMMs over the packed arenas"}}
    if have_gather:
        gpack_ms = max_over_ranks(torch, e[3].elapsed_time(e[4]) / reps, dev, world)
        gms = max_over_ranks(torch, e[4].elapsed_time(e[5]) / reps, dev, world)
        modes["gathered"] = {"pack_ms": gpack_ms, "gemm_ms": gms,
                             "what": "pack A columns only; the stage-1 GEMM gathers the selected B^T rows with "
                                     "TMA gather4 (bit-identical results)"}
        if gpack_ms + gms < pack_ms + ms:  # report the faster pipeline
            pack_ms, ms = gpack_ms, gms
    mode = min(modes, key=lambda k: modes[k]["pack_ms"] + modes[k]["gemm_ms"])
    _, tflops_peak, peak_kind = peaks()
    achieved = flops / (ms * 1e-3) / 1e12
    out = {"workload": "config3: LLaMA-7B decoder layer (q,k,v,o,gate,up,down) ratio 0.6, 16 prompts x 2048 tokens, "
                       "per-prompt expert subsets routed on device, bf16 (z rounded to bf16 between stages)",
           "tokens_per_s": P * T / ((ms + route_ms + pack_ms) * 1e-3) * world,
           "gemm_tokens_per_s": P * T / (ms * 1e-3) * world,
           "ms_per_layer": ms, "route_ms": route_ms, "pack_ms": pack_ms,
           "pack_on_device": have_dev_pack, "mode": mode, "modes": modes,
           "baselines": {"packed_gemms_cublas": None if cub_ms is None else {
               "ms_per_layer": cub_ms, "tflops": flops / (cub_ms * 1e-3) / 1e12,
               "what": "the same packed per-prompt GEMMs through cuBLAS (torch.bmm over the 16 prompts, "
                       "z rounded to bf16 between the stages, CUDA graph)"}},
           "roofline": {"bound": "tensor", "achieved": achieved, "peak": tflops_peak, "unit": "TFLOP/s",
                        "frac": achieved / tflops_peak, "flops_per_layer": flops, "peak_kind": peak_kind,
                        "kernel": "k_umma_grouped2 (tcgen05.mma cta_group::2 kind::f16, TMA, TMEM; 2 grouped "
                                  "launches per linear)"}}
    del layers, routers, outs, X, X2, Xo
    torch.cuda.empty_cache()
    return out


# ======================================================================= config 1 (fp32, CPU ref in full)

def config1_arm(args, local_rank, cpu: bool):
    """BASELINE config 1: one q_proj-shaped layer (4096x4096, ratio 0.6: K=819,
    r_store=1638), fp32, one prompt: route from the 128-token prefill (bit-exact
    router), 128-token prefill + 32 decode steps reusing S (RoutingProvider,
    model.hpp:96-106).  The reference CPU path runs the same work in full
    (mean_pool/score/select_topk f64, aggregate_layout + aggregated_forward<float>)
    and the two outputs are compared."""
    import torch
    import paper_2605_08568_b200 as pg
    from oracle import pyoracle
    dev = torch.device("cuda", local_rank)
    m = n = D_MODEL
    r, K = dims(m, n)
    T, D = 128, 32
    o = pyoracle.Oracle("port")
    A = o.gaussian(101, (m, r)) / np.sqrt(K)
    B = o.gaussian(102, (n, r)) / np.sqrt(n)
    theta = o.gaussian(103, (r, n))
    X = o.gaussian(104, (n, T)).astype(np.float32)
    Xd = o.gaussian(105, (n, D)).astype(np.float32)
    L = pg.FactorizedLayer(A, B, K, dtype="f32")
    router = pg.RouterParams(theta, np.zeros(r))
    xg = torch.from_numpy(X).to(dev)
    xdg = [torch.from_numpy(np.ascontiguousarray(Xd[:, j:j + 1])).to(dev) for j in range(D)]
    ys = [torch.empty(m, 1, device=dev) for _ in range(D)]

    def run():
        sel = pg.route_select(router, xg, K)[0]
        agg_sel = sel  # device selection, reused by every call (route once, reuse)
        yp = pg.masked_forward(L, agg_sel, xg)
        for j in range(D):
            pg.masked_forward(L, agg_sel, xdg[j], out=ys[j])
        return sel, yp

    for _ in range(2):
        run()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 5
    e0.record()
    for _ in range(reps):
        sel, yp = run()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    out = {"workload": "config1: q_proj 4096x4096 ratio 0.6 (K=819, r_store=1638), fp32, 1 prompt: route + "
                       "128-token prefill + 32 decode steps reusing S", "ms_gpu": ms,
           "tokens_per_s_gpu": (T + D) / (ms * 1e-3)}
    if cpu:
        kind = "reference" if pyoracle.available("reference") else "port"
        oc = pyoracle.Oracle(kind)
        t0 = time.perf_counter()
        want = oc.select_topk(oc.score(theta, np.zeros(r), oc.mean_pool(X.astype(np.float64))), K)
        agg = oc.aggregate_layout(A, B, [want], PSI, elem=4)
        t1 = time.perf_counter()
        yc = agg.forward(0, X)
        ycd = [agg.forward(0, np.ascontiguousarray(Xd[:, j:j + 1])) for j in range(D)]
        t2 = time.perf_counter()
        got = sel.cpu().numpy().astype(np.uint32)
        ygp = yp.cpu().numpy()
        rel_p = float(np.abs(ygp - yc).max() / np.abs(yc).max())
        rel_d = max(float(np.abs(ys[j].cpu().numpy() - ycd[j]).max() / np.abs(ycd[j]).max()) for j in range(D))
        out.update({"cpu_kind": kind, "cpu_cores": 1, "ms_cpu_route_pack": (t1 - t0) * 1e3,
                    "ms_cpu_forward": (t2 - t1) * 1e3,
                    "tokens_per_s_cpu": (T + D) / (t2 - t0), "selection_bit_exact": bool(np.array_equal(got, want)),
                    "rel_err_prefill_vs_cpu": rel_p, "rel_err_decode_vs_cpu": rel_d})
    return out


# ======================================================================= config 5 (13B, expert-sharded)

LIN13 = {"q": (5120, 5120), "k": (5120, 5120), "v": (5120, 5120), "o": (5120, 5120),
         "up": (13824, 5120), "gate": (13824, 5120), "down": (5120, 13824)}


def config5_arm(args, rank, world, local_rank, T_pre=256, n_dec=8, reps=10):
    """BASELINE config 5: one LLaMA-13B-shaped decoder layer's 7 rank-expert
    linears at ratio 0.4 (K = 1536 / 2241, r_store = 3072 / 4482: stored experts
    exceed dense storage), expert-sharded (expert e on rank e mod G,
    dist.py), mixed work per step: a T=256 prefill chunk then 8 decode tokens,
    every linear's partial all-reduced over NCCL (the only collective).  Each
    rank holds 1/G of the experts (weights generated on device for the rank's
    own columns); selections from the reference generator."""
    import torch
    import paper_2605_08568_b200 as pg
    from paper_2605_08568_b200 import dist as pgd
    dev = torch.device("cuda", local_rank)
    g = torch.Generator(device=dev).manual_seed(13 + rank)
    ldims = {}
    for nm, (m, n) in LIN13.items():
        K = pg.single_layer_k(m, n, 0.4)
        ldims[nm] = (pg.store_rank(K, n), K)
    pats = pg.make_patterns(5151, 1, [ldims[nm] for nm in LIN13])[0]
    lins = {}
    for j, (nm, (m, n)) in enumerate(LIN13.items()):
        r, K = ldims[nm]
        cols = len(range(rank, r, world))
        bt = (torch.randn(cols, n, device=dev, generator=g) / n ** 0.5).to(torch.bfloat16)
        a = (torch.randn(m, cols, device=dev, generator=g) / K ** 0.5).to(torch.bfloat16)
        mine = pgd.shard_selection(pats[j], world, rank)
        loc = (mine // world).astype(np.uint32) if mine.size else np.zeros(1, np.uint32)
        if not mine.size:  # this rank owns none of the selected experts: it contributes an exact zero partial
            bt, a = bt[:1].zero_(), a[:, :1].contiguous().zero_()
        L = pg.FactorizedLayer.from_device(bt, a, int(loc.size), layer_id=f"b0.{nm}")
        agg = pg.aggregate_layout(L, [pg.RankSelection(loc)], 0.9)
        lins[nm] = (agg, m, n, mine.size)
    xp = torch.randn(T_pre, 5120, device=dev, generator=g).to(torch.bfloat16)
    xd = torch.randn(5120, device=dev, generator=g).to(torch.bfloat16)
    xpf = torch.randn(T_pre, 13824, device=dev, generator=g).to(torch.bfloat16)
    xdf = torch.randn(13824, device=dev, generator=g).to(torch.bfloat16)
    yd = {nm: torch.empty(m, device=dev) for nm, (_, m, _, _) in lins.items()}
    st = torch.cuda.Stream(device=dev)

    def reduce(y):
        if world > 1:
            torch.distributed.all_reduce(y)

    act = torch.empty(13824, device=dev, dtype=torch.bfloat16)
    # --c5-peer 1 (world > 1): the decode token's all-reduces fused into the
    # kernels over NVLink peer memory -- q, k, v, o through pg_agg_forward_peer,
    # the MLP block through pg_mlp_forward_peer (one launch) -- no NCCL call
    use_peer = bool(getattr(args, "c5_peer", 0)) and world > 1
    if use_peer:
        import ctypes as C
        from paper_2605_08568_b200.api import _dtype_code, _ptr, call
        grp = torch.distributed.group.WORLD
        pbuf = {nm: pgd.PeerBuffer(LIN13[nm][0], world, rank, group=grp) for nm in ("q", "k", "v", "o")}
        pbuf["mlp"] = pgd.PeerBuffer(2 * 13824 + 5120, world, rank, group=grp)
        f32 = _dtype_code(torch.float32)
        zeros3 = (C.c_size_t * 3)(0, 0, 0)

    def decode_token_peer():
        s = torch.cuda.current_stream(dev).cuda_stream
        for nm in ("q", "k", "v", "o"):
            call("pg_agg_forward_peer", lins[nm][0].handle, 0, _ptr(xd), _ptr(yd[nm]), f32, rank, world,
                 pbuf[nm].ptrs, 0, s)
        call("pg_mlp_forward_peer", lins["up"][0].handle, lins["gate"][0].handle, lins["down"][0].handle, zeros3,
             _ptr(xd), _ptr(act), _ptr(yd["down"]), f32, rank, world, pbuf["mlp"].ptrs, 0, s)

    def decode_token():
        if use_peer:
            decode_token_peer()
            return
        if world == 1:
            # one shard holds every expert: q/k/v as one fused module launch, o, and
            # the MLP block as one k_chain launch (up/gate -> silu -> down)
            pg.module_forward([lins[nm][0] for nm in ("q", "k", "v")], 0, xd, out_dtype=torch.float32,
                              outs=[yd[nm] for nm in ("q", "k", "v")])
            pg.aggregated_forward(lins["o"][0], 0, xd, out_dtype=torch.float32, out=yd["o"])
            pg.mlp_forward(lins["up"][0], lins["gate"][0], lins["down"][0], 0, xd, out_dtype=torch.float32,
                           out=yd["down"], act=act)
            return
        for nm, (agg, m, n, own) in lins.items():  # sharded: every linear's partial all-reduced
            pg.aggregated_forward(agg, 0, xdf if n == 13824 else xd, out_dtype=torch.float32, out=yd[nm])
            reduce(yd[nm])

    # prefill chunk: linears that read the same hidden state run as one grouped
    # tcgen05 launch per stage (q/k/v, then up/gate: the same x served by three /
    # two layouts, x replicated per layout inside the step); o and down alone
    groups = [("q", "k", "v"), ("o",), ("up", "gate"), ("down",)]
    gx = {gr: torch.empty(len(gr) * T_pre, LIN13[gr[0]][1], device=dev, dtype=torch.bfloat16) for gr in groups}
    gy = {gr: torch.empty(len(gr) * T_pre, LIN13[gr[0]][0], device=dev) for gr in groups}

    def step():
        for gr in groups:
            n = LIN13[gr[0]][1]
            x = xpf if n == 13824 else xp
            if len(gr) == 1:
                pg.aggregated_forward_batched(lins[gr[0]][0], [0], [0, T_pre], x, out_dtype=torch.float32,
                                              out=gy[gr])
            else:
                gx[gr].view(len(gr), T_pre, n).copy_(x.expand(len(gr), T_pre, n))
                pg.prefill_batched([lins[nm][0] for nm in gr], [T_pre * i for i in range(len(gr) + 1)], gx[gr],
                                   out_dtype=torch.float32, out=gy[gr])
            reduce(gy[gr])
        for _ in range(n_dec):  # decode tokens reusing S
            decode_token()

    def decode():  # decode alone (the HBM-bound part): 8 tokens through the 7 sharded linears
        for _ in range(n_dec):
            decode_token()

    with torch.cuda.stream(st):
        for _ in range(3):
            step()
    st.synchronize()
    # one CUDA graph per step (and per 8-token decode run): the per-linear launches
    # are shorter than their Python dispatch; NCCL all-reduces are captured too
    graphs = {}
    try:
        # world > 1: eager (NCCL all-reduces are not captured; no multi-GPU box to validate that here)
        for key, fn in ((("step", step), ("decode", decode)) if world == 1 else ()):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=st):
                fn()
            graphs[key] = gr
    except Exception:  # noqa: BLE001 -- eager fallback, reported below
        graphs = {}
    run_step = graphs["step"].replay if graphs else step
    run_dec = graphs["decode"].replay if graphs else decode
    barrier(torch, world)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(st):
        run_step()
        e0.record(st)
        for _ in range(reps):
            run_step()
        e1.record(st)
    st.synchronize()
    ms = max_over_ranks(torch, e0.elapsed_time(e1) / reps, dev, world)
    with torch.cuda.stream(st):
        run_dec()
        e0.record(st)
        for _ in range(reps):
            run_dec()
        e1.record(st)
    st.synchronize()
    us_dec = max_over_ranks(torch, e0.elapsed_time(e1) / reps / n_dec * 1e3, dev, world)
    hbm_peak, tensor_peak, peak_kind = peaks()
    dec_bytes = sum(own * (m + n) * 2 for (_, m, n, own) in lins.values())  # this rank's selected experts
    flops = 2 * T_pre * sum(ldims[nm][1] * (m + n) for nm, (m, n) in LIN13.items())
    return {"workload": f"config5: LLaMA-13B decoder layer (q,k,v,o 5120x5120, gate/up 5120->13824, down "
                        f"13824->5120) ratio 0.4, expert-sharded over {world} GPU(s) (e mod G), per step 1 x "
                        f"T={T_pre} prefill chunk (q/k/v and up/gate grouped per stage) + {n_dec} decode tokens through all 7 "
                        f"linears, partial outputs "
                        f"all-reduced (NCCL) per linear; bf16 weights, f32 outputs",
            "ms_per_step": ms, "tokens_per_s": (T_pre + n_dec) / (ms * 1e-3),
            "decode_us_per_token": us_dec, "decode_tokens_per_s": 1e6 / us_dec,
            "decode_roofline": {"bound": "hbm", "alg_bytes_per_token_rank0": dec_bytes,
                                "achieved": dec_bytes / (us_dec * 1e-6) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                                "frac": dec_bytes / (us_dec * 1e-6) / 1e9 / hbm_peak, "peak_kind": peak_kind},
            "prefill_flops_per_step": flops, "graph": bool(graphs),
            "decode_path": "world 1: q/k/v fused module + o + fused MLP block (k_chain), 3 launches per token"
            if world == 1 else ("fused peer reduction: q, k, v, o (pg_agg_forward_peer) + the MLP block in one launch "
                                "(pg_mlp_forward_peer), 5 launches per token, no NCCL" if use_peer else
                                "per linear: aggregated_forward + NCCL all-reduce of the partial"),
            "collective": ("decode: partials pushed as tagged words over NVLink peer memory (CUDA IPC), summed in "
                           "rank order in-kernel; prefill: NCCL all-reduce" if use_peer else
                           "torch.distributed.all_reduce (NCCL) of every linear's partial") if world > 1
            else "none (world 1: one shard holds every expert)"}


# ======================================================================= main

def dry_run(args, rank, world):
    """The multi-process plumbing of a --gpus N run without a GPU (CPU tests):
    one process per rank, a gloo group, this rank's share of the config-4
    prompts (weak: 256 per rank; strong: 256 split by pattern affinity), a
    barrier and the max-over-ranks reduction the timed region uses."""
    import torch
    import torch.distributed as dist
    from paper_2605_08568_b200 import dist as pgd
    if world > 1:
        dist.init_process_group("gloo")
    prompts = (pgd.partition_by_pattern(list(range(N_PROMPTS)), world)[rank] if args.scaling == "strong"
               else list(range(N_PROMPTS)))
    t = 1.0 + rank  # stand-in per-rank time: the line must carry the slowest rank's
    tmax = max_over_ranks(torch, t, torch.device("cpu"), world)
    counts = [len(prompts)]
    if world > 1:
        buf = [None] * world
        dist.all_gather_object(buf, prompts)
        counts = [len(b) for b in buf]
        covered = sorted(p for b in buf for p in b)
    else:
        covered = prompts
    if rank == 0:
        print(json.dumps({"dry_run": True, "n_gpus": world, "scaling": args.scaling, "max_over_ranks": tmax,
                          "prompts_per_rank": counts, "prompts_covered": len(set(covered)),
                          "global_tokens": len(covered) if args.scaling == "strong" else N_PROMPTS * world}),
              flush=True)
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--scaling", default="weak", choices=["weak", "strong"])
    ap.add_argument("--layers", type=int, default=N_LAYERS, help=argparse.SUPPRESS)
    ap.add_argument("--secondary", type=int, default=1, help="also run configs 1-3 (secondary objects)")
    ap.add_argument("--cpu", type=int, default=1, help="time the reference CPU path (rank 0, N=1)")
    ap.add_argument("--c5-peer", type=int, default=0,
                    help="config 5 at N > 1: decode all-reduces fused into the kernels over NVLink peer memory")
    ap.add_argument("--dry-run", action="store_true",
                    help="launch plumbing only (no GPU): ranks, gloo process group, prompt partition, max-over-ranks")
    args = ap.parse_args()
    args.warmup = max(3, args.warmup)
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        # one process per GPU: re-execute under torch.distributed.run
        cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
               "--master-addr", "127.0.0.1", "--master-port", os.environ.get("MASTER_PORT", "29517"),
               os.path.abspath(__file__)] + sys.argv[1:]
        sys.exit(subprocess.call(cmd))
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))

    if args.dry_run:
        dry_run(args, rank, world)
        return
    if args.impl == "reference":
        if rank != 0:
            return
        ref = reference_config4(repeats=max(1, min(args.steps, 3)))
        line = {"metric": METRIC, "value": ref["value"], "unit": "tokens/s", "n_gpus": world, "steps": args.steps,
                "warmup": args.warmup, "ms_per_step": N_PROMPTS / ref["value"] * 1e3,
                "higher_is_better": True, "scaling": args.scaling, "vs_baseline": None, "dtype": "f32",
                "data": "synthetic", "impl": "reference",
                "config": config4_config(N_LAYERS, N_PROMPTS // world if args.scaling == "strong" else N_PROMPTS,
                                         world, args.scaling),
                "method": {"kernel": "reference CPU ExecEngine<float>: aggregate_layout + aggregated_forward<float> "
                                     "(exec_engine.hpp:112-236), compiled from /root/reference (oracle/_ref)"},
                "cpu_baseline": {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model",
                                                     "nproc", "extrapolated", "ms_per_layer_per_prompt")},
                "e2e": {"value": ref["value"], "unit": "tokens/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
        print(json.dumps(line), flush=True)
        return

    import torch
    torch.cuda.set_device(local_rank)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
    out = config4_arm(args, rank, world, local_rank)
    if args.secondary:
        out["decode_b1"] = config2_arm(args, rank, world, local_rank)
        out["prefill"] = config3_arm(args, rank, world, local_rank)
        out["config5"] = config5_arm(args, rank, world, local_rank)
        if rank == 0:
            out["config1"] = config1_arm(args, local_rank, cpu=bool(args.cpu) and world == 1)
    if rank == 0 and world == 1 and args.cpu:
        ref = reference_config4()
        out["cpu_baseline"] = {k: ref[k] for k in ("value", "unit", "cores", "kind", "sample", "cpu_model", "nproc",
                                                   "extrapolated", "ms_per_layer_per_prompt")}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
