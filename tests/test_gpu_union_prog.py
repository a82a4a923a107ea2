"""K5e: a whole heterogeneous decode step as ONE persistent launch
(union_prog.cu, pg_union_prog_*), BASELINE config 4.

Every module of every layer (q/k/v, o, up/gate, down: stage 1 masked by each
token's selection, stage 2) runs in one kernel, the stages chained by device
ready counters.  Bars:
  * each module's outputs vs a plain PyTorch fp32 reference of the same two
    GEMMs on the program's own inputs (Z rounded to bf16, the selection mask
    applied per token): max|d|/max|ref| <= 4e-3 for bf16 outputs (half a bf16
    ulp of the output, <= 1.95e-3, plus accumulation order, which may flip a
    bf16 rounding of Z), 2e-3 for f32 outputs;
  * the end of the chain vs the per-module union path (module_forward_union,
    itself checked against the f64 oracle in test_gpu_prefill.py) run layer by
    layer: <= 2e-2 (bf16 roundings of Z and of every output compound through
    the chain; the two paths split K differently);
  * deterministic across launches, graph replays and repeated runs.
"""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

LIN = ("q", "k", "v", "o", "up", "gate", "down")
GROUPS = (("q", "k", "v"), ("o",), ("up", "gate"), ("down",))
TOL_BF16_OUT = 4e-3
SRC = {"q": "x", "k": "x", "v": "x", "o": "v", "up": "o", "gate": "o", "down": "up"}


@pytest.fixture(scope="module")
def pg():
    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    import paper_2605_08568_b200 as m
    return m


def rel(a, b):
    a = a.double()
    b = b.double()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-300))


def build(pg, D, F, rho_dims, layers, P, seed):
    """layers of rank-expert linears (B^T expert-major, A [m, r]) with P
    selections each from the reference's pattern generator."""
    shapes = {"q": (D, D), "k": (D, D), "v": (D, D), "o": (D, D), "up": (F, D), "gate": (F, D), "down": (D, F)}
    g = torch.Generator(device="cuda").manual_seed(seed)
    stack = []
    for li in range(layers):
        dims = [rho_dims[nm] for nm in LIN]
        pats = pg.make_patterns(seed + 17 * li, P, dims)
        lay = {}
        for j, nm in enumerate(LIN):
            m, n = shapes[nm]
            r, K = dims[j]
            bt = (torch.randn(r, n, device="cuda", generator=g) / n ** 0.5).to(torch.bfloat16)
            a = (torch.randn(m, r, device="cuda", generator=g) / K ** 0.5).to(torch.bfloat16)
            L = pg.FactorizedLayer.from_device(bt, a, K, layer_id=f"b{li}.{nm}")
            masks = torch.zeros(P, r, device="cuda")
            for p in range(P):
                masks[p, torch.from_numpy(np.asarray(pats[p][j].indices, np.int64)).cuda()] = 1.0
            lay[nm] = (L, pg.SelectionBatch(L, [pats[p][j] for p in range(P)]), bt, a, masks)
        stack.append(lay)
    return stack, shapes


def program(pg, stack, shapes, x, T, out_dtype=torch.bfloat16):
    prog = pg.UnionProgram(T)
    bufs = []
    src = x
    for lay in stack:
        b = {"x": src}
        for grp in GROUPS:
            for nm in grp:
                b[nm] = torch.empty(T, shapes[nm][0], device="cuda", dtype=out_dtype)
            prog.add_module([lay[nm][0] for nm in grp], [lay[nm][1] for nm in grp], b[SRC[grp[0]]],
                            [b[nm] for nm in grp])
        bufs.append(b)
        src = b["down"]
    return prog, bufs


def module_ref(lay, nm, xin, pid):
    _, _, bt, a, masks = lay[nm]
    z = ((xin.float() @ bt.float().t()) * masks[pid]).to(torch.bfloat16).float()
    return z @ a.float().t()


@pytest.mark.parametrize("D,F,T,layers,P", [(512, 1024, 96, 3, 12), (512, 1024, 256, 2, 40),
                                            (1024, 2816, 5, 2, 3), (512, 1024, 1, 1, 1), (512, 1024, 33, 2, 7)])
def test_union_program_small(pg, D, F, T, layers, P):
    dims = {nm: (300, 150) for nm in ("q", "k", "v", "o")}
    dims.update({"up": (700, 350), "gate": (700, 350), "down": (640, 320)})
    stack, shapes = build(pg, D, F, dims, layers, P, seed=100 + T)
    pid = torch.from_numpy(np.random.default_rng(T).integers(0, P, T).astype(np.int32)).cuda()
    x = torch.randn(T, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(T)).to(torch.bfloat16)
    prog, bufs = program(pg, stack, shapes, x, T)
    assert prog.info()[0] == 8 * layers
    n0 = pg.launch_count()
    prog.run(pid)
    assert pg.launch_count() == n0 + 1
    torch.cuda.synchronize()
    for lay, b in zip(stack, bufs):
        for nm in LIN:
            want = module_ref(lay, nm, b[SRC[nm]], pid.long())
            assert rel(b[nm].float(), want) <= TOL_BF16_OUT, nm
    # chain end vs the per-module union path run layer by layer
    h = x
    for lay in stack:
        c = {"x": h}
        for grp in GROUPS:
            ys = pg.module_forward_union([lay[nm][0] for nm in grp], [lay[nm][1] for nm in grp], pid, c[SRC[grp[0]]],
                                         out_dtype=torch.bfloat16)
            c.update(zip(grp, ys))
        h = c["down"]
    assert rel(bufs[-1]["down"].float(), h.float()) <= 2e-2
    # deterministic across launches (launch tags, counters are cumulative)
    first = bufs[-1]["down"].clone()
    for _ in range(3):
        prog.run(pid)
    torch.cuda.synchronize()
    assert torch.equal(bufs[-1]["down"], first)


def test_union_program_config4_shapes_graph(pg):
    """LLaMA-7B shapes at ratio 0.6 (r_store 1638 / 2388), 256 tokens from 256
    prompts, 2 layers: per-module parity, and CUDA-graph replays equal eager."""
    D, F, T, P = 4096, 11008, 256, 256
    dims = {nm: (1638, 819) for nm in ("q", "k", "v", "o")}
    dims.update({"up": (2388, 1194), "gate": (2388, 1194), "down": (2388, 1194)})
    stack, shapes = build(pg, D, F, dims, 2, P, seed=17171)
    pid = torch.arange(T, device="cuda", dtype=torch.int32)
    x = torch.randn(T, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(4)).to(torch.bfloat16)
    prog, bufs = program(pg, stack, shapes, x, T)
    prog.run(pid)
    torch.cuda.synchronize()
    for lay, b in zip(stack, bufs):
        for nm in LIN:
            assert rel(b[nm].float(), module_ref(lay, nm, b[SRC[nm]], pid.long())) <= TOL_BF16_OUT, nm
    eager = bufs[-1]["down"].clone()
    st = torch.cuda.Stream()
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr, stream=st):
        prog.run(pid)
    for _ in range(3):
        gr.replay()
    torch.cuda.synchronize()
    assert torch.equal(bufs[-1]["down"], eager)


def test_union_program_f32_out_and_errors(pg):
    D, F, T, P = 512, 1024, 64, 8
    dims = {nm: (300, 150) for nm in ("q", "k", "v", "o")}
    dims.update({"up": (700, 350), "gate": (700, 350), "down": (640, 320)})
    stack, shapes = build(pg, D, F, dims, 1, P, seed=7)
    lay = stack[0]
    pid = torch.from_numpy(np.random.default_rng(1).integers(0, P, T).astype(np.int32)).cuda()
    x = torch.randn(T, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(5)).to(torch.bfloat16)
    # f32 outputs (the last module of a program: f32 cannot feed another stage)
    prog = pg.UnionProgram(T)
    y = torch.empty(T, D, device="cuda", dtype=torch.float32)
    prog.add_module([lay["q"][0]], [lay["q"][1]], x, [y])
    prog.run(pid)
    torch.cuda.synchronize()
    assert rel(y, module_ref(lay, "q", x, pid.long())) <= 2e-3
    # an output that overwrites an earlier module's input is refused
    prog2 = pg.UnionProgram(T)
    o = torch.empty(T, D, device="cuda", dtype=torch.bfloat16)
    prog2.add_module([lay["q"][0]], [lay["q"][1]], x, [o])
    with pytest.raises(ValueError):
        prog2.add_module([lay["o"][0]], [lay["o"][1]], o, [x])
    with pytest.raises(IndexError):
        prog2.run([P] * T)


def test_union_program_token_groups(pg):
    """Two independent token groups as separate dependency chains of one
    program (tok_offset): each group's rows equal a single-chain program over
    the whole batch within accumulation order (the split schedules differ)."""
    D, F, T, P = 512, 1024, 128, 16
    dims = {nm: (300, 150) for nm in ("q", "k", "v", "o")}
    dims.update({"up": (700, 350), "gate": (700, 350), "down": (640, 320)})
    stack, shapes = build(pg, D, F, dims, 2, P, seed=21)
    pid = torch.from_numpy(np.random.default_rng(9).integers(0, P, T).astype(np.int32)).cuda()
    x = torch.randn(T, D, device="cuda", generator=torch.Generator(device="cuda").manual_seed(8)).to(torch.bfloat16)
    prog, bufs = program(pg, stack, shapes, x, T)
    prog.run(pid)
    half = T // 2
    prog2 = pg.UnionProgram(half)
    bufs2 = []
    src = x
    for lay in stack:
        b = {"x": src}
        for grp in GROUPS:
            for nm in grp:
                b[nm] = torch.empty(T, shapes[nm][0], device="cuda", dtype=torch.bfloat16)
            for c in range(2):
                rows = slice(c * half, (c + 1) * half)
                prog2.add_module([lay[nm][0] for nm in grp], [lay[nm][1] for nm in grp], b[SRC[grp[0]]][rows],
                                 [b[nm][rows] for nm in grp], tok_offset=c * half, weights_reused=c == 0)
        bufs2.append(b)
        src = b["down"]
    prog2.run(pid)
    torch.cuda.synchronize()
    for lay, b in zip(stack, bufs2):
        for nm in LIN:
            assert rel(b[nm].float(), module_ref(lay, nm, b[SRC[nm]], pid.long())) <= TOL_BF16_OUT, nm
    assert rel(bufs2[-1]["down"].float(), bufs[-1]["down"].float()) <= 2e-2
    with pytest.raises(ValueError):
        prog2.run(pid[:half])  # one pattern id per token of the program (2 groups)
