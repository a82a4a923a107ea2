"""Config-4 step through the persistent union program vs per-module launches
(CUDA-graph replay, CUDA events).  usage: python tools/experiments/exp_prog.py [layers]"""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import bench  # noqa: E402
import paper_2605_08568_b200 as pg  # noqa: E402

layers = int(sys.argv[1]) if len(sys.argv) > 1 else 32
dev = torch.device("cuda", 0)
T = 256
stack, ldims = bench.build_stack(pg, torch, dev, list(range(T)), layers)
tp = torch.arange(T, device=dev, dtype=torch.int32)
x = torch.randn(T, bench.D_MODEL, device=dev).to(torch.bfloat16)
CH = int(os.environ.get("EXP_CHAINS", "1"))  # independent token groups interleaved as separate chains
Tc = T // CH
prog = pg.UnionProgram(Tc)
bufs = []
src = x
for lay in stack:
    b = {"x": src}
    for grp in bench.GROUPS:
        for nm in grp:
            b[nm] = torch.empty(T, bench.LIN[nm][0], device=dev, dtype=torch.bfloat16)
        for c in range(CH):
            rows = slice(c * Tc, (c + 1) * Tc)
            prog.add_module([lay[nm][0] for nm in grp], [lay[nm][1] for nm in grp], b[bench.SRC[grp[0]]][rows],
                            [b[nm][rows] for nm in grp], tok_offset=c * Tc, weights_reused=(c + 1 < CH))
    bufs.append(b)
    src = b["down"]
st = torch.cuda.Stream()
with torch.cuda.stream(st):
    t0 = time.time()
    prog.run(tp)
    st.synchronize()
    print("first run (alloc) s", time.time() - t0, "info", prog.info(), flush=True)


def timeit(fn, reps=20):
    with torch.cuda.stream(st):
        for _ in range(3):
            fn()
        ev = [torch.cuda.Event(enable_timing=True) for _ in range(reps + 1)]
        ev[0].record(st)
        for i in range(reps):
            fn()
            ev[i + 1].record(st)
    st.synchronize()
    return float(np.median([ev[i].elapsed_time(ev[i + 1]) for i in range(reps)]))


ms = timeit(lambda: prog.run(tp))
print(f"program: {ms:.3f} ms/step for {layers} layers = {ms / layers * 1e3:.1f} us/layer, {T / ms * 1e3:.0f} tok/s", flush=True)
# per-module path on the same buffers for reference
def modules():
    for lay, b in zip(stack, bufs):
        for grp in bench.GROUPS:
            pg.module_forward_union([lay[n][0] for n in grp], [lay[n][1] for n in grp], tp, b[bench.SRC[grp[0]]],
                                    out_dtype=torch.bfloat16, outs=[b[n] for n in grp])
with torch.cuda.stream(st):
    modules()
st.synchronize()
ref = bufs[-1]["down"].clone()
with torch.cuda.stream(st):
    prog.run(tp)
st.synchronize()
d = (bufs[-1]["down"].float() - ref.float()).abs().max() / ref.float().abs().max()
print("program vs modules rel", float(d))
gr = torch.cuda.CUDAGraph()
with torch.cuda.graph(gr, stream=st):
    modules()
ms2 = timeit(lambda: gr.replay())
print(f"modules (graph): {ms2:.3f} ms/step = {ms2 / layers * 1e3:.1f} us/layer", flush=True)
if os.environ.get("PG_PROG_DBG"):
    import ctypes as C
    grid = prog.info()[1]
    buf = (C.c_uint64 * (grid * 64))()
    have = C.c_int()
    pg._lib.call("pg_union_prog_debug", prog.handle, buf, grid * 64, C.byref(have))
    a = np.frombuffer(buf, dtype=np.uint64).reshape(grid, 64).astype(np.int64)
    t0 = a[:, 0].min()
    names = ["qkv1", "qkv2", "o1", "o2", "ug1", "ug2", "d1", "d2"]
    def col(k):
        v = a[:, k]
        v = (v[v > 0] - t0) / 1e3
        return f"{np.median(v):7.1f}/{v.max():7.1f}" if v.size else "      -/      -"
    print("phase  W_first      X_first      X_last       acc0_ready   epi_p0       epi_all      flags        done   (med/max us)")
    for f in range(8):
        print(f"{names[f]:5s} " + " ".join(col(k) for k in (49 + f, 33 + f, 41 + f, (57 + f) if f < 7 else 63, 1 + f, 9 + f, 17 + f, 25 + f)))
