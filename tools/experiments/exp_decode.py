"""Decode-chain experiment driver (timing only, no parity): MLP block decode
step with R weight replicas, optional prefetch, fused vs unfused, single
linear.  Usage: python tools/experiments/exp_decode.py [replicas] [steps]"""
import os
import sys
import time

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import paper_2605_08568_b200 as pg  # noqa: E402
import bench  # noqa: E402


def main():
    R = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    steps = int(sys.argv[2]) if len(sys.argv) > 2 else 512
    dev = torch.device("cuda", 0)
    sh = bench.shapes()
    blocks = [bench.build_block(pg, torch, sh, dev, j) for j in range(R)]
    pats = pg.make_patterns(17171, 1, [(sh[k][3], sh[k][2]) for k in ("up", "gate", "down")])[0]
    aggs = [{k: pg.aggregate_layout(b[k], [p], 0.9) for k, p in zip(("up", "gate", "down"), pats)} for b in blocks]
    x = torch.randn(4096, device=dev).to(torch.bfloat16)
    y = torch.empty(4096, device=dev)
    act = torch.empty(11008, device=dev, dtype=torch.bfloat16)
    up = torch.empty(11008, device=dev)
    st = torch.cuda.Stream()

    def run(fn, n=steps):
        with torch.cuda.stream(st):
            for i in range(32):
                fn(i)
            g = torch.cuda.CUDAGraph()
            with torch.cuda.graph(g, stream=st):
                for i in range(64):
                    fn(i)
            g.replay()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record(st)
            for _ in range(n // 64):
                g.replay()
            e1.record(st)
        torch.cuda.synchronize()
        ts = [e0.elapsed_time(e1) / (n // 64 * 64) * 1e3]
        for _ in range(4):  # more trials: report the median
            with torch.cuda.stream(st):
                e0.record(st)
                for _ in range(n // 64):
                    g.replay()
                e1.record(st)
            torch.cuda.synchronize()
            ts.append(e0.elapsed_time(e1) / (n // 64 * 64) * 1e3)
        return sorted(ts)[len(ts) // 2]

    mlp = lambda i: pg.mlp_forward(aggs[i % R]["up"], aggs[i % R]["gate"], aggs[i % R]["down"], 0, x, out=y, act=act)
    lin = lambda i: pg.aggregated_forward(aggs[i % R]["up"], 0, x, out=up)
    lind = lambda i: pg.aggregated_forward(aggs[i % R]["down"], 0, act, out=y)
    only = os.environ.get("EXP_ONLY")
    for name, fn in (("mlp", mlp), ("up", lin), ("down", lind)):
        if only and name != only:
            continue
        print(f"R={R} prefetch={os.environ.get('PG_CHAIN_PREFETCH', '1')}: {name} {run(fn):.1f} us", flush=True)
        if os.environ.get("PG_CHAIN_DBG"):
            stamps()




def stamps():
    """PG_CHAIN_DBG=1: per-phase breakdown of the last chain launch (us from CTA start)."""
    import ctypes as C
    import numpy as np
    from paper_2605_08568_b200 import _lib
    buf = (C.c_uint64 * (1024 * 16))()
    _lib.call("pg_chain_debug_dump", buf, 1024 * 16)
    a = np.frombuffer(buf, dtype=np.uint64).reshape(1024, 16)[:148].astype(np.int64)
    t0 = a[:, 0].min()
    names = ["start", "x0", "s1done0", "bar0", "z0", "s2done0", "xstaged0", "x1", "s1done1", "bar1", "z1", "s2done1",
             "prod_done", "end", "s1data1"]
    for k, nm in enumerate(names):
        col = a[:, k]
        if (col > 0).all():
            print(f"{nm:9s} min {(col.min() - t0) / 1e3:7.2f} med {(np.median(col) - t0) / 1e3:7.2f} "
                  f"max {(col.max() - t0) / 1e3:7.2f} us")
            if nm in ("start", "s1done0", "s2done0", "s1done1", "prod_done", "s1data1") and os.environ.get("EXP_LATE"):
                late = np.argsort(col)[-8:][::-1]
                print("    latest CTAs:", [(int(c), round((col[c] - t0) / 1e3, 2)) for c in late])


if __name__ == "__main__":
    main()
