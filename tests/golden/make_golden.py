"""Generate tests/golden/*.npz from the REFERENCE compiled here (oracle/_ref).

Run in the build container (needs /root/reference): `python tests/golden/make_golden.py`.
Inputs are regenerated from seeds with the reference's own Rng (rng.hpp:10-41),
so the fixture stores seeds + shapes + reference outputs only.
"""
import ctypes as C
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
sys.path.insert(0, ROOT)
from oracle import build as obuild  # noqa: E402
from oracle import pyoracle  # noqa: E402


def main():
    obuild.build()
    ref = pyoracle.Oracle("reference")
    f = ref.lib.ref_fill_gaussian
    f.argtypes = [C.c_uint64, C.POINTER(C.c_double), C.c_size_t]

    def gauss(seed, shape):
        out = np.empty(int(np.prod(shape)))
        f(seed, out.ctypes.data_as(C.POINTER(C.c_double)), out.size)
        return out.reshape(shape)

    n, T, r, K, m, N = 256, 16, 96, 40, 128, 64
    seeds = dict(seed_x=501, seed_theta=502, seed_emb=503, seed_A=504, seed_B=505)
    x = gauss(seeds["seed_x"], (n, T))
    theta = gauss(seeds["seed_theta"], (r, n))
    h = ref.mean_pool(x)
    z = ref.score(theta, np.zeros(r), h)
    sel = ref.select_topk(z, K)
    emb = gauss(seeds["seed_emb"], (N, n))
    q = emb[7] + 0.05 * gauss(506, (n,))
    entry, sim, hit = ref.retrieve(emb, 0.8, q)
    A = gauss(seeds["seed_A"], (m, r))
    B = gauss(seeds["seed_B"], (n, r))
    y = ref.masked_forward(A, B, sel, x)
    np.savez_compressed(
        os.path.join(os.path.dirname(__file__), "route_cache_values.npz"),
        x_shape=np.array([n, T]), theta_shape=np.array([r, n]), emb_shape=np.array([N, n]),
        A_shape=np.array([m, r]), B_shape=np.array([n, r]), K=np.array(K), min_sim=np.array(0.8),
        h=h, logits=z, sel=sel, query=q, entry=np.array(entry), similarity=np.array(sim),
        hit=np.array(hit), y_masked=y, **{k: np.array(v) for k, v in seeds.items()})
    print("entry", entry, "sim", sim, "hit", hit, "sel[:8]", sel[:8])


if __name__ == "__main__":
    main()
