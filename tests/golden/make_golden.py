"""Generate the golden fixtures from the UNMODIFIED reference (oracle/_ref).

    python tests/golden/make_golden.py

Each fixture is one ClusterConfig run for a few iterations on 2^-8-grid
inputs clipped to +-4 (exactly representable in fp32 and fp64 through every
add of the pipeline, SURVEY 7 hard part 1), storing the inputs, the global
sparse gradient, every worker's residual carry and the ledger maxima after
each iteration.  The fixtures pin the oracle and the device path on boxes
where /root/reference does not exist.
"""
import os
import zlib
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.join(HERE, "..", "..", "oracle"))
from pyoracle import Oracle, make_config  # noqa: E402

CASES = [
    # name, P, N, k, d, sag, residual, timing, iters
    ("p4_d1_gres_opt", 4, 1000, 40, 1, "none", "gres", "optimized", 3),
    ("p6_d1_gres_naive", 6, 997, 60, 1, "none", "gres", "naive", 3),
    ("p5_d1_pres_opt", 5, 503, 35, 1, "none", "pres", "optimized", 3),
    ("p4_d1_lres_opt", 4, 640, 32, 1, "none", "lres", "optimized", 3),
    ("p8_d2_rsag_gres", 8, 800, 64, 2, "rsag", "gres", "optimized", 3),
    ("p8_d8_rsag_gres", 8, 512, 64, 8, "rsag", "gres", "optimized", 3),
    ("p6_d3_bsag_gres", 6, 600, 60, 3, "bsag", "gres", "optimized", 4),
    ("p6_d2_bsag_naive", 6, 606, 48, 2, "bsag", "gres", "naive", 3),
    ("p7_d7_bsag_pres", 7, 490, 70, 7, "bsag", "pres", "optimized", 3),
    ("p9_d3_bsag_gres", 9, 905, 90, 3, "bsag", "gres", "optimized", 3),
]


def grid(rng, shape):
    g = rng.standard_normal(shape)
    return np.clip(np.round(g * 256) / 256, -4, 4)


def main():
    ref = Oracle("ref")
    for name, P, N, k, d, sag, residual, timing, iters in CASES:
        rng = np.random.default_rng(zlib.crc32(name.encode()))
        p = ref.pipeline(make_config(P, N, k, d, sag, residual, timing))
        out = {"cfg": np.array([P, N, k, d]), "modes": np.array([sag, residual, timing]),
               "iters": np.array(iters)}
        for it in range(iters):
            g = grid(rng, (P, N))
            info = p.allreduce(g)
            gi, gv = p.global_gradient()
            out[f"g{it}"] = g
            out[f"gi{it}"] = gi
            out[f"gv{it}"] = gv
            for w in range(P):
                out[f"carry{it}_{w}"] = p.carry(w)
            out[f"ledger{it}"] = np.array([info["max_rounds"], info["max_scalars"]])
        np.savez_compressed(os.path.join(HERE, f"{name}.npz"), **out)
        print("wrote", name)


if __name__ == "__main__":
    main()
