"""Helpers shared by the GPU parity tests (inputs + oracle comparison)."""
import numpy as np


def gen(kind, shape, rng):
    if kind == "gauss":
        return rng.standard_normal(shape).astype(np.float32)
    if kind == "grid":      # 2^-8 grid clipped to +-4: exact in fp32 and fp64
        g = rng.standard_normal(shape)
        return np.clip(np.round(g * 256) / 256, -4, 4).astype(np.float32)
    if kind == "int":       # tie-heavy, inc tests/support/oracles.hpp:111-117 with max_abs=2
        return rng.integers(-2, 3, shape).astype(np.float32)
    if kind == "zeros":     # mostly zeros + a few spikes
        g = np.zeros(shape, np.float32)
        m = rng.random(shape) < 0.003
        g[m] = rng.standard_normal(int(m.sum())).astype(np.float32)
        return g
    if kind == "mixed":     # explicit -0.0 and ties
        g = rng.integers(-3, 4, shape).astype(np.float32) * 0.5
        g[g == 0] = -0.0
        return g
    raise ValueError(kind)
