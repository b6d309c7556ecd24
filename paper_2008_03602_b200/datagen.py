"""Seeded synthetic inputs shared by tests, bench and the oracle checks.

Holds none of the method's arithmetic: only the input recipe of SURVEY.md
8(d) / DESIGN.md "Input recipe" (numpy PCG64, reproducible on any host):

* x    ~ U[-1, 1)                         (activations, logical NCHW)
* w    ~ U[-1, 1) * sqrt(3 / (Cg R S))    (unit-variance outputs, logical KCRS)
* bias ~ U[-0.1, 0.1)
* integer-exact set: x, w in {-3..3}, bias in {-2..2} (every product and
  partial sum of fp32 accumulation is an exact integer, check O11)

Seeds: data = 20080360 + 1000 * config + layer; sampler = 42 + fraction index.
"""
from __future__ import annotations

import numpy as np

DATA_SEED_BASE = 20080360


def data_seed(config: int, layer: int) -> int:
    return DATA_SEED_BASE + 1000 * config + layer


def sampler_seed(fraction_index: int) -> int:
    return 42 + fraction_index


def make_inputs(shape: dict, seed: int, integer: bool = False):
    """Return (x NCHW, w KCRS, bias K) as float32 numpy arrays."""
    rng = np.random.Generator(np.random.PCG64(seed))
    n, c, h, w, k, r, s = (shape[a] for a in ("n", "c", "h", "w", "k", "r", "s"))
    cg = c // shape.get("groups", 1)
    if integer:
        x = rng.integers(-3, 4, size=(n, c, h, w)).astype(np.float32)
        wt = rng.integers(-3, 4, size=(k, cg, r, s)).astype(np.float32)
        b = rng.integers(-2, 3, size=(k,)).astype(np.float32)
    else:
        x = rng.uniform(-1.0, 1.0, size=(n, c, h, w)).astype(np.float32)
        wt = (rng.uniform(-1.0, 1.0, size=(k, cg, r, s)) * np.sqrt(3.0 / (cg * r * s))).astype(np.float32)
        b = rng.uniform(-0.1, 0.1, size=(k,)).astype(np.float32)
    return x, wt, b


def sample_points(total: int, count: int, seed: int) -> np.ndarray:
    """Fixed output positions for the sampled correctness gate (flat NKPQ
    indices, sorted, without replacement); the whole tensor if it is small."""
    if total <= count:
        return np.arange(total, dtype=np.int64)
    rng = np.random.Generator(np.random.PCG64(seed))
    return np.sort(rng.choice(total, size=count, replace=False)).astype(np.int64)
