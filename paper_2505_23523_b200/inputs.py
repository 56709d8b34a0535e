"""Seeded synthetic inputs shared by the CUDA path's tests/bench and the oracle.

This module holds NONE of the method's arithmetic: it only draws the n input
buffers.  Recipe:

* seed = 2505_23523 + 1000*config + rank, numpy PCG64;
* "normal":  N(0,1) float32 (int32: uniform over the full 32-bit range, which
  exercises wraparound);
* "intval":  integers uniform in [-16, 16] (exact in every dtype for n <= 8);
* "bitmask": x_p[i] = 1 << p (every element of the sum is 2**n - 1; a missed
  or doubled contribution names the faulty rank);
* bfloat16 buffers are returned as uint16 bit patterns: the float32 draw with
  its low 16 bits dropped (truncation, not the method's RNE rounding).
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 2505_23523
PATTERNS = ("normal", "intval", "bitmask")


def seed_for(config: int, rank: int) -> int:
    return SEED_BASE + 1000 * config + rank


def make_input(count: int, dtype: str, rank: int, config: int = 1, pattern: str = "normal") -> np.ndarray:
    rng = np.random.Generator(np.random.PCG64(seed_for(config, rank)))
    if pattern == "normal":
        if dtype == "int32":
            return rng.integers(-(2 ** 31), 2 ** 31, size=count, dtype=np.int64).astype(np.int32)
        f = rng.standard_normal(count, dtype=np.float32)
    elif pattern == "intval":
        f = rng.integers(-16, 17, size=count, dtype=np.int32)
        if dtype == "int32":
            return f
        f = f.astype(np.float32)
    elif pattern == "bitmask":
        if dtype == "int32":
            return np.full(count, 1 << rank, dtype=np.int32)
        f = np.full(count, float(1 << rank), dtype=np.float32)
    else:
        raise ValueError(pattern)
    if dtype == "float32":
        return f
    if dtype == "bfloat16":
        return (f.view(np.uint32) >> np.uint32(16)).astype(np.uint16)
    raise ValueError(dtype)


def make_inputs(n: int, count: int, dtype: str, config: int = 1, pattern: str = "normal"):
    return [make_input(count, dtype, p, config, pattern) for p in range(n)]
