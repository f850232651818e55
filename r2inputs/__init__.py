"""Seeded synthetic input generators shared by the oracle, the tests and bench.py.

This module holds NO arithmetic of the method (no reduction, no rounding rule,
no geometry).  It only draws the per-rank input buffers, so that the CPU
oracle (`oracle/`) and the CUDA path (`paper_2512_25059_b200/`) read
bit-identical inputs without sharing any code.

Recipe (SURVEY.md §8(d) "Configs as concrete synthetic inputs"):

* seed base ``0x52324343`` ("R2CC"); rank r uses
  ``seed ^ ((r * 0x9E3779B97F4A7C15) mod 2**64)`` with numpy PCG64;
* int32: uniform in [-2**24, 2**24) ("wrap" variant: full int32 range);
* fp32: N(0, 1);
* bf16: N(0, 1) drawn in fp32, then the upper 16 bits of the fp32 pattern are
  kept (truncation -- an input recipe, not the method's rounding).  bf16 data
  is carried as ``uint16`` bit patterns.
"""
from __future__ import annotations

import numpy as np

SEED_BASE = 0x52324343
GOLDEN = 0x9E3779B97F4A7C15
DTYPES = ("int32", "float32", "bfloat16")


def rank_seed(seed: int, rank: int) -> int:
    return (seed ^ ((rank * GOLDEN) % (1 << 64))) % (1 << 64)


def rank_input(n_elems: int, dtype: str, rank: int, seed: int = SEED_BASE,
               dist: str = "default") -> np.ndarray:
    """One rank's input buffer (numpy, host)."""
    rng = np.random.Generator(np.random.PCG64(rank_seed(seed, rank)))
    if dtype == "int32":
        if dist == "wrap":
            return rng.integers(-(2 ** 31), 2 ** 31, size=n_elems, dtype=np.int64).astype(np.int32)
        if dist == "smallint":
            return rng.integers(-16, 16, size=n_elems, dtype=np.int64).astype(np.int32)
        return rng.integers(-(2 ** 24), 2 ** 24, size=n_elems, dtype=np.int64).astype(np.int32)
    if dtype == "float32":
        if dist == "smallint":
            return rng.integers(-16, 16, size=n_elems).astype(np.float32)
        return rng.standard_normal(n_elems, dtype=np.float32)
    if dtype == "bfloat16":
        if dist == "smallint":
            f = rng.integers(-16, 16, size=n_elems).astype(np.float32)
        else:
            f = rng.standard_normal(n_elems, dtype=np.float32)
        return (f.view(np.uint32) >> 16).astype(np.uint16)
    raise ValueError(f"unknown dtype {dtype!r}")


def inputs(n_ranks: int, n_elems: int, dtype: str, seed: int = SEED_BASE,
           dist: str = "default") -> list[np.ndarray]:
    """All ranks' input buffers."""
    return [rank_input(n_elems, dtype, r, seed, dist) for r in range(n_ranks)]


def elem_bytes(dtype: str) -> int:
    return {"int32": 4, "float32": 4, "bfloat16": 2}[dtype]
