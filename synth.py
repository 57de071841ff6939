"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only the random-number recipe of
DESIGN.md §4 (BASELINE.json configs: "re and im i.i.d. uniform[-1,1) from seed
0"; "values standard-normal re/im from the seed").

* ``uniform_c64(N, batch, seed)``: numpy PCG64(seed), float32 draws u in [0,1),
  value = 2u - 1 (exact in fp32), laid out (batch, N, [re, im]) C-order.
* ``normal_c64(N, batch, seed)``: numpy PCG64(seed) standard_normal in float32.
* ``shard_seed(seed, rank)``: rank p of a weak-scaling run draws its own batch
  from the SeedSequence [seed, rank] (rank 0 keeps ``seed`` itself).
"""
from __future__ import annotations

import numpy as np


def _rng(seed):
    return np.random.Generator(np.random.PCG64(seed))


def uniform_c64(N: int, batch: int, seed=0) -> np.ndarray:
    """complex64 (batch, N), re/im i.i.d. uniform[-1, 1)."""
    a = _rng(seed).random((batch, N, 2), dtype=np.float32)
    a *= 2.0
    a -= 1.0
    return a.view(np.complex64).reshape(batch, N)


def normal_c64(N: int, batch: int, seed=0) -> np.ndarray:
    """complex64 (batch, N), re/im i.i.d. standard normal."""
    a = _rng(seed).standard_normal((batch, N, 2), dtype=np.float32)
    return a.view(np.complex64).reshape(batch, N)


def shard_seed(seed: int, rank: int):
    return seed if rank == 0 else [seed, rank]


def make(dist: str, N: int, batch: int, seed=0) -> np.ndarray:
    if dist == "uniform":
        return uniform_c64(N, batch, seed)
    if dist == "normal":
        return normal_c64(N, batch, seed)
    raise ValueError(dist)
