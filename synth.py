"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

Holds none of the method's arithmetic: only the random-number recipe of
DESIGN.md §4 (BASELINE.json configs: "re and im i.i.d. uniform[-1,1) from seed
0"; "values standard-normal re/im from the seed").

* ``uniform_c64(N, batch, seed)``: numpy PCG64(seed), float32 draws u in [0,1),
  value = 2u - 1 (exact in fp32), laid out (batch, N, [re, im]) C-order.
* ``normal_c64(N, batch, seed)``: numpy PCG64(seed) standard_normal in float32.
* ``uniform_c64_rows(N, b0, b1, seed)``: transforms [b0, b1) of ``uniform_c64(N, B, seed)``
  for any B >= b1, drawn without generating the rows before b0: one complex64 element is
  two float32 draws = one 64-bit PCG64 output, so the stream is advanced by N*b0 outputs
  (``PCG64.advance``).  A batch shard or a six-step slab is bit-identical to the same rows
  of the one-GPU input.
* ``shard_range(batch, rank, world)``: the contiguous batch partition
  [floor(rank*B/P), floor((rank+1)*B/P)) of SURVEY §8(e).
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


def uniform_c64_rows(N: int, b0: int, b1: int, seed: int = 0) -> np.ndarray:
    """complex64 (b1 - b0, N): rows [b0, b1) of uniform_c64(N, B, seed), any B >= b1."""
    bg = np.random.PCG64(seed)
    bg.advance(N * b0)  # one 64-bit output per complex element (two float32 draws)
    a = np.random.Generator(bg).random((b1 - b0, N, 2), dtype=np.float32)
    a *= 2.0
    a -= 1.0
    return a.view(np.complex64).reshape(b1 - b0, N)


def shard_range(batch: int, rank: int, world: int):
    """Contiguous batch partition of SURVEY §8(e): rank r owns [floor(rB/P), floor((r+1)B/P))."""
    return (rank * batch) // world, ((rank + 1) * batch) // world


def make(dist: str, N: int, batch: int, seed=0) -> np.ndarray:
    if dist == "uniform":
        return uniform_c64(N, batch, seed)
    if dist == "normal":
        return normal_c64(N, batch, seed)
    raise ValueError(dist)
