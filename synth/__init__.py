"""Seeded synthetic inputs shared by tests, smoke() and bench.py.

This module holds NO arithmetic of the method (no sums, products, stencils):
only a counter-based generator and the workload recipes of DESIGN.md
section 5.  The CUDA library implements the same generator independently
(``ftn_gen_fill``); tests check the two agree bit for bit.

Generator: element t (0-based, array element order = column-major) of array
``array_id`` under ``seed`` gets ``h = splitmix64(seed ^ (array_id << 56) ^ t)``
and, per mode:
  U01     (h >> 11) * 2^-53                 in [0, 1)
  U11     2 * U01 - 1                        in [-1, 1)   (exact)
  INT8    (h >> 11) % 17 - 8                 integer in [-8, 8]
  LINEAR  t
  MOD1024 t mod 1024
  RAW     low bits of h (integer types; two's complement)
"""
from __future__ import annotations

import numpy as np

SEED = 18824  # the paper's arXiv number
U01, U11, INT8, LINEAR, MOD1024, RAW = 1, 2, 3, 4, 5, 6

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def splitmix64(x: np.ndarray) -> np.ndarray:
    """Vigna's splitmix64 finaliser applied to x + golden gamma (uint64, wrapping)."""
    with np.errstate(over="ignore"):
        z = x.astype(np.uint64) + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def values(n: int, seed: int = SEED, array_id: int = 0, mode: int = U01, dtype=np.float64,
           start: int = 0) -> np.ndarray:
    """Elements t = start .. start+n-1 of the generated sequence as a 1-D array."""
    t = np.arange(start, start + n, dtype=np.uint64)
    key = np.uint64((seed ^ (array_id << 56)) & 0xFFFFFFFFFFFFFFFF)
    dtype = np.dtype(dtype)
    if mode == LINEAR:
        return t.astype(np.int64).astype(dtype) if dtype.kind != "f" else t.astype(dtype)
    if mode == MOD1024:
        return (t % np.uint64(1024)).astype(dtype)
    h = splitmix64(key ^ t)
    if mode == U01:
        return ((h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53).astype(dtype)
    if mode == U11:
        u = (h >> np.uint64(11)).astype(np.float64) * 2.0 ** -53
        return (2.0 * u - 1.0).astype(dtype)
    if mode == INT8:
        return ((h >> np.uint64(11)) % np.uint64(17)).astype(np.int64).astype(dtype) - dtype.type(8)
    if mode == RAW:
        if dtype == np.int64:
            return h.view(np.int64)
        if dtype == np.int32:
            return (h & np.uint64(0xFFFFFFFF)).astype(np.uint32).view(np.int32)
        raise ValueError("RAW is for integer types")
    raise ValueError(f"mode {mode}")


def farray(shape, seed: int = SEED, array_id: int = 0, mode: int = U01, dtype=np.float64) -> np.ndarray:
    """A Fortran-ordered array whose element t (array element order) is values()[t]."""
    n = int(np.prod(shape)) if len(shape) else 1
    return values(n, seed, array_id, mode, dtype).reshape(shape, order="F")


def jacobi_init(shape, seed: int = SEED, array_id: int = 0) -> np.ndarray:
    """Jacobi recipe: interior U[0,1), the face where the last
    subscript is its lower bound = 1.0, every other boundary face 0."""
    u = farray(shape, seed, array_id, U01)
    r = len(shape)
    idx = [slice(None)] * r
    for d in range(r):
        for end in (0, -1):
            idx[d] = end
            u[tuple(idx)] = 0.0
            idx[d] = slice(None)
    idx[r - 1] = 0
    u[tuple(idx)] = 1.0
    return u
