"""Seeded synthetic inputs shared by the oracle side and the CUDA side.

This module holds NONE of the method's arithmetic (no PAA, no SAX, no lower
bound, no distance): it only draws the paper's synthetic workload, so both the
oracle (``oracle/``) and the product path (``paper_2009_00166_b200``) can be fed
identical bytes.

Workload ("Datasets"): random walks, x0 ~ N(0,1),
x_t = x_{t-1} + N(0,1); series are z-normalized (SURVEY §8(c) reading 9).
Query workloads (BASELINE.json configs): fresh random walks from a separate seed,
or a dataset member plus N(0, sigma^2) noise per point, re-z-normalized.

Generator: Philox4x32-10, counter = (series id lo, series id hi,
point/4, stream tag), key = (seed lo, seed hi); standard normals by Box-Muller
in double; cumulative sum and z-normalization in double; stored as fp32.
The same counter-based generator is implemented in CUDA in ``datagen.cu`` for
collections too large to draw on the host (config 4 = 102.4 GB).
"""
from __future__ import annotations

import numpy as np

__all__ = [
    "philox4x32", "normals", "random_walks", "noisy_members", "member_ids",
    "config_seeds", "STREAM_WALK", "STREAM_NOISE", "STREAM_PICK",
]

# Stream tags (counter word 3) keep the independent draws apart.
STREAM_WALK = 0
STREAM_NOISE = 1
STREAM_PICK = 2

_M0 = np.uint64(0xD2511F53)
_M1 = np.uint64(0xCD9E8D57)
_W0 = np.uint32(0x9E3779B9)
_W1 = np.uint32(0xBB67AE85)
_MASK32 = np.uint64(0xFFFFFFFF)


def philox4x32(c0, c1, c2, c3, k0, k1, rounds: int = 10):
    """Philox4x32-10 (Salmon et al., SC'11) on uint32 arrays; returns 4 uint32 arrays."""
    c0 = np.asarray(c0, dtype=np.uint32).copy()
    c1 = np.asarray(c1, dtype=np.uint32).copy()
    c2 = np.asarray(c2, dtype=np.uint32).copy()
    c3 = np.asarray(c3, dtype=np.uint32).copy()
    c0, c1, c2, c3 = np.broadcast_arrays(c0, c1, c2, c3)
    c0, c1, c2, c3 = (a.copy() for a in (c0, c1, c2, c3))
    k0 = np.uint32(k0)
    k1 = np.uint32(k1)
    with np.errstate(over="ignore"):
        for _ in range(rounds):
            p0 = _M0 * c0.astype(np.uint64)
            p1 = _M1 * c2.astype(np.uint64)
            hi0 = (p0 >> np.uint64(32)).astype(np.uint32)
            lo0 = (p0 & _MASK32).astype(np.uint32)
            hi1 = (p1 >> np.uint64(32)).astype(np.uint32)
            lo1 = (p1 & _MASK32).astype(np.uint32)
            c0, c1, c2, c3 = hi1 ^ c1 ^ k0, lo1, hi0 ^ c3 ^ k1, lo0
            k0 = np.uint32(k0 + _W0)
            k1 = np.uint32(k1 + _W1)
    return c0, c1, c2, c3


def _split_seed(seed: int):
    seed = int(seed) & 0xFFFFFFFFFFFFFFFF
    return seed & 0xFFFFFFFF, seed >> 32


def normals(ids: np.ndarray, length: int, seed: int, stream: int) -> np.ndarray:
    """Standard normals z[i, t] for series ids ``ids`` (float64, shape [len(ids), length]).

    Counter (id lo, id hi, t // 4, stream); each Philox block gives 4 uint32 ->
    two Box-Muller pairs -> points 4b .. 4b+3.
    """
    ids = np.asarray(ids, dtype=np.uint64)
    nblk = (length + 3) // 4
    k0, k1 = _split_seed(seed)
    idlo = (ids & _MASK32).astype(np.uint32)[:, None]
    idhi = (ids >> np.uint64(32)).astype(np.uint32)[:, None]
    blk = np.arange(nblk, dtype=np.uint32)[None, :]
    r0, r1, r2, r3 = philox4x32(idlo, idhi, blk, np.uint32(stream), k0, k1)
    scale = 2.0 ** -32

    def bm(a, b):
        u1 = (a.astype(np.float64) + 0.5) * scale
        u2 = (b.astype(np.float64) + 0.5) * scale
        rad = np.sqrt(-2.0 * np.log(u1))
        ang = 2.0 * np.pi * u2
        return rad * np.cos(ang), rad * np.sin(ang)

    z0, z1 = bm(r0, r1)
    z2, z3 = bm(r2, r3)
    z = np.stack([z0, z1, z2, z3], axis=-1).reshape(len(ids), nblk * 4)
    return z[:, :length]


def _znorm_f32(x: np.ndarray) -> np.ndarray:
    """z-normalize rows in double (population std); flat rows -> zeros."""
    mu = x.mean(axis=1, keepdims=True)
    sd = np.sqrt(((x - mu) ** 2).mean(axis=1, keepdims=True))
    out = np.where(sd < 1e-8, 0.0, (x - mu) / np.where(sd < 1e-8, 1.0, sd))
    return out.astype(np.float32)


def random_walks(n: int, length: int, seed: int, first_id: int = 0,
                 znorm: bool = True) -> np.ndarray:
    """[n, length] fp32 z-normalized random walks, ids first_id.."""
    ids = np.arange(first_id, first_id + n, dtype=np.uint64)
    out = np.empty((n, length), dtype=np.float32)
    step = max(1, (1 << 22) // max(1, length))
    for a in range(0, n, step):
        b = min(n, a + step)
        z = normals(ids[a:b], length, seed, STREAM_WALK)
        x = np.cumsum(z, axis=1)
        out[a:b] = _znorm_f32(x) if znorm else x.astype(np.float32)
    return out


def member_ids(nq: int, n: int, seed: int) -> np.ndarray:
    """Source ids for member+noise queries: uniform in [0, n) from the query seed."""
    j = np.arange(nq, dtype=np.uint64)
    k0, k1 = _split_seed(seed)
    r0, r1, _, _ = philox4x32((j & _MASK32).astype(np.uint32),
                              (j >> np.uint64(32)).astype(np.uint32),
                              np.uint32(0), np.uint32(STREAM_PICK), k0, k1)
    v = (r1.astype(np.uint64) << np.uint64(32)) | r0.astype(np.uint64)
    return (v % np.uint64(n)).astype(np.int64)


def noisy_members(data: np.ndarray, src: np.ndarray, sigma: float, seed: int) -> np.ndarray:
    """Queries = data[src] + N(0, sigma^2) per point, re-z-normalized (BASELINE configs 2, 5)."""
    length = data.shape[1]
    z = normals(np.arange(len(src), dtype=np.uint64), length, seed, STREAM_NOISE)
    x = data[np.asarray(src)].astype(np.float32) + (sigma * z).astype(np.float32)
    return _znorm_f32(x.astype(np.float64))


def config_seeds(config: int):
    """(dataset seed, query seed) for BASELINE.json config 1..5."""
    ds = 200900166 + int(config)
    return ds, ds + 1000
