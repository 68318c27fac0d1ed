"""GPU twin of datagen (same Philox counter scheme) for collections too large for the host.

ctypes wrapper over datagen/libparis_datagen.so (built by __graft_entry__.build()).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np
import torch

from . import member_ids

_LIB = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libparis_datagen.so")
_lib = None


def _load():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB):
            raise RuntimeError(f"{_LIB} missing: run __graft_entry__.build()")
        lib = ctypes.CDLL(_LIB)
        P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        lib.paris_datagen_walks.argtypes = [P, i64, i32, ctypes.c_uint64, i64, P]
        lib.paris_datagen_noisy.argtypes = [P, P, i32, i32, ctypes.c_double, ctypes.c_uint64, P, P]
        _lib = lib
    return _lib


def _st():
    return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)


def walks(n: int, length: int, seed: int, first_id: int = 0, out: torch.Tensor | None = None,
          device="cuda") -> torch.Tensor:
    """[n][length] fp32 z-normalized random walks on the GPU (ids first_id..)."""
    if out is None:
        out = torch.empty((n, length), dtype=torch.float32, device=device)
    rc = _load().paris_datagen_walks(out.data_ptr(), n, length, int(seed) & (2**64 - 1), first_id, _st())
    if rc:
        raise RuntimeError(f"paris_datagen_walks failed ({rc})")
    return out


def noisy_members(data: torch.Tensor, nq: int, sigma: float, seed: int):
    """(queries [nq][len] on the GPU, source ids int64 numpy): data[src] + N(0, sigma^2), re-z-normalized."""
    n, length = data.shape
    src = member_ids(nq, n, seed)
    src_d = torch.from_numpy(src).to(data.device)
    out = torch.empty((nq, length), dtype=torch.float32, device=data.device)
    rc = _load().paris_datagen_noisy(data.data_ptr(), src_d.data_ptr(), nq, length, float(sigma),
                                     int(seed) & (2**64 - 1), out.data_ptr(), _st())
    if rc:
        raise RuntimeError(f"paris_datagen_noisy failed ({rc})")
    return out, src


def config_workload(config: int, device="cuda", n_override: int | None = None):
    """BASELINE.json config 1..5 as (raw [n][len] on GPU, query sets {name: (queries, k list)}).

    Seeds: datagen.config_seeds(config).
    """
    from . import config_seeds
    ds, qs = config_seeds(config)
    spec = {
        1: (100_000, 256), 2: (1_000_000, 256), 3: (10_000_000, 128),
        4: (100_000_000, 256), 5: (20_000_000, 256),
    }[config]
    n, length = spec
    if n_override:
        n = n_override
    raw = walks(n, length, ds, device=device)
    sets = {}
    if config in (1, 3, 4):
        nq = {1: 100, 3: 1000, 4: 100}[config]
        sets["fresh"] = (walks(nq, length, qs, device=device), [1])
    elif config == 2:
        q, _ = noisy_members(raw, 1000, 0.05, qs)
        sets["noise0.05"] = (q, [1, 10])
    else:
        for i, sg in enumerate((0.01, 0.02, 0.05, 0.1, 0.2)):
            q, _ = noisy_members(raw, 200, sg, qs + i)
            sets[f"noise{sg}"] = (q, [1, 100])
    return raw, sets


__all__ = ["walks", "noisy_members", "config_workload", "np"]
