"""CPU oracle for the ParIS+ exact k-NN hot path -- TEST INFRASTRUCTURE ONLY.

Thin ctypes wrapper over ``oracle/oracle.c`` (plain C, double precision,
single-threaded; every function cites the PAPER.md passage it follows).  Only
``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (cpu_baseline leg and
``--impl reference``) may import this package.  The product path
(``paper_2009_00166_b200``) never imports it and shares no code with it.

Layouts: raw / queries [n][len] fp32 row-major; SAX here is row-major [n][w]
(the paper's SAX[p] array) -- the CUDA path stores [w][n].
"""
from __future__ import annotations

import ctypes
import os
import subprocess
import threading

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_SRC = os.path.join(_HERE, "oracle.c")
_LIB = os.path.join(_HERE, "liboracle.so")
_lock = threading.Lock()
_lib = None

CFLAGS = ["-O2", "-ffp-contract=off", "-fno-fast-math", "-fPIC", "-shared", "-std=c99"]


def build(force: bool = False) -> str:
    """Compile oracle.c -> liboracle.so with gcc (no -ffast-math, no FMA contraction)."""
    if force or not os.path.exists(_LIB) or os.path.getmtime(_LIB) < os.path.getmtime(_SRC):
        tmp = _LIB + f".tmp{os.getpid()}"
        subprocess.check_call(["gcc", *CFLAGS, "-o", tmp, _SRC, "-lm"])
        os.replace(tmp, _LIB)
    return _LIB


def _load():
    global _lib
    with _lock:
        if _lib is None:
            build()
            lib = ctypes.CDLL(_LIB)
            P = ctypes.c_void_p
            i64, i32, dbl = ctypes.c_int64, ctypes.c_int, ctypes.c_double
            lib.oracle_cuts.argtypes = [i32, P]
            lib.oracle_paa.argtypes = [P, i32, i32, P]
            lib.oracle_sax_symbol.argtypes = [dbl, P, i32]
            lib.oracle_summarize.argtypes = [P, i64, i32, i32, i32, P]
            lib.oracle_lb_table.argtypes = [P, i32, i32, i32, P]
            lib.oracle_lb2.argtypes = [P, P, i32, i32]
            lib.oracle_lb2.restype = dbl
            lib.oracle_ed2.argtypes = [P, P, i32]
            lib.oracle_ed2.restype = dbl
            lib.oracle_ed2_abandon.argtypes = [P, P, i32, dbl]
            lib.oracle_ed2_abandon.restype = dbl
            lib.oracle_knn_bruteforce.argtypes = [P, i64, i32, P, i32, i32, P, P]
            lib.oracle_knn_pruned.argtypes = [P, P, i64, i32, i32, i32, P, i32, i32, P, P, P]
            _lib = lib
    return _lib


def _p(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


def _f32(a):
    return np.ascontiguousarray(a, dtype=np.float32)


def cuts(card: int) -> np.ndarray:
    """Breakpoints cut_1..cut_{card-1} (float64, length card-1)."""
    out = np.zeros(256, dtype=np.float64)
    if _load().oracle_cuts(int(card), _p(out)):
        raise ValueError(f"card must be a power of two in [2, 256], got {card}")
    return out[: card - 1].copy()


def paa(x: np.ndarray, w: int) -> np.ndarray:
    """PAA of each row of x ([m][len] or [len]) -> float64 [m][w]."""
    x = _f32(np.atleast_2d(x))
    m, length = x.shape
    if length % w:
        raise ValueError("w must divide len")
    out = np.zeros((m, w), dtype=np.float64)
    lib = _load()
    for i in range(m):
        row = np.ascontiguousarray(x[i])
        lib.oracle_paa(_p(row), length, w, _p(out[i]))
    return out


def sax_symbol(v: float, card: int) -> int:
    c = np.zeros(256, dtype=np.float64)
    lib = _load()
    lib.oracle_cuts(int(card), _p(c))
    return int(lib.oracle_sax_symbol(float(v), _p(c), int(card)))


def summarize(raw: np.ndarray, w: int, card: int) -> np.ndarray:
    """SAX words of every row -> uint8 [n][w] (row-major)."""
    raw = _f32(raw)
    n, length = raw.shape
    out = np.zeros((n, w), dtype=np.uint8)
    rc = _load().oracle_summarize(_p(raw), n, length, w, card, _p(out))
    if rc:
        raise ValueError(f"oracle_summarize failed ({rc})")
    return out


def lb_table(qpaa: np.ndarray, length: int, w: int, card: int) -> np.ndarray:
    """MINDIST dictionaries T[s][c] = (len/w) * delta^2 (float64 [w][card])."""
    qpaa = np.ascontiguousarray(qpaa, dtype=np.float64)
    T = np.zeros((w, card), dtype=np.float64)
    if _load().oracle_lb_table(_p(qpaa), length, w, card, _p(T)):
        raise ValueError("bad card")
    return T


def lb2(T: np.ndarray, words: np.ndarray) -> np.ndarray:
    """LB^2 of each word (uint8 [m][w]) from table T (float64 [w][card])."""
    T = np.ascontiguousarray(T, dtype=np.float64)
    words = np.ascontiguousarray(np.atleast_2d(words), dtype=np.uint8)
    w, card = T.shape
    lib = _load()
    return np.array([lib.oracle_lb2(_p(T), _p(np.ascontiguousarray(words[i])), w, card)
                     for i in range(words.shape[0])], dtype=np.float64)


def ed2(a: np.ndarray, b: np.ndarray) -> float:
    a, b = _f32(a), _f32(b)
    return float(_load().oracle_ed2(_p(a), _p(b), a.shape[-1]))


def ed2_abandon(a: np.ndarray, b: np.ndarray, limit: float) -> float:
    a, b = _f32(a), _f32(b)
    return float(_load().oracle_ed2_abandon(_p(a), _p(b), a.shape[-1], float(limit)))


def knn_bruteforce(raw: np.ndarray, queries: np.ndarray, k: int):
    """Plain k-NN: (ids int64 [nq][k], d2 float64 [nq][k]) ascending by (d2, id)."""
    raw, queries = _f32(raw), _f32(np.atleast_2d(queries))
    n, length = raw.shape
    nq = queries.shape[0]
    idx = np.zeros((nq, k), dtype=np.int64)
    d2 = np.zeros((nq, k), dtype=np.float64)
    rc = _load().oracle_knn_bruteforce(_p(raw), n, length, _p(queries), nq, k, _p(idx), _p(d2))
    if rc:
        raise ValueError(f"oracle_knn_bruteforce failed ({rc})")
    return idx, d2


def knn_pruned(raw: np.ndarray, sax_nw: np.ndarray, queries: np.ndarray, k: int, w: int,
               card: int, stats: np.ndarray | None = None):
    """LB-pruned exact k-NN over row-major SAX [n][w]; returns (ids, d2) like knn_bruteforce.

    stats (int64[3], optional, accumulated): LB computations, raw series read, BSF updates.
    """
    raw, queries = _f32(raw), _f32(np.atleast_2d(queries))
    sax_nw = np.ascontiguousarray(sax_nw, dtype=np.uint8)
    n, length = raw.shape
    nq = queries.shape[0]
    idx = np.zeros((nq, k), dtype=np.int64)
    d2 = np.zeros((nq, k), dtype=np.float64)
    st = None
    if stats is not None:
        assert stats.dtype == np.int64 and stats.size >= 3
        st = _p(stats)
    rc = _load().oracle_knn_pruned(_p(raw), _p(sax_nw), n, length, w, card, _p(queries), nq, k,
                                   _p(idx), _p(d2), st)
    if rc:
        raise ValueError(f"oracle_knn_pruned failed ({rc})")
    return idx, d2
