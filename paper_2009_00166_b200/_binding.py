"""ctypes binding for libparis.so (include/paris.h).  Marshalling only."""
from __future__ import annotations

import ctypes
import os
import re
import threading
from dataclasses import dataclass

import torch

_PKG = os.path.dirname(os.path.abspath(__file__))
_ROOT = os.path.dirname(_PKG)
_LIBPATH = os.path.join(_PKG, "libparis.so")
_HEADER = os.path.join(_ROOT, "include", "paris.h")

PARIS_EINVAL = -1
PARIS_ECONFIG = -2
PARIS_ECUDA = -3
PARIS_ENOMEM = -4
PARIS_MAX_K = 1024

_lock = threading.Lock()
_lib = None


class ParisError(RuntimeError):
    def __init__(self, code: int, msg: str):
        super().__init__(f"libparis error {code}: {msg}")
        self.code = code


class _Config(ctypes.Structure):
    _fields_ = [("batch", ctypes.c_int32), ("seed_div", ctypes.c_int32),
                ("wave_a", ctypes.c_int32), ("reserved", ctypes.c_int32 * 5), ("tau_in", ctypes.c_void_p)]


class _Stats(ctypes.Structure):
    _fields_ = [("candidates", ctypes.c_void_p), ("refined", ctypes.c_void_p),
                ("tau_seed", ctypes.c_void_p), ("lb_blocks", ctypes.c_void_p),
                ("bsf_updates", ctypes.c_void_p), ("raw16_rows", ctypes.c_void_p),
                ("paa_rows", ctypes.c_void_p)]


class _Aux(ctypes.Structure):
    _fields_ = [("raw_bf16", ctypes.c_void_p), ("paa16", ctypes.c_void_p), ("w2", ctypes.c_int32),
                ("reserved", ctypes.c_int32)]


class _KProf(ctypes.Structure):
    _fields_ = [("name", ctypes.c_char * 48), ("launches", ctypes.c_int64),
                ("total_ms", ctypes.c_double)]


@dataclass
class KnnConfig:
    batch: int = 0      # queries per SAX pass: flat 1..16 (default 16), index 1..64 (default 64)
    seed_div: int = 0   # seed sample = n / seed_div (0 = 16)
    wave_a: int = 0     # k = 1: first refinement wave per query (0 = 2048)
    force_direct: bool = False  # test hook: use the direct-load LB kernels even where the TMA-tiled ones apply
    sorted_refine: bool = False  # k = 1: refine the bucket-sorted lists (K5 scatter) instead of the unsorted waves
    index_seeds: int = 0        # index mode: seed series around the leaf (0 = 1024, 2048 from 5e7 series, 32k for k > 1; 64 with host raw and no bf16 copy)
    seed_from_out: bool = False  # test hook: seed from the rows already in out_idx/out_dist (device)
    tau_in: "torch.Tensor | None" = None  # [nq] float32 CUDA: external bound of each query's k-th NN distance
    cap: int = 0                # test hook: candidate-buffer capacity per query (forces the overflow fallback)


def library_path() -> str:
    return _LIBPATH


def load():
    """Load libparis.so (must have been built: __graft_entry__.build()).  Raises if missing."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(_LIBPATH):
            raise ParisError(PARIS_ECUDA, f"CUDA extension not built: {_LIBPATH} is missing "
                             "(run python -c 'import __graft_entry__ as g; g.build()')")
        lib = ctypes.CDLL(_LIBPATH)
        P, i64, i32 = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int32
        lib.paris_summarize.argtypes = [P, i64, i32, i32, i32, P, P]
        lib.paris_summarize.restype = ctypes.c_int
        lib.paris_summarize_file.argtypes = [ctypes.c_char_p, i64, i64, i32, i32, i32, P, P, i32, P]
        lib.paris_summarize_file.restype = ctypes.c_int
        lib.paris_map_raw_file.argtypes = [ctypes.c_char_p, i64, i64, ctypes.POINTER(ctypes.c_void_p)]
        lib.paris_map_raw_file.restype = ctypes.c_int
        lib.paris_unmap_raw_file.argtypes = [P, i64]
        lib.paris_unmap_raw_file.restype = ctypes.c_int
        lib.paris_knn_exact.argtypes = [P, P, i64, P, i32, i32, P, P, i32, i32, i32, P]
        lib.paris_knn_exact.restype = ctypes.c_int
        lib.paris_knn_exact_ex.argtypes = [P, P, i64, P, i32, i32, P, P, i32, i32, i32, P,
                                           ctypes.POINTER(_Config), ctypes.POINTER(_Stats)]
        lib.paris_knn_exact_ex.restype = ctypes.c_int
        lib.paris_index_build.argtypes = [P, i64, i32, i32, P, P, P, P]
        lib.paris_index_build.restype = ctypes.c_int
        lib.paris_knn_index_ex.argtypes = [P, P, P, P, i64, P, i32, i32, P, P, i32, i32, i32, P,
                                           ctypes.POINTER(_Config), ctypes.POINTER(_Stats)]
        lib.paris_knn_index_ex.restype = ctypes.c_int
        lib.paris_knn_index_x.argtypes = [P, P, P, P, P, i64, P, i32, i32, P, P, i32, i32, i32, P,
                                          ctypes.POINTER(_Config), ctypes.POINTER(_Stats)]
        lib.paris_knn_index_x.restype = ctypes.c_int
        lib.paris_knn_index_aux.argtypes = [P, P, P, P, i64, P, i32, i32, P, P, i32, i32, i32, P,
                                            ctypes.POINTER(_Aux), ctypes.POINTER(_Config), ctypes.POINTER(_Stats)]
        lib.paris_knn_index_aux.restype = ctypes.c_int
        lib.paris_paa_f16.argtypes = [P, i64, i32, i32, P, P]
        lib.paris_paa_f16.restype = ctypes.c_int
        lib.paris_raw_bf16.argtypes = [P, i64, i32, P, P]
        lib.paris_raw_bf16.restype = ctypes.c_int
        lib.paris_knn_index.argtypes = [P, P, P, P, i64, P, i32, i32, P, P, i32, i32, i32, P]
        lib.paris_knn_index.restype = ctypes.c_int
        lib.paris_knn_approx.argtypes = [P, P, i64, P, i32, i32, P, P, i32, i32, i32, P, ctypes.POINTER(_Config)]
        lib.paris_knn_approx.restype = ctypes.c_int
        lib.paris_knn_index_approx.argtypes = [P, P, P, P, i64, P, i32, i32, P, P, i32, i32, i32, P,
                                               ctypes.POINTER(_Config)]
        lib.paris_knn_index_approx.restype = ctypes.c_int
        lib.paris_knn_nb.argtypes = [P, P, i64, P, i32, P, P, i32, i32, i32, P, ctypes.POINTER(_Config),
                                     ctypes.POINTER(_Stats)]
        lib.paris_knn_nb.restype = ctypes.c_int
        lib.paris_merge_topk.argtypes = [P, P, i32, i32, i32, P, P, P]
        lib.paris_merge_topk.restype = ctypes.c_int
        lib.paris_release_workspace.restype = None
        lib.paris_last_error.restype = ctypes.c_char_p
        lib.paris_version.restype = i32
        lib.paris_profile_enable.argtypes = [i32]
        lib.paris_profile_read.argtypes = [ctypes.POINTER(_KProf), i32]
        lib.paris_profile_read.restype = i32
        lib.paris_launch_count.restype = i64
        lib.paris_debug_cuts.argtypes = [i32, P]
        lib.paris_debug_cuts.restype = ctypes.c_int
        lib.paris_debug_read_probe.argtypes = [P, i64, P]
        lib.paris_debug_read_probe.restype = ctypes.c_int
        lib.paris_debug_hfma2_probe.argtypes = [i32, i32, P]
        lib.paris_debug_hfma2_probe.restype = ctypes.c_int
        lib.paris_debug_gf_mma.argtypes = [P, i64, P, P, P, i32, P]
        lib.paris_debug_gf_mma.restype = ctypes.c_int
        lib.paris_debug_set_variant.argtypes = [i32, i32]
        lib.paris_debug_set_variant.restype = i32
        lib.paris_debug_half_dir.argtypes = [ctypes.c_double, i32]
        lib.paris_debug_half_dir.restype = ctypes.c_uint16
        _lib = lib
        return lib


def symbols():
    """Function names declared in include/paris.h."""
    txt = open(_HEADER).read()
    txt = re.sub(r"/\*.*?\*/", "", txt, flags=re.S)
    return sorted(set(re.findall(r"\b(paris_\w+)\s*\(", txt)))


def last_error() -> str:
    return load().paris_last_error().decode()


def version() -> int:
    return int(load().paris_version())


def _check(rc: int):
    if rc != 0:
        raise ParisError(rc, last_error())


def _stream(stream):
    if stream is None:
        return ctypes.c_void_p(torch.cuda.current_stream().cuda_stream)
    if isinstance(stream, torch.cuda.Stream):
        return ctypes.c_void_p(stream.cuda_stream)
    return ctypes.c_void_p(int(stream))


def _need_cuda(t: torch.Tensor, name: str):
    if not t.is_cuda:
        raise ValueError(f"{name} must be a CUDA tensor (the index lives in HBM)")
    if not t.is_contiguous():
        raise ValueError(f"{name} must be contiguous")


def summarize(raw: torch.Tensor, w: int = 16, card: int = 256, out: torch.Tensor | None = None,
              stream=None) -> torch.Tensor:
    """PAA + iSAX of every row of raw ([n][len] fp32) -> uint8 [w][n] (segment-major, CUDA).

    raw may be a CUDA tensor or a host tensor (pinned or pageable): host rows are
    streamed to the device in double-buffered chunks; `out` is always
    device memory (the current CUDA device when not given).
    """
    lib = load()
    if not raw.is_contiguous():
        raise ValueError("raw must be contiguous")
    if raw.dtype != torch.float32 or raw.dim() != 2:
        raise ValueError("raw must be [n][len] float32")
    n, length = raw.shape
    if out is None:
        out = torch.empty((w, n), dtype=torch.uint8, device=raw.device if raw.is_cuda else "cuda")
    _need_cuda(out, "out")
    if out.dtype != torch.uint8 or out.numel() != n * w:
        raise ValueError("out must be uint8 with n*w elements")
    _check(lib.paris_summarize(raw.data_ptr(), n, length, w, card, out.data_ptr(), _stream(stream)))
    return out


def summarize_file(path: str, n: int, length: int, w: int = 16, card: int = 256, offset: int = 0,
                   out: torch.Tensor | None = None, bf16: bool = False, direct_io: bool = False, stream=None):
    """paris_summarize_file: PAA + iSAX of n rows of `length` fp32 stored in a file (from byte
    `offset`) -> uint8 [w][n] on the current CUDA device; with bf16=True also the [n][len]
    bf16 copy (paris_raw_bf16 of the same rows).  Returns sax, or (sax, raw16)."""
    lib = load()
    if out is None:
        out = torch.empty((w, n), dtype=torch.uint8, device="cuda")
    _need_cuda(out, "out")
    r16 = torch.empty((n, length), dtype=torch.int16, device=out.device) if bf16 else None
    _check(lib.paris_summarize_file(os.fsencode(path), int(offset), int(n), int(length), int(w), int(card),
                                    out.data_ptr(), r16.data_ptr() if bf16 else None, 1 if direct_io else 0,
                                    _stream(stream)))
    return (out, r16) if bf16 else out


class MappedRaw:
    """A raw file mapped read-only and registered with CUDA (paris_map_raw_file): `.tensor` is
    a [n][len] fp32 host tensor the k-NN calls accept as raw (pinned).  close() unmaps."""

    def __init__(self, path: str, n: int, length: int, offset: int = 0):
        lib = load()
        self.bytes = int(n) * int(length) * 4
        ptr = ctypes.c_void_p()
        _check(lib.paris_map_raw_file(os.fsencode(path), int(offset), self.bytes, ctypes.byref(ptr)))
        self.ptr = ptr.value
        buf = (ctypes.c_char * self.bytes).from_address(self.ptr)
        self.tensor = torch.frombuffer(buf, dtype=torch.float32).view(n, length)

    def close(self):
        if self.ptr:
            self.tensor = None
            load().paris_unmap_raw_file(self.ptr, self.bytes)
            self.ptr = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()


PARIS_INDEX_BLOCK = 64
PARIS_INDEX_TILE = 2048


@dataclass
class Index:
    """iSAX-ordered SAX array (paris_index_build): sorted SoA words, ids, block envelopes."""
    sax_sorted: torch.Tensor   # uint8 [ceil(n/2048)][w][2048] tile-major (include/paris.h)
    perm: torch.Tensor         # int32 [n] (uint32 ids)
    env: torch.Tensor          # uint8 [ceil(n/64)][2][w]
    w: int
    card: int


def index_build(sax: torch.Tensor, w: int = 16, card: int = 256, stream=None) -> Index:
    """Sort the SAX array by its iSAX key and compute block envelopes (CUDA)."""
    lib = load()
    _need_cuda(sax, "sax")
    if sax.dtype != torch.uint8 or sax.dim() != 2 or sax.shape[0] != w:
        raise ValueError("sax must be uint8 [w][n]")
    n = sax.shape[1]
    nblk = (n + PARIS_INDEX_BLOCK - 1) // PARIS_INDEX_BLOCK
    ntile = (n + PARIS_INDEX_TILE - 1) // PARIS_INDEX_TILE
    out = torch.zeros((ntile, w, PARIS_INDEX_TILE), dtype=torch.uint8, device=sax.device)
    perm = torch.empty(n, dtype=torch.int32, device=sax.device)
    env = torch.empty((nblk, 2, w), dtype=torch.uint8, device=sax.device)
    _check(lib.paris_index_build(sax.data_ptr(), n, w, card, out.data_ptr(), perm.data_ptr(), env.data_ptr(),
                                 _stream(stream)))
    return Index(out, perm, env, w, card)


def raw_bf16(raw: torch.Tensor, stream=None) -> torch.Tensor:
    """bf16 copy of raw ([n][len] fp32, CUDA) for the refinement pre-filter (paris_raw_bf16)."""
    lib = load()
    _need_cuda(raw, "raw")
    if raw.dtype != torch.float32 or raw.dim() != 2:
        raise ValueError("raw must be [n][len] float32")
    out = torch.empty(raw.shape, dtype=torch.int16, device=raw.device)  # bf16 bits
    _check(lib.paris_raw_bf16(raw.data_ptr(), raw.shape[0], raw.shape[1], out.data_ptr(), _stream(stream)))
    return out


def paa_f16(raw: torch.Tensor, w2: int = 64, stream=None) -> torch.Tensor:
    """fp16 PAA of every row of raw at w2 segments (paris_paa_f16) -> int16 bits [n][w2] (CUDA):
    the PAA refinement pre-filter of knn_index(..., paa16=...)."""
    lib = load()
    _need_cuda(raw, "raw")
    if raw.dtype != torch.float32 or raw.dim() != 2:
        raise ValueError("raw must be [n][len] float32")
    out = torch.empty((raw.shape[0], w2), dtype=torch.int16, device=raw.device)
    _check(lib.paris_paa_f16(raw.data_ptr(), raw.shape[0], raw.shape[1], w2, out.data_ptr(), _stream(stream)))
    return out


def knn_index(raw: torch.Tensor, index: Index, queries: torch.Tensor, k: int = 1,
              out_idx: torch.Tensor | None = None, out_dist: torch.Tensor | None = None, stream=None,
              config: KnnConfig | None = None, stats: bool = False, raw16: torch.Tensor | None = None,
              sync: bool | None = None, paa16: torch.Tensor | None = None):
    """Exact k-NN over an Index (paris_knn_index); same results as knn_exact.  Refinement
    pre-filters: raw16 = the bf16 copy of raw (raw_bf16, paris_knn_index_x); paa16 = the fp16
    PAA of raw (paa_f16, paris_knn_index_aux)."""
    return knn_exact(raw, index.sax_sorted, queries, k=k, w=index.w, card=index.card, out_idx=out_idx,
                     out_dist=out_dist, stream=stream, config=config, stats=stats, _index=index, _raw16=raw16,
                     sync=sync, _paa16=paa16)


def knn_nb(raw: torch.Tensor, sax: torch.Tensor, queries: torch.Tensor, w: int = 16, card: int = 256,
           out_idx: torch.Tensor | None = None, out_dist: torch.Tensor | None = None, stream=None,
           config: KnnConfig | None = None, stats: bool = False, sync: bool | None = None):
    """Exact 1-NN with nb-ParIS+ (paris_knn_nb): per-worker BSF copies, fused LB -> refine."""
    return knn_exact(raw, sax, queries, k=1, w=w, card=card, out_idx=out_idx, out_dist=out_dist, stream=stream,
                     config=config, stats=stats, _nb=True, sync=sync)


def _make_config(config, nq: int):
    if config is None:
        return None
    cfg = _Config(config.batch, config.seed_div, config.wave_a)
    cfg.reserved[0] = 1 if config.force_direct else 0
    cfg.reserved[1] = 1 if config.sorted_refine else 0
    cfg.reserved[2] = int(config.index_seeds)
    cfg.reserved[3] = 1 if config.seed_from_out else 0
    cfg.reserved[4] = int(config.cap)
    if config.tau_in is not None:
        t = config.tau_in
        if not (t.is_cuda and t.dtype == torch.float32 and t.is_contiguous() and t.numel() == nq):
            raise ValueError("tau_in must be a contiguous float32 CUDA tensor of nq entries")
        cfg.tau_in = t.data_ptr()
    return cfg


def knn_approx(raw: torch.Tensor, sax, queries: torch.Tensor, k: int = 1, w: int = 16, card: int = 256,
               index: Index | None = None, config: KnnConfig | None = None, stream=None):
    """Approximate k-NN (paris_knn_approx / paris_knn_index_approx): the k best
    seed series per query with their true distances; `sax` is the flat SAX array, or pass
    `index` (then sax may be None).  Returns (idx int64 [nq][k], dist float32 [nq][k]) on
    the device of `queries` (CUDA)."""
    lib = load()
    if queries.dim() == 1:
        queries = queries.unsqueeze(0)
    queries = queries.contiguous()
    n, length = raw.shape
    nq = queries.shape[0]
    out_idx = torch.empty((nq, k), dtype=torch.int64, device=queries.device)
    out_dist = torch.empty((nq, k), dtype=torch.float32, device=queries.device)
    cfg = _make_config(config, nq)
    if index is not None:
        rc = lib.paris_knn_index_approx(raw.data_ptr(), index.sax_sorted.data_ptr(), index.perm.data_ptr(),
                                        index.env.data_ptr(), n, queries.data_ptr(), nq, k, out_idx.data_ptr(),
                                        out_dist.data_ptr(), length, index.w, index.card, _stream(stream),
                                        ctypes.byref(cfg) if cfg else None)
    else:
        _need_cuda(sax, "sax")
        rc = lib.paris_knn_approx(raw.data_ptr(), sax.data_ptr(), n, queries.data_ptr(), nq, k, out_idx.data_ptr(),
                                  out_dist.data_ptr(), length, w, card, _stream(stream),
                                  ctypes.byref(cfg) if cfg else None)
    _check(rc)
    return out_idx, out_dist


def knn_exact(raw: torch.Tensor, sax: torch.Tensor, queries: torch.Tensor, k: int = 1,
              w: int = 16, card: int = 256, out_idx: torch.Tensor | None = None,
              out_dist: torch.Tensor | None = None, stream=None,
              config: KnnConfig | None = None, stats: bool = False, _index: Index | None = None,
              _nb: bool = False, _raw16: torch.Tensor | None = None, sync: bool | None = None,
              _paa16: torch.Tensor | None = None):
    """Exact k-NN of every query (rows of `queries`, CUDA or host) over raw/sax.

    sax (and the index) are CUDA tensors; raw is CUDA or pinned host memory (the
    candidates' rows are then read through the host mapping).

    Returns (idx int64 [nq][k], dist float32 [nq][k]) on the device of `queries`
    (or the given out tensors); with stats=True also a dict of per-query counters.
    The library call is asynchronous on the stream; with host outputs the binding waits
    for the stream before returning unless sync=False (then the caller synchronizes).
    """
    lib = load()
    if not (raw.is_cuda or raw.is_pinned()):
        raise ValueError("raw must be a CUDA tensor or a pinned host tensor (SURVEY f3)")
    if not raw.is_contiguous():
        raise ValueError("raw must be contiguous")
    _need_cuda(sax, "sax")
    if not queries.is_contiguous():
        queries = queries.contiguous()
    if queries.dtype != torch.float32:
        raise ValueError("queries must be float32")
    if queries.dim() == 1:
        queries = queries.unsqueeze(0)
    n, length = raw.shape
    nq = queries.shape[0]
    if queries.shape[1] != length:
        raise ValueError("query length differs from series length")
    if _index is None and (sax.dtype != torch.uint8 or sax.numel() != n * w):
        raise ValueError("sax must be uint8 [w][n]")
    dev = queries.device
    pin = (not queries.is_cuda) and torch.cuda.is_available()
    if out_idx is None:
        out_idx = torch.empty((nq, k), dtype=torch.int64, device=dev, pin_memory=pin)
    if out_dist is None:
        out_dist = torch.empty((nq, k), dtype=torch.float32, device=dev, pin_memory=pin)
    cfg = _make_config(config, nq)
    st = None
    arrays = None
    if stats:
        arrays = (torch.zeros(nq, dtype=torch.int64), torch.zeros(nq, dtype=torch.int64),
                  torch.zeros(nq, dtype=torch.float32), torch.zeros(nq, dtype=torch.int64),
                  torch.zeros(nq, dtype=torch.int64), torch.zeros(nq, dtype=torch.int64),
                  torch.zeros(nq, dtype=torch.int64))
        st = _Stats(arrays[0].data_ptr(), arrays[1].data_ptr(), arrays[2].data_ptr(), arrays[3].data_ptr(),
                    arrays[4].data_ptr(), arrays[5].data_ptr(), arrays[6].data_ptr())
    if _nb:
        if k != 1:
            raise ValueError("knn_nb answers 1-NN (nb-ParIS+, Alg7-8)")
        rc = lib.paris_knn_nb(raw.data_ptr(), sax.data_ptr(), n, queries.data_ptr(), nq, out_idx.data_ptr(),
                              out_dist.data_ptr(), length, w, card, _stream(stream),
                              ctypes.byref(cfg) if cfg else None, ctypes.byref(st) if st else None)
    elif _index is None:
        rc = lib.paris_knn_exact_ex(raw.data_ptr(), sax.data_ptr(), n, queries.data_ptr(), nq, k,
                                    out_idx.data_ptr(), out_dist.data_ptr(), length, w, card,
                                    _stream(stream), ctypes.byref(cfg) if cfg else None,
                                    ctypes.byref(st) if st else None)
    elif _paa16 is not None:
        _need_cuda(_paa16, "paa16")
        if _paa16.dim() != 2 or _paa16.shape[0] != n or _paa16.element_size() != 2:
            raise ValueError("paa16 must be the [n][w2] 16-bit PAA of raw (paa_f16)")
        if _raw16 is not None:
            _need_cuda(_raw16, "raw16")
        aux = _Aux(_raw16.data_ptr() if _raw16 is not None else None, _paa16.data_ptr(), int(_paa16.shape[1]), 0)
        rc = lib.paris_knn_index_aux(raw.data_ptr(), sax.data_ptr(), _index.perm.data_ptr(), _index.env.data_ptr(), n,
                                     queries.data_ptr(), nq, k, out_idx.data_ptr(), out_dist.data_ptr(), length, w,
                                     card, _stream(stream), ctypes.byref(aux), ctypes.byref(cfg) if cfg else None,
                                     ctypes.byref(st) if st else None)
    elif _raw16 is not None:
        _need_cuda(_raw16, "raw16")
        if _raw16.shape != raw.shape or _raw16.element_size() != 2:
            raise ValueError("raw16 must be the [n][len] 16-bit copy of raw (raw_bf16)")
        rc = lib.paris_knn_index_x(raw.data_ptr(), _raw16.data_ptr(), sax.data_ptr(), _index.perm.data_ptr(),
                                   _index.env.data_ptr(), n, queries.data_ptr(), nq, k, out_idx.data_ptr(),
                                   out_dist.data_ptr(), length, w, card, _stream(stream),
                                   ctypes.byref(cfg) if cfg else None, ctypes.byref(st) if st else None)
    else:
        rc = lib.paris_knn_index_ex(raw.data_ptr(), sax.data_ptr(), _index.perm.data_ptr(), _index.env.data_ptr(),
                                    n, queries.data_ptr(), nq, k, out_idx.data_ptr(), out_dist.data_ptr(),
                                    length, w, card, _stream(stream), ctypes.byref(cfg) if cfg else None,
                                    ctypes.byref(st) if st else None)
    _check(rc)
    if sync is None:
        sync = not (out_idx.is_cuda and out_dist.is_cuda)
    if sync:
        if stream is None:
            torch.cuda.current_stream().synchronize()
        elif isinstance(stream, torch.cuda.Stream):
            stream.synchronize()
        else:
            torch.cuda.ExternalStream(int(stream)).synchronize()
    if stats:
        return out_idx, out_dist, {"candidates": arrays[0], "refined": arrays[1],
                                   "tau_seed": arrays[2], "lb_blocks": arrays[3], "bsf_updates": arrays[4],
                                   "raw16_rows": arrays[5], "paa_rows": arrays[6]}
    return out_idx, out_dist


def release_workspace():
    """Free the library's cached k-NN workspace (paris_release_workspace; synchronizes)."""
    load().paris_release_workspace()


def merge_topk(dist: torch.Tensor, idx: torch.Tensor, stream=None):
    """Merge gathered per-shard rows dist/idx [R][nq][k] into the global [nq][k] (CUDA)."""
    lib = load()
    _need_cuda(dist, "dist")
    _need_cuda(idx, "idx")
    if dist.dtype != torch.float32 or idx.dtype != torch.int64 or dist.shape != idx.shape or dist.dim() != 3:
        raise ValueError("dist float32 / idx int64, both [R][nq][k]")
    R, nq, k = dist.shape
    out_idx = torch.empty((nq, k), dtype=torch.int64, device=dist.device)
    out_dist = torch.empty((nq, k), dtype=torch.float32, device=dist.device)
    _check(lib.paris_merge_topk(dist.data_ptr(), idx.data_ptr(), R, nq, k, out_idx.data_ptr(), out_dist.data_ptr(),
                                _stream(stream)))
    return out_idx, out_dist


def profile_enable(on: bool = True):
    load().paris_profile_enable(1 if on else 0)


def profile_reset():
    load().paris_profile_reset()


def profile_read() -> dict:
    """{kernel name: (launches, total device ms)} since the last reset (synchronizes)."""
    lib = load()
    n = lib.paris_profile_read(None, 0)
    buf = (_KProf * max(1, n))()
    n = lib.paris_profile_read(buf, n)
    return {buf[i].name.decode(): (int(buf[i].launches), float(buf[i].total_ms)) for i in range(n)}


def launch_count() -> int:
    return int(load().paris_launch_count())


def debug_read_probe(t: torch.Tensor, stream=None):
    """Stream the bytes of a CUDA tensor with read-only loads (the read-only HBM peak probe)."""
    _need_cuda(t, "t")
    _check(load().paris_debug_read_probe(t.data_ptr(), t.numel() * t.element_size() // 16 * 16, _stream(stream)))


def debug_hfma2_probe(iters: int, blocks_per_sm: int = 4, stream=None) -> float:
    """Launch the fp16x2 FMA probe; returns the fp16 FMAs it performs (time it with events)."""
    _check(load().paris_debug_hfma2_probe(int(iters), int(blocks_per_sm), _stream(stream)))
    import torch as _t
    sms = _t.cuda.get_device_properties(_t.cuda.current_device()).multi_processor_count
    return float(sms) * blocks_per_sm * 512 * iters * 8 * 2


def debug_gf_mma(sax_sorted, n: int, tabw, bmat, swap_desc: int = 0, stream=None):
    """paris_debug_gf_mma: the tensor-core filter's raw accumulators, [n, 64] fp32 (device)."""
    import torch as _t
    out = _t.empty((int(n), 64), dtype=_t.float32, device=sax_sorted.device)
    _check(load().paris_debug_gf_mma(sax_sorted.data_ptr(), int(n), tabw.data_ptr(), bmat.data_ptr(), out.data_ptr(),
                                     int(swap_desc), _stream(stream)))
    return out


def debug_set_variant(key: int, value: int) -> int:
    """Tuning hook (paris_debug_set_variant): A/B of kernel variants, identical results."""
    return int(load().paris_debug_set_variant(int(key), int(value)))


def debug_half_dir(v: float, direction: int) -> int:
    """IEEE binary16 bits of v rounded down (direction < 0) or up (> 0) -- for tests."""
    return int(load().paris_debug_half_dir(float(v), int(direction)))


def debug_cuts(card: int):
    """The library's own N(0,1) breakpoints (fp64) -- for tests."""
    import numpy as np
    out = np.zeros(256, dtype=np.float64)
    _check(load().paris_debug_cuts(card, out.ctypes.data))
    return out[: card - 1].copy()
