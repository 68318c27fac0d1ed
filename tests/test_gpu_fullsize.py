"""Parity at BASELINE.json's full sizes, in bench.py's launch configuration, on sampled queries
the CPU oracle answers one by one: the oracle's LB-pruned exact scan (itself pinned to brute
force) over the full collection, on the oracle's own SAX (independent of the CUDA summarize).

* C4 (1e8 x 256): exactly the bench's default call (and the flat path's: 100 queries through the tensor-core filter) -- ``knn_index(..., raw16=raw_bf16(raw),
  paa16=paa_f16(raw, 64))``, k = 1, all 100 queries in ONE call (a 64-query pass and a 36-query
  pass, the PAA and bf16 refinement pre-filters, the 2048-series leaf seed) -- queries sampled
  from both passes; the flat path too.
* C5 (2e7 x 256): the query-hardness sweep's k = 100 mode at sigma = 0.2 and sigma = 0.01
  (bench.py's query sets), index path with the bf16 copy passed as the bench does, and flat.
* C3 (1e7 x 128): calls of 64 queries (BASELINE config 3), two calls, queries from both.
* C1, C2: one call of all queries, k = 1 and k = 10.

The C4 host copy is 102.4 GB (each test is skipped when the host RAM is too small)."""
import numpy as np
import pytest

import datagen
import oracle
from tests._parity import check_knn

pytestmark = pytest.mark.gpu

SHAPES = {1: (100_000, 256), 2: (1_000_000, 256), 3: (10_000_000, 128), 4: (100_000_000, 256),
          5: (20_000_000, 256)}


@pytest.fixture(scope="module")
def P():
    import __graft_entry__ as ge
    ge.build()
    import paper_2009_00166_b200 as p
    return p


def _need_ram(config):
    import psutil
    n, length = SHAPES[config]
    if psutil.virtual_memory().available < 1.3 * n * length * 4:
        pytest.skip("host RAM too small for the oracle's copy of this config")


def _raw(config):
    from datagen import gpu as dg
    ds, qs = datagen.config_seeds(config)
    n, length = SHAPES[config]
    return dg.walks(n, length, ds, device="cuda"), qs


def _oracle_rows(x, sax_o, qh, rows, k):
    return oracle.knn_pruned(x, sax_o, qh[rows], k, 16, 256)


def _true_dist_rows(x, qh, gi, gd, rows):
    """Every returned distance is the true distance of the returned id."""
    for r in rows:
        for j in range(gi.shape[1]):
            d = np.sqrt(oracle.ed2(x[gi[r, j]], qh[r]))
            assert abs(d - gd[r, j]) <= 1e-5 * max(1.0, gd[r, j]), (r, j, d, gd[r, j])


@pytest.mark.timeout(1800)  # 102 GB to the host + the oracle's own summarize of 1e8 series (~4.5 min)
def test_c4_bench_call_parity(P):
    """C4, the bench's exact default call: index path + bf16 pre-filter, 100 queries in one call."""
    import torch
    _need_ram(4)
    from datagen import gpu as dg
    raw, qs = _raw(4)
    nq = 100
    q = dg.walks(nq, 256, qs, device="cuda")           # bench.py: fresh random walks, query seed
    sax = P.summarize(raw, 16, 256)
    idx = P.index_build(sax, 16, 256)
    raw16 = P.raw_bf16(raw)
    paa16 = P.paa_f16(raw, 64)
    gi, gd, st = P.knn_index(raw, idx, q, k=1, raw16=raw16, paa16=paa16, stats=True)    # one call: 64 + 36
    assert st["paa_rows"].sum() > 0, "the PAA pre-filter did not run"
    del raw16, paa16, idx
    gi_f, gd_f = P.knn_exact(raw, sax, q, k=1)          # flat path, the bench's call: 64 + 36 slots through k_gf
    del sax
    torch.cuda.empty_cache()
    x = raw.cpu().numpy()
    del raw
    qh = q.cpu().numpy()
    gi, gd, gi_f, gd_f = gi.cpu().numpy(), gd.cpu().numpy(), gi_f.cpu().numpy(), gd_f.cpu().numpy()
    sample = np.array([0, 31, 63, 64, 81, 99])      # first pass: 0..63, second: 64..99
    sax_o = oracle.summarize(x, 16, 256)
    ri, rd2 = _oracle_rows(x, sax_o, qh, sample, 1)
    check_knn(x, qh[sample], gi[sample], gd[sample], ri, rd2)
    check_knn(x, qh[sample], gi_f[sample], gd_f[sample], ri, rd2)
    _true_dist_rows(x, qh, gi, gd, range(nq))
    # both paths are exact: same distances on every row (ids may differ only under ties)
    assert np.allclose(gd_f, gd, rtol=1e-6, atol=0), "flat (k_gf) and index paths disagree"
    assert (gi_f == gi).mean() >= 0.99


@pytest.mark.timeout(1500)
def test_c5_k100_hardness_parity(P):
    """C5, k = 100 at sigma = 0.2 (hard: ~5e5 candidates per query) and sigma = 0.01 (easy),
    the bench's query sets (query seed + 101 * (set + 1)), index path with the bf16 copy
    passed as bench.py passes it, and the flat path."""
    import torch
    _need_ram(5)
    from datagen import gpu as dg
    raw, qs = _raw(5)
    sax = P.summarize(raw, 16, 256)
    idx = P.index_build(sax, 16, 256)
    raw16 = P.raw_bf16(raw)
    sets = {}
    paa16 = P.paa_f16(raw, 64)
    for si, sig in ((0, 0.01), (4, 0.2)):
        q, _ = dg.noisy_members(raw, 200, sig, qs + 101 * (si + 1))
        gi, gd = P.knn_index(raw, idx, q, k=100, raw16=raw16, paa16=paa16)   # all 200: 4 passes
        fi, fd = P.knn_exact(raw, sax, q[:2], k=100)
        sets[sig] = (q.cpu().numpy(), gi.cpu().numpy(), gd.cpu().numpy(), fi.cpu().numpy(), fd.cpu().numpy())
    del raw16, paa16, idx, sax
    torch.cuda.empty_cache()
    x = raw.cpu().numpy()
    del raw
    sax_o = oracle.summarize(x, 16, 256)
    for sig, (qh, gi, gd, fi, fd) in sets.items():
        rows = np.array([0, 1, 130])                 # passes 1 and 3
        ri, rd2 = _oracle_rows(x, sax_o, qh, rows, 100)
        check_knn(x, qh[rows], gi[rows], gd[rows], ri, rd2)
        check_knn(x, qh[:2], fi[:2], fd[:2], ri[:2], rd2[:2])
        _true_dist_rows(x, qh, gi, gd, [2, 199])


@pytest.mark.timeout(1200)
def test_c3_calls_of_64_parity(P):
    """C3: queries processed in calls of 64 (BASELINE config 3), two calls checked."""
    import torch
    _need_ram(3)
    from datagen import gpu as dg
    raw, qs = _raw(3)
    q = dg.walks(128, 128, qs, device="cuda")
    sax = P.summarize(raw, 16, 256)
    idx = P.index_build(sax, 16, 256)
    raw16 = P.raw_bf16(raw)
    paa16 = P.paa_f16(raw, 32)                       # bench.py's default at len 128
    out = [P.knn_index(raw, idx, q[c:c + 64], k=1, raw16=raw16, paa16=paa16) for c in (0, 64)]
    fl = [P.knn_exact(raw, sax, q[c:c + 64], k=1) for c in (0, 64)]
    gi = torch.cat([o[0] for o in out]).cpu().numpy()
    gd = torch.cat([o[1] for o in out]).cpu().numpy()
    fi = torch.cat([o[0] for o in fl]).cpu().numpy()
    fd = torch.cat([o[1] for o in fl]).cpu().numpy()
    del raw16, paa16, idx, sax
    torch.cuda.empty_cache()
    x = raw.cpu().numpy()
    del raw
    qh = q.cpu().numpy()
    rows = np.array([0, 40, 63, 64, 100, 127])
    sax_o = oracle.summarize(x, 16, 256)
    ri, rd2 = _oracle_rows(x, sax_o, qh, rows, 1)
    check_knn(x, qh[rows], gi[rows], gd[rows], ri, rd2)
    check_knn(x, qh[rows], fi[rows], fd[rows], ri, rd2)


@pytest.mark.timeout(900)
@pytest.mark.parametrize("config", [1, 2])
def test_c1_c2_parity(P, config):
    """C1 (fresh queries) and C2 (member + N(0, 0.05^2) queries): one call of all queries,
    k = 1 (index + bf16, and flat) and k = 10 (index)."""
    import torch
    _need_ram(config)
    from datagen import gpu as dg
    raw, qs = _raw(config)
    nq = 100 if config == 1 else 1000
    if config == 2:
        q, _ = dg.noisy_members(raw, nq, 0.05, qs)
    else:
        q = dg.walks(nq, 256, qs, device="cuda")
    sax = P.summarize(raw, 16, 256)
    idx = P.index_build(sax, 16, 256)
    raw16 = P.raw_bf16(raw)
    paa16 = P.paa_f16(raw, 64)
    gi, gd = P.knn_index(raw, idx, q, k=1, raw16=raw16, paa16=paa16)
    fi, fd = P.knn_exact(raw, sax, q, k=1)
    ti, td = P.knn_index(raw, idx, q, k=10, paa16=paa16)
    x = raw.cpu().numpy()
    qh = q.cpu().numpy()
    rows = np.arange(0, nq, nq // 10)
    sax_o = oracle.summarize(x, 16, 256)
    ri, rd2 = _oracle_rows(x, sax_o, qh, rows, 1)
    check_knn(x, qh[rows], gi.cpu().numpy()[rows], gd.cpu().numpy()[rows], ri, rd2)
    check_knn(x, qh[rows], fi.cpu().numpy()[rows], fd.cpu().numpy()[rows], ri, rd2)
    r10, d10 = _oracle_rows(x, sax_o, qh, rows[:3], 10)
    check_knn(x, qh[rows[:3]], ti.cpu().numpy()[rows[:3]], td.cpu().numpy()[rows[:3]], r10, d10)
