"""Parity at BASELINE.json's full sizes, in bench.py's launch configuration (index path with
32 queries per SAX pass, flat path with 16), on sampled queries the CPU oracle answers one by
one: the oracle's LB-pruned exact scan (itself pinned to brute force) over the full collection.

All five configs at full size (C4: 102.4 GB of raw copied to the host; the GPU boxes have
~196 GB of RAM); the oracle's SAX is computed by the oracle (independent of the CUDA
summarize).  C1-C3 and C5 check 5 sampled queries (+ k = 10 on two), C4 checks 3."""
import numpy as np
import pytest

import datagen
import oracle
from tests._parity import check_knn

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__ as ge
    ge.build()
    import paper_2009_00166_b200 as p
    return p


def _workload(config, nq):
    import torch
    from datagen import gpu as dg
    ds, qs = datagen.config_seeds(config)
    n, length = {1: (100_000, 256), 2: (1_000_000, 256), 3: (10_000_000, 128), 4: (100_000_000, 256),
                 5: (20_000_000, 256)}[config]
    raw = dg.walks(n, length, ds, device="cuda")
    if config in (2, 5):
        q, _ = dg.noisy_members(raw, nq, 0.05 if config == 2 else 0.2, qs)
    else:
        q = dg.walks(nq, length, qs, device="cuda")
    return raw, q


@pytest.mark.timeout(1200)  # C4: 102 GB to the host + the oracle's own summarize of 1e8 series (~4.5 min)
@pytest.mark.parametrize("config", [1, 2, 3, 5, 4])
def test_full_size_sampled_parity(P, config):
    import psutil
    import torch
    n_bytes = {1: 1e5 * 256, 2: 1e6 * 256, 3: 1e7 * 128, 4: 1e8 * 256, 5: 2e7 * 256}[config] * 4
    if psutil.virtual_memory().available < 1.3 * n_bytes:
        pytest.skip("host RAM too small for the oracle's copy of this config")
    nq = 40                                   # two index passes (32 + 8), three flat passes
    raw, q = _workload(config, nq)
    sax = P.summarize(raw, 16, 256)
    idx = P.index_build(sax, 16, 256)
    gi_i, gd_i = P.knn_index(raw, idx, q, k=1)
    gi_f, gd_f = P.knn_exact(raw, sax, q, k=1)
    k10_i, k10_d = P.knn_index(raw, idx, q[:5], k=10)
    del idx, sax
    torch.cuda.empty_cache()
    x = raw.cpu().numpy()
    del raw
    qh = q.cpu().numpy()
    sample = np.arange(0, nq, 8) if config != 4 else np.array([0, 17, 39])  # spread over the passes
    sax_o = oracle.summarize(x, 16, 256)      # the oracle's own SAX
    ri, rd2 = oracle.knn_pruned(x, sax_o, qh[sample], 1, 16, 256)
    check_knn(x, qh[sample], gi_i.cpu().numpy()[sample], gd_i.cpu().numpy()[sample], ri, rd2)
    check_knn(x, qh[sample], gi_f.cpu().numpy()[sample], gd_f.cpu().numpy()[sample], ri, rd2)
    if config != 4:
        ri10, rd10 = oracle.knn_pruned(x, sax_o, qh[:2], 10, 16, 256)
        check_knn(x, qh[:2], k10_i.cpu().numpy()[:2], k10_d.cpu().numpy()[:2], ri10, rd10)
    # every returned distance is the true distance of the returned id (all rows)
    for r in range(nq):
        assert abs(np.sqrt(oracle.ed2(x[gi_i[r, 0].item()], qh[r])) - gd_i[r, 0].item()) <= 1e-5 * max(1.0, gd_i[r, 0].item())
