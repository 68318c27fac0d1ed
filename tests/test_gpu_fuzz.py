"""Randomized parity sweep of the CUDA path (through the C ABI) against the oracle:
seeded random shapes, cardinalities, k, batch sizes and paths (flat, flat with the
bucket-sorted refine, index, index with the bf16 pre-filter, index with raw in pinned
host memory, nb), plus the k > 1 selection's tie fallback (thousands of exact
duplicates, so the distance window cannot be narrowed below the sort buffer)."""
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


def _case(seed):
    rng = np.random.default_rng(seed)
    length = int(rng.choice([64, 128, 256]))
    n = int(rng.integers(1, 2500)) * 16
    nq = int(rng.integers(1, 90))
    k = int(rng.choice([1, 1, 2, 7, 33]))
    k = min(k, n)
    card = int(rng.choice([16, 64, 256]))
    path = str(rng.choice(["flat", "index", "index16", "nb", "host", "sorted"]))
    batch = int(rng.choice([0, 1, 5, 16, 33]))
    return dict(seed=seed, length=length, n=n, nq=nq, k=k, card=card, path=path, batch=batch)


@pytest.mark.parametrize("seed", list(range(60)))
def test_random_parity(P, seed):
    import torch
    c = _case(1000 + seed)
    if c["path"] == "nb" and c["k"] != 1:
        c["path"] = "flat"
    x = datagen.random_walks(c["n"], c["length"], 2000 + seed)
    q = datagen.random_walks(c["nq"], c["length"], 3000 + seed)
    if c["nq"] > 3:
        q[:2] = x[[0, c["n"] - 1]]
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, c["card"])
    cfg = P.KnnConfig(batch=c["batch"], sorted_refine=c["path"] == "sorted")
    if c["path"] in ("flat", "sorted"):
        gi, gd = P.knn_exact(xd, sax, qd, k=c["k"], card=c["card"], config=cfg)
    elif c["path"] == "host":  # raw in pinned host memory, index path with the bf16 copy in HBM
        idx = P.index_build(sax, 16, c["card"])
        gi, gd = P.knn_index(torch.from_numpy(x).pin_memory(), idx, qd, k=c["k"], config=cfg,
                             raw16=P.raw_bf16(xd))
    elif c["path"] == "nb":
        gi, gd = P.knn_nb(xd, sax, qd, card=c["card"], config=cfg)
    else:
        idx = P.index_build(sax, 16, c["card"])
        r16 = P.raw_bf16(xd) if c["path"] == "index16" else None
        gi, gd = P.knn_index(xd, idx, qd, k=c["k"], config=cfg, raw16=r16)
    ri, rd2 = oracle.knn_bruteforce(x, q, c["k"])
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)


@pytest.mark.parametrize("path", ["flat", "index"])
def test_k_select_tie_fallback(P, path):
    """5000 exact copies of one series and a query equal to it: the k = 100 results are the
    100 lowest ids among the copies (ties -> lower id), whatever the selection path."""
    import torch
    n, length = 20_000, 256
    x = datagen.random_walks(n, length, 4242)
    dup = np.arange(3, n, 4)[:5000]
    x[dup] = x[1]
    q = np.stack([x[1], datagen.random_walks(1, length, 4343)[0]])
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    qd = torch.from_numpy(q).cuda()
    if path == "flat":
        gi, gd = P.knn_exact(xd, sax, qd, k=100)
    else:
        gi, gd = P.knn_index(xd, P.index_build(sax, 16, 256), qd, k=100)
    expect = np.sort(np.r_[1, dup])[:100]
    np.testing.assert_array_equal(gi[0].cpu().numpy(), expect)
    assert float(gd[0].max()) == 0.0
    ri, rd2 = oracle.knn_bruteforce(x, q, 100)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
