"""f4: paris_merge_topk (the exact merge of per-shard k-NN rows) vs a numpy definition, and
the sharded search run as shards in one process against the oracle."""
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


@pytest.mark.parametrize("R,nq,k", [(1, 3, 1), (2, 5, 10), (8, 7, 100), (3, 4, 1024)])
def test_merge_matches_definition(P, R, nq, k):
    import torch
    rng = np.random.default_rng(R * 1000 + k)
    d = np.sort(rng.integers(0, 50, (R, nq, k)).astype(np.float32) / 7.0, axis=2)   # many ties
    i = rng.permutation(R * nq * k * 3)[: R * nq * k].reshape(R, nq, k).astype(np.int64)
    i[:, :, -1] = np.where(rng.random((R, nq)) < 0.3, -1, i[:, :, -1])              # some empty slots
    d[:, :, -1] = np.where(i[:, :, -1] < 0, np.inf, d[:, :, -1])
    gi, gd = P.merge_topk(torch.from_numpy(d).cuda(), torch.from_numpy(i).cuda())
    for q in range(nq):
        dd = d[:, q, :].reshape(-1).astype(np.float64)
        ii = i[:, q, :].reshape(-1)
        dd = np.where(ii < 0, np.inf, dd)
        order = np.lexsort((ii.astype(np.uint64), dd))[:k]
        np.testing.assert_array_equal(gi[q].cpu().numpy(), ii[order])
        np.testing.assert_array_equal(gd[q].cpu().numpy(), dd[order].astype(np.float32))


@pytest.mark.parametrize("path", ["index", "flat"])
def test_sharded_search_in_one_process(P, path):
    """Shards searched one after another, rows merged by paris_merge_topk == oracle on the whole."""
    import torch
    from paper_2009_00166_b200 import parallel as par
    n, k = 50_000 + 16 * 7, 10
    x = datagen.random_walks(n, 256, 5)
    q = datagen.random_walks(6, 256, 6)
    q[0] = x[n - 3]
    qd = torch.from_numpy(q).cuda()
    rows_i, rows_d = [], []
    for r in range(3):
        lo, hi = par.shard_range(n, r, 3)
        xs = torch.from_numpy(x[lo:hi]).cuda()
        sax = P.summarize(xs, 16, 256)
        local = (par.local_index_search(xs, P.index_build(sax, 16, 256)) if path == "index"
                 else par.local_flat_search(xs, sax))
        li, ld = local(qd, k)
        rows_i.append(torch.where(li >= 0, li + lo, li))
        rows_d.append(ld)
    gi, gd = P.merge_topk(torch.stack(rows_d), torch.stack(rows_i))
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert gi[0, 0].item() == n - 3
