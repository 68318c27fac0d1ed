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


@pytest.mark.parametrize("k,raw16", [(1, True), (1, False), (10, False)])
def test_sharded_search_with_tau_exchange(P, k, raw16):
    """The tau_seed exchange of SURVEY §8(e) in one process: every shard's approximate answer
    (paris_knn_index_approx) bounds the global k-th distance; the minimum over shards is
    passed to every shard's exact search (config.tau_in) -- shards whose series all lie
    beyond it return empty rows -- and the merged rows equal the oracle on the whole."""
    import torch
    from paper_2009_00166_b200 import parallel as par
    n, R = 60_000 + 16 * 3, 3
    x = datagen.random_walks(n, 256, 15)
    q = datagen.random_walks(7, 256, 16)
    q[0] = x[n - 5]        # a member of the last shard: the others must come back empty or beyond it
    q[3] = x[100] * 0.999
    qd = torch.from_numpy(q).cuda()
    shards = []
    for r in range(R):
        lo, hi = par.shard_range(n, r, R)
        xs = torch.from_numpy(x[lo:hi]).cuda()
        sax = P.summarize(xs, 16, 256)
        idx = P.index_build(sax, 16, 256)
        shards.append((lo, xs, idx, P.raw_bf16(xs) if raw16 else None))
    taus = torch.stack([par.approx_index_search(xs, idx)(qd, k) for _, xs, idx, _ in shards])
    # an approximate answer is k real series: its k-th distance bounds the true k-th distance
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    assert (taus.cpu().numpy() >= np.sqrt(rd2[:, k - 1])[None, :] * (1 - 1e-6)).all()
    tau = taus.min(dim=0).values.contiguous()
    rows_i, rows_d = [], []
    for lo, xs, idx, r16 in shards:
        li, ld = par.local_index_search(xs, idx, raw16=r16)(qd, k, tau)
        rows_i.append(torch.where(li >= 0, li + lo, li))
        rows_d.append(ld)
    gi, gd = P.merge_topk(torch.stack(rows_d), torch.stack(rows_i))
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert gi[0, 0].item() == n - 5
    if k == 1:
        assert (rows_i[0][0] < 0).all()   # shard 0 holds nothing within the member query's bound (0)


def test_approx_rows_are_true_distances(P):
    """paris_knn_approx / paris_knn_index_approx: ascending rows of real series with their
    true distances (flat: the LB-best seeds of a prefix sample; index: the query's leaf)."""
    import torch
    n, k = 30_000 + 16, 5
    x = datagen.random_walks(n, 128, 25)
    q = datagen.random_walks(4, 128, 26)
    q[2] = x[17]
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    for ai, ad in (P.knn_approx(xd, sax, qd, k=k), P.knn_approx(xd, None, qd, k=k, index=idx)):
        ai, ad = ai.cpu().numpy(), ad.cpu().numpy()
        for r in range(4):
            assert (np.diff(ad[r]) >= 0).all() and len(set(ai[r].tolist())) == k
            for j in range(k):
                assert abs(np.sqrt(oracle.ed2(x[ai[r, j]], q[r])) - ad[r, j]) <= 1e-5 * max(1.0, ad[r, j])
            assert ad[r, k - 1] >= np.sqrt(rd2[r, k - 1]) * (1 - 1e-6)
    # the leaf of a member query holds the member itself
    ai, ad = P.knn_approx(xd, None, qd, k=1, index=idx)
    assert ai[2, 0].item() == 17 and ad[2, 0].item() == 0.0
