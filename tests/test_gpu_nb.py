"""f2 nb-ParIS+ (paris_knn_nb, Alg7-8) through the C ABI vs the oracle: exact 1-NN with
per-worker BSF copies; stats (raw series read, BSF-copy updates) are consistent."""
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


@pytest.mark.parametrize("n,nq,length", [(1000, 1, 256), (4100, 3, 256), (40_000, 16, 256), (40_000, 21, 128),
                                         (123_456, 9, 256)])
def test_nb_parity(P, n, nq, length):
    import torch
    x = datagen.random_walks(n, length, 700 + n)
    q = datagen.random_walks(nq, length, 701 + nq)
    q[0] = x[n // 5]
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    gi, gd, st = P.knn_nb(xd, sax, torch.from_numpy(q).cuda(), stats=True)
    ri, rd2 = oracle.knn_bruteforce(x, q, 1)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert gi[0, 0].item() == n // 5 and gd[0, 0].item() == 0.0
    assert np.all(st["refined"].numpy() >= 1)
    assert np.all(st["bsf_updates"].numpy() <= st["refined"].numpy())


def test_nb_noisy_and_ties(P):
    import torch
    n = 50_000
    x = datagen.random_walks(n, 256, 31)
    x[40_000] = x[7]
    src = datagen.member_ids(10, n, 32)
    q = datagen.noisy_members(x, src, 0.1, 32)
    q[0] = x[7]
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    gi, gd = P.knn_nb(xd, sax, torch.from_numpy(q).cuda())
    ri, rd2 = oracle.knn_bruteforce(x, q, 1)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert gi[0, 0].item() in (7, 40_000)


def test_nb_rejects_k_gt_1(P):
    import torch
    x = torch.zeros((64, 256), device="cuda")
    sax = P.summarize(x, 16, 256)
    with pytest.raises(ValueError):
        P.knn_exact(x, sax, x[:1], k=2, _nb=True)
