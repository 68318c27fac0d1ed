"""Tensor-core filter of the index LB pass (k_gf, DESIGN.md f1; MINDIST P:1107-1123).

The unit test checks the tcgen05 path (table lookups -> A rows in shared memory -> three
MMAs per 128 series -> TMEM -> registers) against the same sum written out in fp64 from
the same fp16 inputs, and measures the accumulation error that the filter's margin
(kGfAccRel = 2^-17 of the sum of |products|) has to cover.  The search tests compare the
variant with the oracle and with the default index pass."""
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


def _tile_major(words):
    """[n, 16] uint8 -> the index's tile-major array (whole 2048-series tiles)."""
    n = words.shape[0]
    nt = (n + 2047) // 2048
    buf = np.zeros((nt, 16, 2048), dtype=np.uint8)
    pad = np.zeros((nt * 2048, 16), dtype=np.uint8)
    pad[:n] = words
    buf[:] = pad.reshape(nt, 2048, 16).transpose(0, 2, 1)
    return buf


@pytest.mark.parametrize("n", [16, 272, 4096 + 48, 300_000])
def test_gf_mma_unit(P, n):
    import torch
    rng = np.random.default_rng(900 + n % 97)
    words = rng.integers(0, 256, size=(n, 16), dtype=np.uint8)
    c = rng.uniform(-3.0, 3.0, 256).astype(np.float16)
    g = rng.uniform(-2.0, 9.0, 256).astype(np.float16)
    tabw = (c.view(np.uint16).astype(np.uint32) | (g.view(np.uint16).astype(np.uint32) << 16)).astype(np.uint32)
    B = np.zeros((64, 48), dtype=np.float16)
    B[:, 0:32:2] = (-2.0 * rng.uniform(-3.0, 3.0, (64, 16))).astype(np.float16)
    B[:, 1:32:2] = 1.0
    B[:, 32] = rng.uniform(-30.0, 30.0, 64).astype(np.float16)
    B[:, 33] = rng.uniform(-0.01, 0.01, 64).astype(np.float16)
    A = np.zeros((n, 34), dtype=np.float64)
    A[:, 0:32:2] = c.astype(np.float64)[words]
    A[:, 1:32:2] = g.astype(np.float64)[words]
    A[:, 32] = 1.0
    A[:, 33] = 1.0
    Bd = B[:, :34].astype(np.float64)
    want = A @ Bd.T
    mag = np.abs(A) @ np.abs(Bd).T
    sd = torch.from_numpy(_tile_major(words)).cuda()
    td = torch.from_numpy(tabw.view(np.int32)).cuda()
    bd = torch.from_numpy(B.view(np.int16)).cuda()
    res = {}
    for swap in (0, 1):
        got = P.debug_gf_mma(sd, n, td, bd, swap_desc=swap).cpu().numpy().astype(np.float64)
        res[swap] = float(np.max(np.abs(got - want) / mag))
    print(f"gf_mma n={n}: max |err| / sum|products| = {res[0]:.3e} (swapped descriptors: {res[1]:.3e}); "
          f"margin 2^-17 = {2.0 ** -17:.3e}")
    assert res[0] <= 2.0 ** -17 / 4, res


@pytest.mark.parametrize("n,nq,k,card", [(70_000, 40, 1, 256), (70_000, 64, 4, 256), (33_008, 7, 10, 64),
                                          (200_000, 100, 1, 256)])
def test_knn_index_gf_parity(P, n, nq, k, card):
    import torch
    x = datagen.random_walks(n, 256, 920 + k)
    q = datagen.random_walks(nq, 256, 921 + k)
    q[1] = x[n - 3]
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, card)
    idx = P.index_build(sax, 16, card)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    hi, hd, st0 = P.knn_index(xd, idx, qd, k=k, stats=True)
    old = P.debug_set_variant(3, 1)
    try:
        gi, gd, st1 = P.knn_index(xd, idx, qd, k=k, stats=True)
    finally:
        P.debug_set_variant(3, old)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert torch.equal(gi, hi) and torch.equal(gd, hd)
    # the filter ran (no envelope blocks were bounded) and kept a comparable candidate set
    assert int(st1["lb_blocks"].sum()) == 0 and int(st0["lb_blocks"].sum()) > 0
    c0, c1 = int(st0["candidates"].sum()), int(st1["candidates"].sum())
    print(f"candidates: k_lbi {c0}, k_gf {c1}")
    assert c1 <= c0 * 1.01 + 16  # fp32 MINDIST is at least as tight as the fp16 one


@pytest.mark.parametrize("n,nq,k", [(70_000, 40, 1), (50_000 + 16, 64, 3), (33_008, 100, 1), (20_000, 9, 5)])
def test_knn_flat_gf_parity(P, n, nq, k):
    """paris_knn_exact behind the filter: 64 query slots per pass of the flat [16][n] array
    (seeds per 16-slot sub-batch), same rows as the default flat path and the oracle."""
    import torch
    x = datagen.random_walks(n, 256, 940 + k)
    q = datagen.random_walks(nq, 256, 941 + k)
    q[nq - 1] = x[7]
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, 256)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    old = P.debug_set_variant(3, 0)
    try:
        hi, hd, st0 = P.knn_exact(xd, sax, qd, k=k, stats=True)  # k_lbt, 16 slots per pass
        P.debug_set_variant(3, 2)
        gi, gd, st1 = P.knn_exact(xd, sax, qd, k=k, stats=True)  # k_gf, 64 slots per pass (the default)
    finally:
        P.debug_set_variant(3, old)
    assert old == 2
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert torch.equal(gi, hi) and torch.equal(gd, hd)
    c0, c1 = int(st0["candidates"].sum()), int(st1["candidates"].sum())
    print(f"flat candidates: k_lbt {c0}, k_gf {c1}")


def test_knn_flat_gf_unnormalized_falls_back(P):
    import torch
    n = 40_000
    x = datagen.random_walks(n, 256, 950)
    q = datagen.random_walks(20, 256, 951)
    q[17] = q[17] * 40.0 + 25.0
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, 256)
    ri, rd2 = oracle.knn_bruteforce(x, q, 2)
    gi, gd = P.knn_exact(xd, sax, qd, k=2)  # the filter is the flat path's default
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)


def test_knn_index_gf_unnormalized_falls_back(P):
    """Query PAA beyond +-16: the filter declines the pass and the block pass + k_lbi run."""
    import torch
    n = 40_000
    x = datagen.random_walks(n, 256, 930)
    q = datagen.random_walks(5, 256, 931)
    q[2] = q[2] * 40.0 + 25.0
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    ri, rd2 = oracle.knn_bruteforce(x, q, 2)
    old = P.debug_set_variant(3, 1)
    try:
        gi, gd, st = P.knn_index(xd, idx, qd, k=2, stats=True)
    finally:
        P.debug_set_variant(3, old)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert int(st["lb_blocks"].sum()) > 0
