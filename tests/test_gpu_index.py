"""f1 index (paris_index_build / paris_knn_index) through the C ABI vs independent definitions:
the interleaved iSAX key computed here in numpy from the oracle's SAX words, the sort order
(key, id), the block envelopes, and exact k-NN against the oracle's brute force."""
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


def _keys(words_nw, card):
    """Definition (include/paris.h): bits 7..4 of the 8-bit-scaled symbols, interleaved
    most significant first over segments 0..15."""
    shift = 8 - int(np.log2(card))
    sym = (words_nw.astype(np.uint64) << np.uint64(shift)) & np.uint64(0xFF)
    key = np.zeros(words_nw.shape[0], dtype=np.uint64)
    for b in range(7, 3, -1):
        for s in range(16):
            key = (key << np.uint64(1)) | ((sym[:, s] >> np.uint64(b)) & np.uint64(1))
    return key


@pytest.mark.parametrize("n,card", [(16, 256), (2048, 256), (5000 * 16, 256), (4096 + 48, 64), (3000 * 16, 8)])
def test_index_build_matches_definition(P, n, card):
    import torch
    x = datagen.random_walks(n, 256, 300 + n)
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, card)
    idx = P.index_build(sax, 16, card)
    words = sax.cpu().numpy().T.copy()                  # [n][16] (GPU SAX is parity-tested elsewhere)
    keys = _keys(words, card)
    order = np.lexsort((np.arange(n), keys))            # by (key, id)
    perm = idx.perm.cpu().numpy().astype(np.int64)
    np.testing.assert_array_equal(perm, order)
    T = P.PARIS_INDEX_TILE
    ntile = (n + T - 1) // T
    tiled = idx.sax_sorted.cpu().numpy()
    assert tiled.shape == (ntile, 16, T)
    flat = tiled.transpose(1, 0, 2).reshape(16, ntile * T)[:, :n]   # tile-major -> [w][n]
    np.testing.assert_array_equal(flat, sax.cpu().numpy()[:, perm])
    env = idx.env.cpu().numpy()
    ss = words[perm]
    for blk in range(env.shape[0]):
        B = P.PARIS_INDEX_BLOCK
        seg = ss[blk * B:(blk + 1) * B]
        np.testing.assert_array_equal(env[blk, 0], seg.min(0))
        np.testing.assert_array_equal(env[blk, 1], seg.max(0))


@pytest.mark.parametrize("n,nq,k", [(2048, 3, 1), (40_000, 16, 1), (40_000, 5, 10), (100_000, 21, 1), (100_000, 32, 1), (60_000, 45, 10),
                                    (100_000, 9, 100), (6000 * 16, 1, 1), (50_000, 64, 1), (50_000, 65, 3),
                                    (40_000, 100, 1), (30_000, 128, 2)])
def test_knn_index_parity(P, n, nq, k):
    import torch
    x = datagen.random_walks(n, 256, 500 + n)
    q = datagen.random_walks(nq, 256, 501 + nq)
    q[0] = x[n // 3]                                    # member query: distance 0
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    gi, gd = P.knn_index(xd, idx, torch.from_numpy(q).cuda(), k=k)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert gi[0, 0].item() == n // 3 and gd[0, 0].item() == 0.0


def test_knn_index_noisy_members_and_ties(P):
    import torch
    n = 60_000
    x = datagen.random_walks(n, 256, 77)
    x[1000] = x[10]
    x[59_999] = x[10]
    src = datagen.member_ids(12, n, 78)
    q = datagen.noisy_members(x, src, 0.05, 78)
    q[0] = x[10]
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    for k in (1, 3, 50):
        gi, gd = P.knn_index(xd, idx, torch.from_numpy(q).cuda(), k=k)
        ri, rd2 = oracle.knn_bruteforce(x, q, k)
        check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    gi, _ = P.knn_index(xd, idx, torch.from_numpy(q[:1]).cuda(), k=3)
    assert sorted(gi[0].tolist()) == [10, 1000, 59_999]


def test_knn_index_same_as_flat(P):
    """Index and flat scans return the same rows (both exact)."""
    import torch
    n = 80_000
    x = datagen.random_walks(n, 128, 91)
    q = datagen.random_walks(16, 128, 92)
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    a_i, a_d = P.knn_exact(xd, sax, qd, k=5)
    b_i, b_d = P.knn_index(xd, idx, qd, k=5)
    np.testing.assert_allclose(a_d.cpu().numpy(), b_d.cpu().numpy(), rtol=1e-6)


def test_index_rejects_bad_shapes(P):
    import torch
    sax = torch.zeros((16, 20), dtype=torch.uint8, device="cuda")
    with pytest.raises(P.ParisError):
        P.index_build(sax, 16, 256)   # n % 16 != 0


def test_knn_index_overflow_rescan(P):
    """A one-series seed and all-zero queries flood the candidate buffer (count > cap): the
    first pass refines only the stored candidates, the re-scan starts from its result."""
    import torch
    n = 100_000 - 96
    x = datagen.random_walks(n, 128, 41)
    q = np.zeros((3, 128), dtype=np.float32)
    q[1] = x[5]
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    for k in (1, 1000):
        gi, gd, st = P.knn_index(xd, idx, torch.from_numpy(q).cuda(), k=k,
                                 config=P.KnnConfig(index_seeds=1, cap=65536), stats=True)
        ri, rd2 = oracle.knn_bruteforce(x, q, k)
        check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)


@pytest.mark.parametrize("card,length,k", [(64, 256, 1), (16, 256, 3), (256, 128, 1), (8, 128, 5)])
def test_knn_index_cardinalities_and_lengths(P, card, length, k):
    """The index path at every supported shape the LB tables take: cardinalities below 256
    (symbols scaled to 8 bits in the key; region tables of the smaller card) and len 128."""
    import torch
    n, nq = 30_000, 70
    x = datagen.random_walks(n, length, 600 + card + length)
    q = datagen.random_walks(nq, length, 601 + card)
    q[:5] = x[[0, 7, 29_999, 15_000, 123]]
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, card)
    idx = P.index_build(sax, 16, card)
    gi, gd = P.knn_index(xd, idx, torch.from_numpy(q).cuda(), k=k)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)


@pytest.mark.parametrize("scale,shift", [(1.0, 0.0), (1e6, 3e6), (1e-4, 0.0)])
@pytest.mark.parametrize("k", [1, 4])
def test_knn_index_bf16_prefilter(P, scale, shift, k):
    """paris_knn_index_x: the bf16 pre-filter only drops candidates whose rigorous lower bound
    exceeds the BSF -> results identical to paris_knn_index_ex and to the oracle, on z-normalized
    data, on data far from unit scale (the bound is relative to ||x~||), with near-member queries
    (distances of the order of the bf16 rounding), exact duplicates (ties) and k > 1 (ignored)."""
    import torch
    n, nq, length = 40_000, 40, 256
    x = datagen.random_walks(n, length, 700 + k) * np.float32(scale) + np.float32(shift)
    q = datagen.random_walks(nq, length, 701 + k) * np.float32(scale) + np.float32(shift)
    rng = np.random.default_rng(5)
    q[:6] = x[[3, 3000, 39_999, 20_000, 77, 5]] + (1e-3 * scale * rng.standard_normal((6, length))).astype(np.float32)
    x[9] = x[3]                                          # duplicate of a near-member's source (tie)
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    r16 = P.raw_bf16(xd)
    qd = torch.from_numpy(q).cuda()
    gi, gd, st = P.knn_index(xd, idx, qd, k=k, raw16=r16, stats=True)
    hi, hd = P.knn_index(xd, idx, qd, k=k)
    assert torch.equal(gi, hi) and torch.equal(gd, hd)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    if k == 1 and scale == 1.0:
        assert gi[0, 0].item() == 3                      # tie with id 9: the lower id
        _, _, st0 = P.knn_index(xd, idx, qd, k=k, stats=True)
        assert st["refined"].sum() < st0["refined"].sum()  # fp32 rows actually skipped


def test_raw_bf16_definition(P):
    import torch
    x = torch.randn(1000, 64, device="cuda") * 100
    r = P.raw_bf16(x)
    ref = x.to(torch.bfloat16).view(torch.int16)
    assert torch.equal(r, ref)


@pytest.mark.parametrize("k", [1, 7, 1000])
def test_knn_overflow_fallback_mixed(P, k):
    """Device-side overflow handling: in one call, some queries flood their candidate
    buffers (all-zero queries with a one-series seed: nearly every LB is tiny) while the
    others do not; the flooded ones are completed by the gated fused scan (k_fallback),
    the rest must be untouched by it.  Both paths, two passes of the index path, and
    k > 1 rows whose first pass kept fewer than k results.  Checked against brute force."""
    import torch
    n, length, nq = 70_000 - 16 * 3, 128, 70
    x = datagen.random_walks(n, length, 4242)
    q = datagen.random_walks(nq, length, 4243)
    flood = [0, 5, 63, 64, 69]
    q[flood] = 0.0
    q[10] = x[77]
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    cfg = P.KnnConfig(index_seeds=1, seed_div=n, cap=65536)
    gi, gd, st = P.knn_index(xd, idx, qd, k=k, config=cfg, stats=True)
    fi, fd = P.knn_exact(xd, sax, qd, k=k, config=cfg)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    check_knn(x, q, fi.cpu().numpy(), fd.cpu().numpy(), ri, rd2)
    cap = 65536
    assert (st["candidates"].numpy()[flood] > cap).all(), "the flooded queries did not overflow"


@pytest.mark.parametrize("scale,shift,w2,with16,length", [(1.0, 0.0, 64, False, 256), (1.0, 0.0, 32, False, 256),
                                                         (1.0, 0.0, 64, True, 256), (1.0, 0.0, 32, False, 128),
                                                         (1e4, 3e4, 64, False, 256), (1e-4, 0.0, 64, True, 256)])
def test_knn_index_paa_prefilter(P, scale, shift, w2, with16, length):
    """paris_knn_index_aux: the fp16 PAA pre-filter (then optionally the bf16 one) only drops
    candidates whose rigorous PAA lower bound exceeds the BSF -> results identical to the
    unfiltered index search and to the oracle: z-normalized data, data far from unit scale
    (PAA means beyond the fp16 range are stored as NaN: no pruning on them), tiny scale
    (fp16 subnormals), near-member queries, exact duplicates (ties)."""
    import torch
    n, nq = 40_000, 40
    x = datagen.random_walks(n, length, 800 + w2) * np.float32(scale) + np.float32(shift)
    q = datagen.random_walks(nq, length, 801 + w2) * np.float32(scale) + np.float32(shift)
    rng = np.random.default_rng(6)
    q[:6] = x[[3, 3000, 39_999, 20_000, 77, 5]] + (1e-3 * scale * rng.standard_normal((6, length))).astype(np.float32)
    x[9] = x[3]                                          # duplicate of a near-member's source (tie)
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    paa = P.paa_f16(xd, w2)
    r16 = P.raw_bf16(xd) if with16 else None
    qd = torch.from_numpy(q).cuda()
    gi, gd, st = P.knn_index(xd, idx, qd, k=1, paa16=paa, raw16=r16, stats=True)
    hi, hd = P.knn_index(xd, idx, qd, k=1)
    assert torch.equal(gi, hi) and torch.equal(gd, hd)
    ri, rd2 = oracle.knn_bruteforce(x, q, 1)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert gi[0, 0].item() == 3                          # tie with id 9: the lower id
    assert st["paa_rows"].sum() > 0
    if scale == 1.0:
        _, _, st0 = P.knn_index(xd, idx, qd, k=1, stats=True)
        assert st["refined"].sum() < st0["refined"].sum()  # fp32 rows actually skipped


def test_paa_f16_definition(P):
    """paris_paa_f16 = the fp64 segment means rounded to nearest fp16 (NaN beyond the fp16 range)."""
    import torch
    x = (torch.randn(2000, 256, device="cuda", dtype=torch.float64) * 3).float()
    x[7] *= 1e5
    for w2 in (32, 64):
        got = P.paa_f16(x, w2).view(torch.float16).float().cpu().numpy()
        m = x.double().view(2000, w2, -1).mean(-1).cpu().numpy()
        ref = m.astype(np.float32).astype(np.float16).astype(np.float32)
        ok = np.abs(m) < 65000
        assert np.array_equal(got[ok], ref[ok])
        assert np.isnan(got[~ok]).all() and (~ok).any()


@pytest.mark.parametrize("k,w2,length", [(4, 64, 256), (100, 64, 256), (10, 32, 128)])
def test_knn_index_paa_prefilter_k(P, k, w2, length):
    """k > 1 with the PAA pre-filter (k_refine_kx): each candidate below the live k-th
    threshold meets the PAA bound before its raw row -- the exact top-k, equal to the
    unfiltered search and to the oracle (member queries, ties)."""
    import torch
    n, nq = 30_000 + 16, 20
    x = datagen.random_walks(n, length, 900 + k)
    q = datagen.random_walks(nq, length, 901 + k)
    q[:3] = x[[11, 29_000, 500]]
    x[12] = x[11]                                      # a tie at distance 0
    xd = torch.from_numpy(x).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    paa = P.paa_f16(xd, w2)
    qd = torch.from_numpy(q).cuda()
    gi, gd, st = P.knn_index(xd, idx, qd, k=k, paa16=paa, stats=True)
    hi, hd, st0 = P.knn_index(xd, idx, qd, k=k, stats=True)
    assert torch.equal(gi, hi) and torch.equal(gd, hd)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    assert st["paa_rows"].sum() > 0 and st["refined"].sum() < st0["refined"].sum()


@pytest.mark.parametrize("key,values", [(0, (24, 30)), (1, (0, 1)), (2, (0, 1)), (3, (0, 1))])
def test_kernel_variants_identical(P, key, values):
    """Tuning variants (paris_debug_set_variant): the index LB pass at 24 and 30 consumer warps,
    the batch-1 flat LB as k_lb1 / k_lb1t, and the pre-filtered refine with and without its
    loads pipelined, return identical rows, equal to the oracle's."""
    import torch
    n = 70_000
    x = datagen.random_walks(n, 256, 610)
    q = datagen.random_walks(40, 256, 611)
    q[3] = x[n - 5]
    xd = torch.from_numpy(x).cuda()
    qd = torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256) if key != 1 else None
    r16, p16 = (P.raw_bf16(xd), P.paa_f16(xd, 64)) if key == 2 else (None, None)
    ri, rd2 = oracle.knn_bruteforce(x, q, 1 if key == 2 else 4)
    outs = []
    old = P.debug_set_variant(key, values[0])
    try:
        for v in values:
            P.debug_set_variant(key, v)
            if key in (0, 3):
                gi, gd = P.knn_index(xd, idx, qd, k=4)
            elif key == 2:
                gi, gd = P.knn_index(xd, idx, qd, k=1, raw16=r16, paa16=p16)
            else:
                gi, gd = P.knn_exact(xd, sax, qd, k=4, config=P.KnnConfig(batch=1))
            check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
            outs.append((gi.cpu(), gd.cpu()))
    finally:
        P.debug_set_variant(key, old)
    assert all(torch.equal(o[0], outs[0][0]) and torch.equal(o[1], outs[0][1]) for o in outs)
