"""CUDA path (through the C ABI) vs the CPU oracle, element by element, on seeded inputs.

Small sizes span several tiles and ragged tails; edge cases: n = 1, 15, 16, 17,
odd n (byte-granular SAX tails), constant series (PAA exactly on the median cut),
PAA planted on cuts, exact duplicate series (ties -> lower id), member queries
(distance 0), k = n, every supported cardinality, non-default (len, w).
"""
import numpy as np
import pytest

import datagen
import oracle
from tests._parity import check_knn, sax_mismatches

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import __graft_entry__ as ge
    ge.build()
    import paper_2009_00166_b200 as p
    return p


@pytest.fixture(scope="module")
def torch_dev():
    import torch
    return torch, torch.device("cuda:0")


def _to(torch_dev, a):
    torch, dev = torch_dev
    return torch.from_numpy(np.ascontiguousarray(a)).to(dev)


# ---------------------------------------------------------------- summarize
@pytest.mark.parametrize("n", [1, 15, 16, 17, 511, 1000, 4099, 100_003])
@pytest.mark.parametrize("length", [128, 256])
def test_summarize_parity_sizes(P, torch_dev, n, length):
    x = datagen.random_walks(n, length, 1000 + n + length)
    sax = P.summarize(_to(torch_dev, x), 16, 256).cpu().numpy()
    bad, exempt, _ = sax_mismatches(x, sax, 16, 256)
    assert len(bad) == 0, bad[:10]


@pytest.mark.parametrize("length,w", [(256, 8), (256, 4), (256, 2), (256, 1), (128, 32),
                                      (512, 16), (1024, 64), (96, 12), (100, 5), (384, 16)])
@pytest.mark.parametrize("card", [2, 8, 64, 256])
def test_summarize_parity_shapes(P, torch_dev, length, w, card):
    x = datagen.random_walks(777, length, 7 + length + w)
    sax = P.summarize(_to(torch_dev, x), w, card).cpu().numpy()
    bad, _, _ = sax_mismatches(x, sax, w, card)
    assert len(bad) == 0, bad[:10]


def test_summarize_planted_cuts_exact(P, torch_dev):
    """Segments whose PAA equals fp32(cut) or sits within an ulp of it: the CUDA path decides
    with the exact PAA (fp64 recheck), so it agrees with the fp64 oracle even inside the window."""
    card, w, length = 256, 16, 256
    cuts = oracle.cuts(card)
    rng = np.random.default_rng(0)
    rows = []
    for i in range(2000):
        c = cuts[rng.integers(0, card - 1, w)].astype(np.float32)
        c = np.nextafter(c, np.float32(rng.choice([-np.inf, np.inf])), dtype=np.float32) \
            if i % 3 == 0 else c
        seg = np.repeat(c, length // w).astype(np.float32)
        # perturb points but keep the segment mean exactly (pairs +e/-e)
        e = rng.normal(0, 0.5, length // 2).astype(np.float32)
        pert = np.stack([e, -e], 1).reshape(-1)
        rows.append(seg + pert if i % 2 else seg)
    x = np.stack(rows).astype(np.float32)
    x[:5] = 0.0  # constant series: PAA exactly 0 = the median cut -> upper region
    sax = P.summarize(_to(torch_dev, x), w, card).cpu().numpy()
    ref = oracle.summarize(x, w, card)
    got = sax.reshape(w, -1).T
    mism = np.argwhere(got != ref)
    # only segments whose exact PAA is within 1e-6 of a cut may differ (north_star); count them
    paa = oracle.paa(x, w)
    near = np.min(np.abs(paa[..., None] - cuts), axis=-1) < 1e-6
    assert all(near[i, j] for i, j in mism)
    assert np.all(got[:5] == card // 2)
    assert len(mism) <= 0.001 * got.size, len(mism)


def test_summarize_unaligned_output_rows(P, torch_dev):
    """n % 16 != 0: every SAX row starts unaligned; tail tiles use byte stores."""
    for n in (129, 130, 255, 257, 1023):
        x = datagen.random_walks(n, 256, n)
        sax = P.summarize(_to(torch_dev, x), 16, 256).cpu().numpy()
        bad, _, _ = sax_mismatches(x, sax, 16, 256)
        assert len(bad) == 0, (n, bad[:5])


# ---------------------------------------------------------------- k-NN
def _knn_case(P, torch_dev, x, q, k, w=16, card=256, host=False, config=None):
    xd = _to(torch_dev, x)
    sax = P.summarize(xd, w, card)
    qd = _to(torch_dev, q) if not host else __import__("torch").from_numpy(np.ascontiguousarray(q))
    gi, gd = P.knn_exact(xd, sax, qd, k=k, w=w, card=card, config=config)
    return gi.cpu().numpy(), gd.cpu().numpy()


@pytest.mark.parametrize("n,k", [(1, 1), (17, 1), (17, 5), (17, 17), (1000, 1), (1000, 10),
                                 (1000, 100), (5003, 1), (5003, 10), (20_000, 1), (20_000, 100)])
def test_knn_parity_bruteforce(P, torch_dev, n, k):
    x = datagen.random_walks(n, 256, 50 + n)
    q = datagen.random_walks(9, 256, 60 + n)
    gi, gd = _knn_case(P, torch_dev, x, q, k)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi, gd, ri, rd2)


@pytest.mark.parametrize("card", [2, 8, 64, 256])
@pytest.mark.parametrize("length,w", [(256, 16), (128, 16), (256, 8), (96, 12)])
def test_knn_parity_card_shape(P, torch_dev, card, length, w):
    x = datagen.random_walks(3001, length, card + length)
    q = datagen.random_walks(5, length, card + length + 1)
    for k in (1, 7):
        gi, gd = _knn_case(P, torch_dev, x, q, k, w=w, card=card)
        ri, rd2 = oracle.knn_bruteforce(x, q, k)
        check_knn(x, q, gi, gd, ri, rd2)


def test_knn_duplicates_members_ties(P, torch_dev):
    n = 4000
    x = datagen.random_walks(n, 256, 99)
    x[1000] = x[10]
    x[3999] = x[10]
    x[2000] = x[20]
    q = np.concatenate([x[[10, 20, 30]], datagen.random_walks(3, 256, 98)])
    gi, gd = _knn_case(P, torch_dev, x, q, 3)
    assert list(gi[0]) == [10, 1000, 3999] and np.all(gd[0] == 0)
    assert list(gi[1][:2]) == [20, 2000] and gd[1][0] == 0
    assert gi[2][0] == 30 and gd[2][0] == 0
    ri, rd2 = oracle.knn_bruteforce(x, q, 3)
    check_knn(x, q, gi, gd, ri, rd2)


def test_knn_noisy_member_queries(P, torch_dev):
    """Config-2/5 style: dataset series + N(0, sigma^2) noise, re-z-normalized."""
    x = datagen.random_walks(30_000, 256, 5)
    for sigma in (0.01, 0.05, 0.2):
        src = datagen.member_ids(8, 30_000, 6)
        q = datagen.noisy_members(x, src, sigma, 6)
        for k in (1, 10, 100):
            gi, gd = _knn_case(P, torch_dev, x, q, k)
            ri, rd2 = oracle.knn_bruteforce(x, q, k)
            check_knn(x, q, gi, gd, ri, rd2)


def test_knn_host_buffers_and_batches(P, torch_dev):
    """Host queries/outputs through the same ABI call; batch sizes 1..8 and ragged last batch."""
    import paper_2009_00166_b200 as p
    x = datagen.random_walks(7000, 128, 3)
    q = datagen.random_walks(19, 128, 4)
    ri, rd2 = oracle.knn_bruteforce(x, q, 4)
    for b in (1, 3, 8):
        gi, gd = _knn_case(P, torch_dev, x, q, 4, host=True, config=p.KnnConfig(batch=b))
        check_knn(x, q, gi, gd, ri, rd2)


@pytest.mark.parametrize("n", [16, 2048, 2064, 9 * 2048 + 400, 150_000])
def test_knn_batch1_tiled_pass(P, torch_dev, n):
    """One query per SAX pass on the tiled layout (k_lb1t: TMA ring of 2048-series tiles,
    ragged last tile): k = 1 and k = 9 against the oracle, member queries (LB = 0
    candidates in the last tile) and a capacity small enough to overflow."""
    import paper_2009_00166_b200 as p
    x = datagen.random_walks(n, 256, 77 + n)
    q = np.concatenate([datagen.random_walks(4, 256, 78 + n), x[[n - 1, n // 2]]])
    for k in (1, 9):
        kk = min(k, n)
        ri, rd2 = oracle.knn_bruteforce(x, q, kk)
        gi, gd = _knn_case(P, torch_dev, x, q, kk, config=p.KnnConfig(batch=1))
        check_knn(x, q, gi, gd, ri, rd2)
        if n >= 2048:
            gi, gd = _knn_case(P, torch_dev, x, q, kk, config=p.KnnConfig(batch=1, seed_div=n, cap=64))
            check_knn(x, q, gi, gd, ri, rd2)


def test_knn_pruned_oracle_and_stats(P, torch_dev):
    """Larger n against the oracle's LB-pruned scan (itself pinned to brute force)."""
    torch, dev = torch_dev
    n = 200_000
    x = datagen.random_walks(n, 256, 123)
    q = datagen.random_walks(6, 256, 124)
    sax_o = oracle.summarize(x, 16, 256)
    ri, rd2 = oracle.knn_pruned(x, sax_o, q, 10, 16, 256)
    xd = _to(torch_dev, x)
    sax = P.summarize(xd, 16, 256)
    gi, gd, st = P.knn_exact(xd, sax, _to(torch_dev, q), k=10, stats=True)
    check_knn(x, q, gi.cpu().numpy(), gd.cpu().numpy(), ri, rd2)
    cand = st["candidates"].numpy()
    refined = st["refined"].numpy()
    assert np.all(refined <= cand) and np.all(cand < n // 4)
    # the seed is an upper bound of the true k-th distance
    assert np.all(st["tau_seed"].numpy() >= np.sqrt(rd2[:, -1]) * (1 - 1e-6))


def test_knn_overflow_rescan(P, torch_dev):
    """A weak seed (seed_div huge -> tiny sample) floods the candidate buffer for k = n-ish;
    the library re-scans the overflowed query with an exact-size buffer."""
    import paper_2009_00166_b200 as p
    n = 70_000  # default capacity is max(65536, n/32) = 65536 < n
    x = datagen.random_walks(n, 128, 8)
    q = -datagen.random_walks(2, 128, 9) * 0.0  # all-zero queries: LB of most series is small
    gi, gd = _knn_case(P, torch_dev, x, q, 1000, config=p.KnnConfig(seed_div=n, cap=65536))
    ri, rd2 = oracle.knn_bruteforce(x, q, 1000)
    check_knn(x, q, gi, gd, ri, rd2)


def test_gpu_datagen_matches_numpy(torch_dev):
    from datagen import gpu
    import __graft_entry__ as ge
    ge.build()
    a = gpu.walks(300, 256, 77, first_id=5).cpu().numpy()
    b = datagen.random_walks(300, 256, 77, first_id=5)
    assert np.max(np.abs(a - b)) < 1e-5
    xd = gpu.walks(100, 128, 1)
    qd, src = gpu.noisy_members(xd, 10, 0.05, 2)
    qn = datagen.noisy_members(xd.cpu().numpy(), src, 0.05, 2)
    assert np.max(np.abs(qd.cpu().numpy() - qn)) < 1e-5


@pytest.mark.parametrize("n", [2048, 4096 + 16, 3 * 2048 + 1024 + 48, 40_000])
@pytest.mark.parametrize("nq", [1, 2, 3, 9, 16, 21])
def test_knn_tiled_path_parity(P, torch_dev, n, nq):
    """n % 16 == 0, w == 16: the TMA-tiled LB kernels (ragged last tile, every query-slot
    layout: single, pairs, dummy slots) against the oracle and the direct-load kernels."""
    import paper_2009_00166_b200 as p
    x = datagen.random_walks(n, 256, 900 + n)
    q = datagen.random_walks(nq, 256, 901 + nq)
    q[0] = x[n // 2]
    for k in (1, 10):
        ri, rd2 = oracle.knn_bruteforce(x, q, k)
        gi, gd = _knn_case(P, torch_dev, x, q, k)
        check_knn(x, q, gi, gd, ri, rd2)
        gi2, gd2 = _knn_case(P, torch_dev, x, q, k, config=p.KnnConfig(force_direct=True))
        check_knn(x, q, gi2, gd2, ri, rd2)


@pytest.mark.parametrize("wave_a", [1, 7, 2048, 1_000_000])
@pytest.mark.parametrize("sorted_refine", [False, True])
def test_knn_refine_waves(P, torch_dev, wave_a, sorted_refine):
    """k = 1 refinement: the two LB waves taken from the unsorted candidate lists (default)
    and from the bucket-sorted lists (K5), for wave cuts from one candidate to all of them,
    on the flat and the index path, against the oracle (noisy members: many near ties)."""
    import paper_2009_00166_b200 as p
    torch, dev = torch_dev
    n = 30_000
    x = datagen.random_walks(n, 256, 4242)
    q = datagen.random_walks(20, 256, 4243)
    q[:10] = datagen.noisy_members(x, np.arange(10) * 2999, 0.2, 4244)
    ri, rd2 = oracle.knn_bruteforce(x, q, 1)
    cfg = p.KnnConfig(wave_a=wave_a, sorted_refine=sorted_refine)
    gi, gd = _knn_case(P, torch_dev, x, q, 1, config=cfg)
    check_knn(x, q, gi, gd, ri, rd2)
    xd = torch.from_numpy(x).to(dev)
    sax = P.summarize(xd, 16, 256)
    idx = P.index_build(sax, 16, 256)
    hi, hd = P.knn_index(xd, idx, torch.from_numpy(q).to(dev), k=1, config=cfg)
    check_knn(x, q, hi.cpu().numpy(), hd.cpu().numpy(), ri, rd2)


@pytest.mark.parametrize("n,w,length,k", [(5003, 8, 64, 1), (5003, 16, 128, 5), (4096, 12, 96, 1), (4096, 16, 256, 1000)])
def test_knn_overflow_fallback_shapes(P, torch_dev, n, w, length, k):
    """The overflow fallback on every layout it has: the generic per-series loop (w != 16 or
    n % 4 != 0) and the 4-series-per-lane form, k = 1 (shared BSF key) and k > 1 (warp lists
    merged): a tiny forced capacity makes most queries overflow."""
    import paper_2009_00166_b200 as p
    x = datagen.random_walks(n, length, 7000 + n + w)
    q = datagen.random_walks(6, length, 7001 + w)
    q[1] = 0.0
    q[4] = x[n - 1]
    gi, gd = _knn_case(P, torch_dev, x, q, k, w=w, config=p.KnnConfig(cap=16, seed_div=n))
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi, gd, ri, rd2)


def test_gpu_member_queries_by_id(torch_dev):
    """Sharded benches build member queries from rows generated by id: identical to
    noisy_members over the whole collection."""
    from datagen import gpu
    import __graft_entry__ as ge
    ge.build()
    xd = gpu.walks(5000, 128, 31)
    a, src_a = gpu.noisy_members(xd, 12, 0.1, 32)
    b, src_b = gpu.member_queries(5000, 128, 31, 12, 0.1, 32)
    assert np.array_equal(src_a, src_b)
    assert torch_equal(a, b)


def torch_equal(a, b):
    import torch
    return bool(torch.equal(a, b))


@pytest.mark.parametrize("k", [1025, 3000, 5003])
def test_knn_large_k_full_sort(P, torch_dev, k):
    """k beyond PARIS_MAX_K up to k = n: every series' distance, keys sorted --
    equal to brute force (k = n is the full sort), on the flat and index paths."""
    import torch
    n = 5003
    x = datagen.random_walks(n, 128, 8100)
    q = datagen.random_walks(3, 128, 8101)
    q[1] = x[4000]
    gi, gd = _knn_case(P, torch_dev, x, q, k, w=16)
    ri, rd2 = oracle.knn_bruteforce(x, q, k)
    check_knn(x, q, gi, gd, ri, rd2)
    assert gi[1, 0] == 4000
