"""Pins for the CPU oracle (oracle/oracle.c) -- each against something other than itself.

Pins used: the worked examples in tests/golden (closed
forms from the paper's definitions), two independent library quantile routines
(scipy ndtri, statistics.NormalDist = AS241), numpy re-implementations that use
a *different* formulation (reshape-mean, searchsorted, clamp-projection for the
lower bound), brute-force minimisation over the iSAX box, the invariants
LB <= ED and monotonicity in cardinality, and brute-force k-NN via a full sort.
"""
import json
import os
import statistics

import numpy as np
import pytest
from scipy.special import ndtri

import datagen
import oracle

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "worked_examples.json")))
CARDS = [2, 4, 8, 16, 32, 64, 128, 256]


# ---------------------------------------------------------------- worked examples
@pytest.mark.parametrize("case", GOLD["paa"])
def test_paa_worked(case):
    got = oracle.paa(np.array(case["x"], np.float32), case["w"])[0]
    assert np.array_equal(got, np.array(case["expect"]))


@pytest.mark.parametrize("case", GOLD["cuts"])
def test_cuts_worked(case):
    got = oracle.cuts(case["card"])
    assert np.allclose(got, case["expect"], atol=case["tol"], rtol=0)


@pytest.mark.parametrize("case", GOLD["sax_symbol"])
def test_sax_worked(case):
    assert oracle.sax_symbol(case["v"], case["card"]) == case["expect"]


@pytest.mark.parametrize("case", GOLD["lb"])
def test_lb_worked(case):
    T = oracle.lb_table(np.array(case["qpaa"]), case["len"], case["w"], case["card"])
    lb = np.sqrt(oracle.lb2(T, np.array([case["word"]], np.uint8))[0])
    assert lb == pytest.approx(case["expect_lb"], rel=1e-15, abs=1e-15)


@pytest.mark.parametrize("case", GOLD["ed"])
def test_ed_worked(case):
    assert np.sqrt(oracle.ed2(np.array(case["a"]), np.array(case["b"]))) == case["expect"]


# ---------------------------------------------------------------- breakpoints
@pytest.mark.parametrize("card", CARDS)
def test_cuts_match_two_library_quantiles(card):
    c = oracle.cuts(card)
    p = np.arange(1, card) / card
    ref1 = ndtri(p)
    nd = statistics.NormalDist()
    ref2 = np.array([nd.inv_cdf(x) for x in p])
    assert np.max(np.abs(c - ref1)) < 2e-15
    assert np.max(np.abs(c - ref2)) < 2e-15
    assert np.all(np.diff(c) > 0)
    # symmetry c[k] = -c[card-2-k] and exact median 0
    assert np.max(np.abs(c + c[::-1])) < 2e-15
    assert c[card // 2 - 1] == 0.0


def test_cuts_reject_bad_card():
    for card in (0, 1, 3, 6, 512):
        with pytest.raises(ValueError):
            oracle.cuts(card)


# ---------------------------------------------------------------- PAA / SAX
def test_paa_matches_reshape_mean():
    x = datagen.random_walks(64, 256, 11)
    for w in (1, 2, 4, 8, 16, 32, 64):
        ref = x.astype(np.float64).reshape(64, w, 256 // w).mean(axis=2)
        assert np.allclose(oracle.paa(x, w), ref, rtol=0, atol=1e-13)


@pytest.mark.parametrize("card", CARDS)
def test_sax_symbol_is_count_of_cuts_below(card):
    rng = np.random.default_rng(card)
    ref_cuts = ndtri(np.arange(1, card) / card)
    v = rng.normal(0, 1.3, 2000)
    v = v[np.min(np.abs(v[:, None] - ref_cuts[None, :]), axis=1) > 1e-9]
    got = np.array([oracle.sax_symbol(x, card) for x in v])
    assert np.array_equal(got, np.searchsorted(ref_cuts, v, side="right"))
    # on-cut values go to the upper region (reading 3)
    for k in range(0, card - 1, max(1, (card - 1) // 7)):
        cut = oracle.cuts(card)[k]
        assert oracle.sax_symbol(cut, card) == k + 1


def test_sax_monotone_and_prefix_consistent():
    v = np.linspace(-4, 4, 3001)
    full = np.array([oracle.sax_symbol(x, 256) for x in v])
    assert np.all(np.diff(full) >= 0) and full[0] == 0 and full[-1] == 255
    for b in range(1, 8):
        card = 1 << b
        sym = np.array([oracle.sax_symbol(x, card) for x in v])
        assert np.array_equal(sym, full >> (8 - b)), b


@pytest.mark.parametrize("len_,w,card", [(256, 16, 256), (128, 16, 256), (256, 8, 4), (96, 12, 64)])
def test_summarize_matches_numpy_pipeline(len_, w, card):
    x = datagen.random_walks(500, len_, 7)
    got = oracle.summarize(x, w, card)
    paa = x.astype(np.float64).reshape(500, w, len_ // w).mean(axis=2)
    ref_cuts = ndtri(np.arange(1, card) / card)
    ref = np.searchsorted(ref_cuts, paa, side="right")
    near = np.min(np.abs(paa[..., None] - ref_cuts), axis=-1) < 1e-9
    assert np.array_equal(got[~near], ref[~near])
    assert got.dtype == np.uint8 and got.max() < card


# ---------------------------------------------------------------- lower bound
def _lu(card):
    c = ndtri(np.arange(1, card) / card)
    return np.concatenate([[-np.inf], c]), np.concatenate([c, [np.inf]])


@pytest.mark.parametrize("card", [2, 8, 64, 256])
def test_lb_is_distance_to_isax_box(card):
    """LB^2 = (len/w) * ||q - clamp(q, L, U)||^2: the squared distance from the query
    PAA to the box of PAA vectors the word admits (a clamp, not the paper's branches)."""
    rng = np.random.default_rng(3 + card)
    length, w = 256, 16
    L, U = _lu(card)
    for _ in range(50):
        q = rng.normal(0, 1, w)
        word = rng.integers(0, card, (1, w)).astype(np.uint8)
        T = oracle.lb_table(q, length, w, card)
        got = oracle.lb2(T, word)[0]
        proj = np.clip(q, L[word[0]], U[word[0]])
        ref = (length / w) * np.sum((q - proj) ** 2)
        assert got == pytest.approx(ref, rel=1e-13, abs=1e-13)
        # brute force: no sampled point of the (finite part of the) box is closer
        lo = np.maximum(L[word[0]], -6.0)
        hi = np.minimum(U[word[0]], 6.0)
        pts = rng.uniform(lo, hi, (400, w))
        assert np.all((length / w) * np.sum((q - pts) ** 2, axis=1) >= got - 1e-12)


@pytest.mark.parametrize("card", [2, 8, 64, 256])
def test_lb_lower_bounds_ed(card):
    """LB(q, SAX(x)) <= ED(q, x) for every pair: 200 x 50 pairs."""
    x = datagen.random_walks(200, 256, 21)
    qs = datagen.random_walks(50, 256, 22)
    sax = oracle.summarize(x, 16, card)
    qp = oracle.paa(qs, 16)
    for j in range(50):
        T = oracle.lb_table(qp[j], 256, 16, card)
        lb = oracle.lb2(T, sax)
        d2 = ((x.astype(np.float64) - qs[j].astype(np.float64)) ** 2).sum(axis=1)
        assert np.all(lb <= d2 * (1 + 1e-12))


def test_lb_monotone_in_cardinality():
    """Refining a segment never lowers the bound: card 2^b words are prefixes."""
    x = datagen.random_walks(300, 128, 31)
    q = datagen.random_walks(5, 128, 32)
    full = oracle.summarize(x, 16, 256)
    qp = oracle.paa(q, 16)
    for j in range(5):
        prev = None
        for b in range(1, 9):
            card = 1 << b
            words = (full >> (8 - b)).astype(np.uint8)
            lb = oracle.lb2(oracle.lb_table(qp[j], 128, 16, card), words)
            if prev is not None:
                assert np.all(lb >= prev - 1e-12)
            prev = lb


def test_lb_zero_for_own_word():
    x = datagen.random_walks(20, 256, 41)
    sax = oracle.summarize(x, 16, 256)
    qp = oracle.paa(x, 16)
    for i in range(20):
        T = oracle.lb_table(qp[i], 256, 16, 256)
        assert oracle.lb2(T, sax[i:i + 1])[0] == 0.0


# ---------------------------------------------------------------- distances
def test_ed2_matches_numpy_and_abandon():
    rng = np.random.default_rng(5)
    a = rng.normal(size=(100, 256)).astype(np.float32)
    b = rng.normal(size=(100, 256)).astype(np.float32)
    for i in range(100):
        ref = float(np.sum((a[i].astype(np.float64) - b[i].astype(np.float64)) ** 2))
        got = oracle.ed2(a[i], b[i])
        assert got == pytest.approx(ref, rel=1e-13)
        assert oracle.ed2_abandon(a[i], b[i], np.inf) == got
        lim = float(rng.uniform(0.5, 1.5) * ref)
        ab = oracle.ed2_abandon(a[i], b[i], lim)
        assert (ab > lim) == (ref > lim)  # classification agrees
        if ref <= lim:
            assert ab == got


# ---------------------------------------------------------------- k-NN
def _sorted_knn(x, q, k):
    d2 = ((x.astype(np.float64)[None] - q.astype(np.float64)[:, None]) ** 2).sum(-1)
    ids = np.stack([np.lexsort((np.arange(x.shape[0]), row))[:k] for row in d2])
    return ids, np.take_along_axis(d2, ids, 1)


@pytest.mark.parametrize("n,k", [(1, 1), (17, 1), (17, 5), (17, 17), (64, 10), (200, 100)])
def test_bruteforce_matches_full_sort(n, k):
    x = datagen.random_walks(n, 64, 100 + n)
    q = datagen.random_walks(4, 64, 200 + n)
    ids, d2 = oracle.knn_bruteforce(x, q, k)
    rid, rd2 = _sorted_knn(x, q, k)
    assert np.array_equal(ids, rid)
    assert np.allclose(d2, rd2, rtol=1e-13, atol=0)


@pytest.mark.parametrize("card", [2, 8, 64, 256])
def test_pruned_equals_bruteforce(card):
    n = 300
    x = datagen.random_walks(n, 128, 300 + card)
    x[50] = x[10]       # exact duplicates: ties resolved to the lower id
    x[51] = x[10]
    q = np.concatenate([datagen.random_walks(6, 128, 400 + card), x[[10, 77]]])
    sax = oracle.summarize(x, 16, card)
    for k in (1, 3, 10, n):
        st = np.zeros(3, np.int64)
        pid, pd2 = oracle.knn_pruned(x, sax, q, k, 16, card, st)
        bid, bd2 = oracle.knn_bruteforce(x, q, k)
        assert np.array_equal(pid, bid), (k, card)
        assert np.array_equal(pd2, bd2)
        assert st[0] == n * len(q) and st[1] <= st[0]
    # member queries: distance 0 at the lowest id of the duplicate group
    bid, bd2 = oracle.knn_bruteforce(x, x[[10, 77]], 3)
    assert list(bid[0]) == [10, 50, 51] and np.all(bd2[0] == 0)
    assert bid[1, 0] == 77 and bd2[1, 0] == 0


def test_pruned_actually_prunes():
    x = datagen.random_walks(3000, 256, 9)
    q = datagen.random_walks(3, 256, 10)
    sax = oracle.summarize(x, 16, 256)
    st = np.zeros(3, np.int64)
    oracle.knn_pruned(x, sax, q, 1, 16, 256, st)
    assert st[1] < 0.5 * st[0]  # LB prunes most series on random walks


def test_knn_rejects_bad_k():
    x = datagen.random_walks(5, 16, 1)
    with pytest.raises(ValueError):
        oracle.knn_bruteforce(x, x[:1], 6)
    with pytest.raises(ValueError):
        oracle.knn_bruteforce(x, x[:1], 0)
