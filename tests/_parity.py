"""Comparison rules for CUDA-path vs oracle parity (north_star tolerances).

- SAX: bit-exact, except a segment whose exact PAA lies within 1e-6 of a cut.
- k-NN: distances within 1e-5 relative of the oracle's; ids exact, except under
  ties, where the oracle distance of the returned id must be within 1e-5 relative
  of the oracle distance at that rank; ids within a row distinct.
"""
import numpy as np

import oracle

SAX_WINDOW = 1e-6
DIST_RTOL = 1e-5


def sax_mismatches(raw: np.ndarray, got_wn: np.ndarray, w: int, card: int):
    """Indices (series, segment) where the GPU symbol differs from the oracle's outside the window."""
    ref = oracle.summarize(raw, w, card)            # [n][w]
    got = np.asarray(got_wn).reshape(w, -1).T       # [n][w]
    paa = oracle.paa(raw, w)
    cuts = oracle.cuts(card)
    near = np.min(np.abs(paa[..., None] - cuts[None, None, :]), axis=-1) < SAX_WINDOW
    diff = got != ref
    return np.argwhere(diff & ~near), int(np.sum(diff & near)), ref


def check_knn(raw: np.ndarray, queries: np.ndarray, got_idx, got_dist, ref_idx, ref_d2, rows=None):
    """Assert the GPU k-NN rows match the oracle's (ref_idx/ref_d2 ascending, float64 d^2)."""
    got_idx = np.asarray(got_idx)
    got_dist = np.asarray(got_dist, dtype=np.float64)
    ref_d = np.sqrt(np.asarray(ref_d2, dtype=np.float64))
    rows = range(got_idx.shape[0]) if rows is None else rows
    for r in rows:
        gi, gd, ri, rd = got_idx[r], got_dist[r], ref_idx[r], ref_d[r]
        assert len(set(gi.tolist())) == len(gi), f"row {r}: duplicate ids {gi}"
        assert np.all(gi >= 0), f"row {r}: missing results {gi}"
        np.testing.assert_allclose(gd, rd, rtol=DIST_RTOL, atol=1e-6, err_msg=f"row {r} distances")
        for j in np.nonzero(gi != ri)[0]:
            d_alt = np.sqrt(oracle.ed2(raw[gi[j]], queries[r]))
            assert abs(d_alt - rd[j]) <= DIST_RTOL * max(rd[j], 1e-6), \
                f"row {r} rank {j}: id {gi[j]} (d={d_alt}) vs oracle id {ri[j]} (d={rd[j]})"
