"""Experiment (CPU, numpy): fraction of (64-series block, query) pairs whose envelope
MINDIST passes tau^2 (live pairs the index LB pass must evaluate) for different
series orders: the iSAX interleaved-bit key (f1 as built) vs keys built from a
PCA projection of the SAX words (Morton order over the top-d components)."""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import datagen
import oracle

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nq, L, W, C = int(__import__("os").environ.get("NQ", "32")), 256, 16, 256
slack = 1.1
x = datagen.random_walks(n, L, 11)
q = datagen.random_walks(nq, L, 12)
sax = oracle.summarize(x, W, C).astype(np.int64)
cuts = oracle.cuts(C)
Lr = np.r_[-np.inf, cuts]
Ur = np.r_[cuts, np.inf]
qp = oracle.paa(q, W)
xf = x.astype(np.float64)
xx = (xf ** 2).sum(1)
tau2 = np.array([(xx - 2 * xf @ q[j].astype(np.float64) + (q[j].astype(np.float64) ** 2).sum()).min()
                 for j in range(nq)]) * slack ** 2


def live_frac(order, B=64):
    ss = sax[order]
    nb = n // B
    ss = ss[:nb * B].reshape(nb, B, W)
    mn, mx = ss.min(axis=1), ss.max(axis=1)
    tot = 0
    for j in range(nq):
        envd = np.zeros(nb)
        for s in range(W):
            v = qp[j, s]
            envd += (L / W) * np.maximum(np.maximum(Lr[mn[:, s]] - v, 0), np.maximum(v - Ur[mx[:, s]], 0)) ** 2
        tot += (envd <= tau2[j]).sum()
    return tot / (nq * nb)


def morton(cols, bits):
    key = np.zeros(n, dtype=np.uint64)
    for b in range(bits - 1, -1, -1):
        for c in cols:
            key = (key << np.uint64(1)) | ((c >> b) & 1).astype(np.uint64)
    return key


isax = morton([sax[:, s] for s in range(W)], 8)
isax = np.zeros(n, dtype=np.uint64)
for b in range(7, 3, -1):
    for s in range(W):
        isax = (isax << np.uint64(1)) | ((sax[:, s] >> b) & 1).astype(np.uint64)
print("isax key       ", round(live_frac(np.lexsort((np.arange(n), isax))), 4), flush=True)
mid = np.r_[cuts[0] - 0.1, (cuts[:-1] + cuts[1:]) / 2, cuts[-1] + 0.1][sax]  # region midpoints
mu = mid.mean(0)
U, S, Vt = np.linalg.svd(mid[:200000] - mu, full_matrices=False)
print("pca energy", np.round(S[:8] ** 2 / (S ** 2).sum(), 3))
for d in ():
    proj = (mid - mu) @ Vt[:d].T
    bits = max(4, 64 // d)
    cols = []
    for c in range(d):
        r = np.argsort(np.argsort(proj[:, c]))  # rank -> uniform quantiles
        cols.append((r * (1 << bits) // n).astype(np.int64))
    key = morton(cols, bits)
    print(f"pca d={d} bits={bits}", round(live_frac(np.lexsort((np.arange(n), key))), 4), flush=True)
o = np.lexsort((np.arange(n), isax))
for B in (16, 32):
    print(f"isax B={B}", round(live_frac(o, B), 4), flush=True)
# key with more bits: bits 7..3 (5 levels) -> 80 bits; approximate by lexsort on two words
hi = isax
lo = np.zeros(n, dtype=np.uint64)
for s in range(W):
    lo = (lo << np.uint64(1)) | ((sax[:, s] >> 3) & 1).astype(np.uint64)
o2 = np.lexsort((np.arange(n), lo, hi))
if n <= 2_000_000:
    print("isax 5 levels B=64", round(live_frac(o2, 64), 4))
