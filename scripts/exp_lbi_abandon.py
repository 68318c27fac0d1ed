"""Experiment (CPU, numpy): how early could the index LB pass abandon a live
(block, query) item?  For the live items of the f1 index (envelope bound <= tau^2),
the segment count after which every one of the block's 64 series already has a
partial MINDIST above tau^2 (partial sums are lower bounds: all terms >= 0).
tau = the exact 1-NN distance x `slack` (the seed is a little worse than ideal)."""
import sys
import time

import numpy as np

sys.path.insert(0, __import__("os").path.dirname(__file__) + "/..")
import datagen
import oracle

n = int(sys.argv[1]) if len(sys.argv) > 1 else 1_000_000
nq = 32
L, W, C = 256, 16, 256
slack = float(sys.argv[2]) if len(sys.argv) > 2 else 1.1
MODE = sys.argv[3] if len(sys.argv) > 3 else "seq"
t0 = time.time()
x = datagen.random_walks(n, L, 11)
q = datagen.random_walks(nq, L, 12)
sax = oracle.summarize(x, W, C).astype(np.int64)  # [n][w]
print(f"gen+sax {time.time() - t0:.1f}s", flush=True)
key = np.zeros(n, dtype=np.uint64)
for b in range(7, 3, -1):
    for s in range(W):
        key = (key << np.uint64(1)) | ((sax[:, s] >> b) & 1).astype(np.uint64)
order = np.lexsort((np.arange(n), key))
ss = sax[order]
nb = n // 64
ss = ss[:nb * 64].reshape(nb, 64, W)
mn, mx = ss.min(axis=1), ss.max(axis=1)
cuts = oracle.cuts(C)
Lr = np.r_[-np.inf, cuts]
Ur = np.r_[cuts, np.inf]
qp = oracle.paa(q, W)
xx = (x.astype(np.float64) ** 2).sum(1)
abandon_hist = np.zeros(W + 1)
items = 0
live_tot = 0
for j in range(nq):
    d2 = xx - 2 * x.astype(np.float64) @ q[j].astype(np.float64) + (q[j].astype(np.float64) ** 2).sum()
    tau2 = d2.min() * slack ** 2
    # per (symbol, segment) contribution (len/w) * dist(qpaa, region)^2
    cont = np.zeros((C, W))
    for s in range(W):
        v = qp[j, s]
        dl = np.maximum(Lr - v, 0)
        du = np.maximum(v - Ur, 0)
        cont[:, s] = (L / W) * np.maximum(dl, du) ** 2
    # envelope bound per block
    envd = np.zeros(nb)
    for s in range(W):
        v = qp[j, s]
        lo = Lr[mn[:, s]]
        hi = Ur[mx[:, s]]
        envd += (L / W) * np.maximum(np.maximum(lo - v, 0), np.maximum(v - hi, 0)) ** 2
    live = np.nonzero(envd <= tau2)[0]
    live_tot += len(live)
    c = cont[ss[live], np.arange(W)[None, None, :]]  # [nlive][64][w]
    if MODE == "absq":
        c = c[:, :, np.argsort(-np.abs(qp[j]))]
    elif MODE == "meanc":  # per item: segments by the block's mean contribution (oracle-ish)
        o = np.argsort(-c.mean(axis=1), axis=1)
        c = np.take_along_axis(c, o[:, None, :], axis=2)
    ps = np.cumsum(c, axis=2)
    allover = (ps > tau2).all(axis=1)  # [nlive][w]: every series above after s+1 segments
    first = np.where(allover.any(axis=1), allover.argmax(axis=1) + 1, W + 1)
    abandon_hist += np.bincount(np.minimum(first, W + 1) - 1, minlength=W + 1)[:W + 1]
    items += len(live)
print(f"live fraction {live_tot / (nq * nb):.4f}  items {items}")
cum = np.cumsum(abandon_hist) / items
for s in (2, 4, 6, 8, 10, 12, 14, 16):
    print(f"abandon by {s:2d} segments: {cum[s - 1]:.3f}")
# work with checks every 4 segments
work = 0.0
for i, cnt in enumerate(abandon_hist):
    s = i + 1
    done = W if s > W else min(W, ((s + 3) // 4) * 4)
    work += cnt * done
print(f"segment work with abandon checks every 4: {work / (items * W):.3f} of full")
