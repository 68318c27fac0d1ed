import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
import datagen, oracle
import paper_2009_00166_b200 as P
n, nq = 40960, 3
x = datagen.random_walks(n, 256, 500 + n)
q = datagen.random_walks(nq, 256, 501 + nq)
q[0] = x[n // 3]
xd = torch.from_numpy(x).cuda(); qd = torch.from_numpy(q).cuda()
sax = P.summarize(xd, 16, 256)
# identity "index": unsorted SAX, perm = arange, envelopes of the unsorted blocks
s = sax.cpu().numpy().T.reshape(-1, 128, 16)
env = torch.from_numpy(np.stack([s.min(1), s.max(1)], 1).copy()).cuda()
ident = P.Index(sax, torch.arange(n, dtype=torch.int32, device="cuda"), env, 16, 256)
full = torch.from_numpy(np.stack([np.zeros((n // 128, 16), np.uint8), np.full((n // 128, 16), 255, np.uint8)], 1)).cuda()
ident_full = P.Index(sax, torch.arange(n, dtype=torch.int32, device="cuda"), full, 16, 256)
ri, rd2 = oracle.knn_bruteforce(x, q, 10)
print("truth", np.sqrt(rd2[:, :3]))
for name, ix in (("ident", ident), ("ident_fullenv", ident_full)):
    gi, gd, st = P.knn_index(xd, ix, qd, k=10, stats=True)
    print(name, gd.cpu().numpy()[:, :3], st)
gi, gd, st = P.knn_exact(xd, sax, qd, k=10, stats=True)
print("flat", gd.cpu().numpy()[:, :3], st)
