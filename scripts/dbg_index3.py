import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
import datagen, oracle
import paper_2009_00166_b200 as P
n, nq = 40000, 2
x = datagen.random_walks(n, 256, 500 + n)
q = datagen.random_walks(5, 256, 501 + 5)[:nq]
q[0] = x[n // 3]
xd = torch.from_numpy(x).cuda(); qd = torch.from_numpy(q).cuda()
sax = P.summarize(xd, 16, 256)
idx = P.index_build(sax, 16, 256)
os.environ["PARIS_DEBUG_DUMP"] = str(n // 3)
print("member id", n // 3, flush=True)
gi, gd, st = P.knn_index(xd, idx, qd, k=10, stats=True)
print(gi.cpu().numpy(), gd.cpu().numpy(), st, flush=True)
