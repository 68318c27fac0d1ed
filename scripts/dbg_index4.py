import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
import datagen, oracle
import paper_2009_00166_b200 as P
n = 100_000 - 96   # n % 16 == 0, ragged last tile
x = datagen.random_walks(n, 128, 41)
q = datagen.random_walks(3, 128, 42) * 0.0
xd = torch.from_numpy(x).cuda(); qd = torch.from_numpy(q).cuda()
sax = P.summarize(xd, 16, 256)
idx = P.index_build(sax, 16, 256)
gi, gd, st = P.knn_index(xd, idx, qd, k=1000, config=P.KnnConfig(index_seeds=1), stats=True)
torch.cuda.synchronize()
print("ok", st)
ri, rd2 = oracle.knn_bruteforce(x, q, 1000)
print(np.abs(gd.cpu().numpy() - np.sqrt(rd2)).max())
