"""Small profiling driver: summarize + one 16-query and one 1-query knn pass (n beyond L2)."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import paper_2009_00166_b200 as P
from datagen import gpu as dg
n = int(os.environ.get("PROF_N", 20_000_000))
length = int(os.environ.get("PROF_LEN", 256))
dev = torch.device("cuda:0")
raw = dg.walks(n, length, 200900164, device=dev)
q = dg.walks(16, length, 200901164, device=dev)
sax = P.summarize(raw, 16, 256)
torch.cuda.synchronize()
i16, d16 = P.knn_exact(raw, sax, q, k=1, config=P.KnnConfig(batch=16))
i1, d1 = P.knn_exact(raw, sax, q[:1], k=1, config=P.KnnConfig(batch=1))
torch.cuda.synchronize()
assert int(i16[0, 0]) == int(i1[0, 0])
print("ok", i16[:4, 0].tolist())
if os.environ.get("PROF_K10"):
    i10, d10 = P.knn_exact(raw, sax, q, k=10, config=P.KnnConfig(batch=16))
    torch.cuda.synchronize()
    print("k10 ok", i10[0, :3].tolist())
