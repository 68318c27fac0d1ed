import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
import datagen, oracle
import paper_2009_00166_b200 as P
n, nq = 40000, 5
x = datagen.random_walks(n, 256, 500 + n)
q = datagen.random_walks(nq, 256, 501 + nq)
q[0] = x[n // 3]
xd = torch.from_numpy(x).cuda(); qd = torch.from_numpy(q).cuda()
sax = P.summarize(xd, 16, 256)
idx = P.index_build(sax, 16, 256)
for k in (1, 10):
    a = P.knn_exact(xd, sax, qd, k=k, stats=True)
    b = P.knn_index(xd, idx, qd, k=k, stats=True)
    print("k", k, "flat", a[2], "\nindex", b[2])
    print(a[1][:, :3].cpu().numpy(), "\n", b[1][:, :3].cpu().numpy())
# block LB check on host for query 0
env = idx.env.cpu().numpy(); perm = idx.perm.cpu().numpy()
pos = int(np.nonzero(perm == n // 3)[0][0])
print("member at sorted pos", pos, "block", pos // 128, "env", env[pos // 128])
print("member word", sax.cpu().numpy()[:, n // 3])
# oracle LB counts for query 0 against the index tau
saxo = oracle.summarize(x, 16, 256)
T = oracle.lb_table(oracle.paa(q[0:1], 16)[0], 256, 16, 256)
lb = oracle.lb2(T, saxo)
b = P.knn_index(xd, idx, qd[:1], k=10, stats=True)
tau = float(b[2]['tau_seed'][0])
print("q0 tau_idx", tau, "#LB<=tau^2", int((lb <= tau * tau * (1 + 1e-5)).sum()), "cand", b[2]['candidates'])
print("q0 alone k=10:", b[1].cpu().numpy())
b1 = P.knn_index(xd, idx, qd[:2], k=10, stats=True)
print("q0,q1 k=10:", b1[1].cpu().numpy()[:, :3], b1[2])
b3 = P.knn_index(xd, idx, qd[:3], k=10, stats=True)
print("q0..q2 k=10:", b3[1].cpu().numpy()[:, :3], b3[2])
