"""Small cases of every kernel path, for compute-sanitizer (one tool per run)."""
import os, sys
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import numpy as np, torch
import __graft_entry__ as ge
ge.build()
import datagen
import paper_2009_00166_b200 as P

def run(n, length, nq, k, index, cfg=None, zero_q=False):
    x = datagen.random_walks(n, length, n + length)
    q = np.zeros((nq, length), np.float32) if zero_q else datagen.random_walks(nq, length, n + 1)
    xd, qd = torch.from_numpy(x).cuda(), torch.from_numpy(q).cuda()
    sax = P.summarize(xd, 16, 256)
    if index:
        idx = P.index_build(sax, 16, 256)
        r = P.knn_index(xd, idx, qd, k=k, config=cfg)
    else:
        r = P.knn_exact(xd, sax, qd, k=k, config=cfg)
    torch.cuda.synchronize()
    print("ok", n, length, nq, k, index, flush=True)

run(1000, 256, 3, 1, False)                       # direct LB kernels (n % 16 != 0)
run(4096 + 16, 256, 5, 3, False)                  # tiled, ragged tile
run(4096 + 16, 128, 17, 1, False)                 # tiled, len 128, two batches
run(6000 * 16 + 48, 256, 3, 10, True)             # index, ragged last tile, k > 1
run(40_000, 256, 33, 1, True)                     # index, two batches (32 + 1)
run(70_000, 128, 2, 1000, True, P.KnnConfig(index_seeds=1), zero_q=True)   # index overflow re-scan
run(70_000, 128, 2, 1000, False, P.KnnConfig(seed_div=70_000), zero_q=True)  # flat overflow re-scan
run(4096 + 48, 256, 40, 2, False)                 # flat behind the tensor-core filter (k_gf), sub-batches 16+16+8
P.debug_set_variant(3, 1)
run(6000 * 16 + 48, 256, 40, 1, True)             # index path through k_gf
P.debug_set_variant(3, 2)
print("all ok")
