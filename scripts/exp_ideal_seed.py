"""How much LB work would an ideal seed save?  knn_index normally, then again seeded with its
own answer (the true NN distance): lb_blocks, candidates and time for both."""
import os, sys, json
sys.path.insert(0, os.environ.get("GRAFT_REPO_ROOT", "."))
import torch
import paper_2009_00166_b200 as P
from datagen import gpu as dg
import datagen
n = int(os.environ.get("EXP_N", 100_000_000)); L = 256
ds, qs = datagen.config_seeds(4)
raw = dg.walks(n, L, ds); q = dg.walks(100, L, qs)
sax = P.summarize(raw, 16, 256); idx = P.index_build(sax, 16, 256)
oi = torch.empty((100, 1), dtype=torch.int64, device="cuda"); od = torch.empty((100, 1), device="cuda")
def run(cfg):
    for _ in range(2): P.knn_index(raw, idx, q, out_idx=oi, out_dist=od, config=cfg)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    P.profile_reset(); P.profile_enable(True)
    e0.record()
    _, _, st = P.knn_index(raw, idx, q, out_idx=oi, out_dist=od, config=cfg, stats=True)
    e1.record(); torch.cuda.synchronize(); P.profile_enable(False)
    return e0.elapsed_time(e1), {k: round(v[1], 3) for k, v in P.profile_read().items()}, \
        float(st["lb_blocks"].double().mean()) / (n / 128), float(st["candidates"].double().mean()), float(st["refined"].double().mean())
print(json.dumps({"normal": run(P.KnnConfig()), "ideal_seed": run(P.KnnConfig(seed_from_out=True))}))
