"""Tuning experiment: block-mask statistics of the C4 index LB pass (PARIS_DEBUG_BMASK) for the
query batch in its generated order and sorted by the queries' own iSAX keys (similar queries in
adjacent slots): live (block, slot) bits, arbitrary-pair items, fixed-pair and fixed-quad items."""
import json
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_00166_b200 as P  # noqa: E402
from datagen import gpu as dg  # noqa: E402

out = sys.argv[1] if len(sys.argv) > 1 else "bmask.jsonl"
raw, sets = dg.config_workload(4)
q = sets["fresh"][0]
sax = P.summarize(raw, 16, 256)
index = P.index_build(sax, 16, 256)
qsax = P.summarize(q.contiguous(), 16, 256)   # [16][nq] segment-major
key = torch.zeros(q.shape[0], dtype=torch.int64, device=q.device)
for b in range(7, 3, -1):
    for s in range(16):
        key = (key << 1) | ((qsax[s].to(torch.int64) >> b) & 1)
orders = {"generated": torch.arange(q.shape[0], device=q.device), "isax_key": torch.argsort(key),
          "paa_mean_slope": torch.argsort(q[:, q.shape[1] // 2:].mean(1) - q[:, :q.shape[1] // 2].mean(1))}
for name, o in orders.items():
    os.environ["PARIS_DEBUG_BMASK"] = out
    with open(out, "a") as f:
        f.write(json.dumps({"order": name}) + "\n")
    P.knn_index(raw, index, q[o].contiguous(), k=1, config=P.KnnConfig(batch=64))
    torch.cuda.synchronize()
print(open(out).read())
