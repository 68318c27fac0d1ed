"""Per-call device times of the index search at a config (calls of 64 queries), each call bracketed
by CUDA events, repeated; reports the slowest calls with their batch index so a slow batch
(algorithmic) can be told from scattered slow calls (host or system jitter).
python scripts/exp_call_times.py --config 3 --variant 2=1 --reps 5"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_00166_b200 as P  # noqa: E402
from datagen import gpu as dg  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--variant", default="")
ap.add_argument("--reps", type=int, default=5)
args = ap.parse_args()
for kv in filter(None, args.variant.split(",")):
    k, v = kv.split("=")
    P.debug_set_variant(int(k), int(v))
raw, sets = dg.config_workload(args.config)
q = list(sets.values())[0][0]
sax = P.summarize(raw, 16, 256)
index = P.index_build(sax, 16, 256)
raw16 = P.raw_bf16(raw)
paa16 = P.paa_f16(raw, 64 if raw.shape[1] % 64 == 0 and raw.shape[1] >= 256 else 32)
cfg = P.KnnConfig(batch=64)
st = torch.cuda.current_stream()
nbat = (q.shape[0] + 63) // 64
times = np.zeros((args.reps, nbat))
for r in range(args.reps + 1):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(nbat + 1)]
    ev[0].record(st)
    for bi in range(nbat):
        P.knn_index(raw, index, q[bi * 64:(bi + 1) * 64], k=1, config=cfg, raw16=raw16, paa16=paa16)
        ev[bi + 1].record(st)
    torch.cuda.synchronize()
    if r == 0:
        continue
    for bi in range(nbat):
        times[r - 1, bi] = ev[bi].elapsed_time(ev[bi + 1])
med = np.median(times, axis=0)
worst = np.argsort(-times.ravel())[:8]
print(json.dumps({"variant": args.variant, "median_per_batch_ms": [round(x, 3) for x in med],
                  "total_ms_per_rep": [round(x, 3) for x in times.sum(1)],
                  "worst": [(int(i // nbat), int(i % nbat), round(float(times.ravel()[i]), 3)) for i in worst]}))
