"""A/B of kernel variants (paris_debug_set_variant) inside one process on one box: the same
collection, index and queries; variants alternate over repetitions so drift and clock changes
hit both.  Prints per-variant median step time and lb_pass time, and checks the results agree.

python scripts/ab_variants.py --config 4 --key 0 --values 0 1 --reps 5
"""
import argparse
import json
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2009_00166_b200 as P  # noqa: E402
from datagen import gpu as dg  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=4)
    ap.add_argument("--key", type=int, default=0)
    ap.add_argument("--values", type=int, nargs="+", default=[0, 1])
    ap.add_argument("--reps", type=int, default=5)
    ap.add_argument("--k", type=int, default=1)
    ap.add_argument("--set", default=None, help="query set name (C5: noise0.2 ...)")
    args = ap.parse_args()
    raw, sets = dg.config_workload(args.config)
    name = args.set or list(sets)[0]
    queries = sets[name][0]
    sax = P.summarize(raw, 16, 256)
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    res = {v: {"step_ms": [], "lb_ms": [], "refine_ms": []} for v in args.values}
    outs = {}
    if args.key == 1:  # batch-1 flat LB
        q = queries[:8]
        cfg = P.KnnConfig(batch=1)
        run = lambda: P.knn_exact(raw, sax, q, k=args.k, config=cfg)  # noqa: E731
    else:
        index = P.index_build(sax, 16, 256)
        raw16 = P.raw_bf16(raw) if raw.shape[1] >= 128 else None
        paa16 = P.paa_f16(raw, 64 if raw.shape[1] % 64 == 0 else 32) if raw16 is not None else None
        cfg = P.KnnConfig(batch=64)
        call_q = 64 if args.config == 3 else queries.shape[0]

        def run():
            outs_i, outs_d = [], []
            for c0 in range(0, queries.shape[0], call_q):
                i, d = P.knn_index(raw, index, queries[c0:c0 + call_q], k=args.k, config=cfg, raw16=raw16,
                                   paa16=paa16)
                outs_i.append(i)
                outs_d.append(d)
            return torch.cat(outs_i), torch.cat(outs_d)
    for v in args.values:  # warm-up of every variant
        P.debug_set_variant(args.key, v)
        outs[v] = run()
    torch.cuda.synchronize()
    for _ in range(args.reps):
        for v in args.values:
            P.debug_set_variant(args.key, v)
            run()
            torch.cuda.synchronize()
            P.profile_reset()
            P.profile_enable(True)
            e0.record(st)
            run()
            e1.record(st)
            torch.cuda.synchronize()
            P.profile_enable(False)
            pr = P.profile_read()
            res[v]["step_ms"].append(e0.elapsed_time(e1))
            res[v]["lb_ms"].append(pr.get("lb_pass", (0, 0.0))[1])
            res[v]["refine_ms"].append(pr.get("refine", (0, 0.0))[1])
    i0, d0 = outs[args.values[0]]
    agree = all(torch.equal(outs[v][0], i0) and torch.equal(outs[v][1], d0) for v in args.values)
    summary = {"config": args.config, "set": name, "key": args.key, "k": args.k, "results_identical": agree}
    for v in args.values:
        summary[f"v{v}"] = {"step_ms_median": float(np.median(res[v]["step_ms"])),
                            "step_ms_min": float(np.min(res[v]["step_ms"])),
                            "lb_ms_median": float(np.median(res[v]["lb_ms"])),
                            "refine_ms_median": float(np.median(res[v]["refine_ms"])),
                            "lb_ms_all": [round(x, 4) for x in res[v]["lb_ms"]]}
    print(json.dumps(summary))


if __name__ == "__main__":
    main()
