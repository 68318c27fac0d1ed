"""Measured peaks beside MEASURED_PEAKS.json: the fp16x2 FMA pipe (paris_debug_hfma2_probe)
and the read-only HBM stream (paris_debug_read_probe).  Prints one JSON line."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2009_00166_b200 as P  # noqa: E402


def fma_peak(iters=20000, blocks=4, reps=5):
    P.debug_hfma2_probe(100, blocks)
    torch.cuda.synchronize()
    best = 0.0
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        ops = P.debug_hfma2_probe(iters, blocks)
        e1.record()
        torch.cuda.synchronize()
        best = max(best, ops / (e0.elapsed_time(e1) / 1e3) / 1e12)
    return best


if __name__ == "__main__":
    out = {"hfma2_tops": {b: fma_peak(blocks=b) for b in (1, 2, 4)}}
    x = torch.empty(8 << 30, dtype=torch.uint8, device="cuda")
    P.debug_read_probe(x)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(3):
        P.debug_read_probe(x)
    e1.record()
    torch.cuda.synchronize()
    out["read_gbs"] = 3 * x.numel() / (e0.elapsed_time(e1) / 1e3) / 1e9
    print(json.dumps(out))
