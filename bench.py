#!/usr/bin/env python
"""Benchmark: ParIS+ exact 1-NN queries/s on B200 (BASELINE.json metric, config 4 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

One step = one paris_knn_exact call answering the config's whole query batch (rows
a3-a8 of SURVEY §8: query PAA, BSF seed, LB pass, candidate order, refinement,
finalize) over a device-resident collection + SAX array.  Summarization (rows a1-a2)
is timed in the same run as its own line item ("summarize").  Inputs are larger than
L2 (config 4: SAX 1.6 GB, raw 102.4 GB vs 126 MB L2), so no flush is needed.

Multi-GPU (torchrun): weak scaling -- every rank holds its own collection of the
config's size and answers its own queries (queries are independent problems); no
data-path collective; the only NCCL calls are the timing barrier/max.
--impl reference: the CPU oracle (oracle/, single thread) timed on a bounded sample of
the same workload, scaled to queries/s over the full collection.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

CONFIGS = {
    1: dict(n=100_000, len=256, nq=100, k=1, queries="fresh", desc="C1: 1e5 x 256 fp32 RW, 100 fresh RW queries, exact 1-NN"),
    2: dict(n=1_000_000, len=256, nq=1000, k=1, queries="noise0.05", desc="C2: 1e6 x 256 fp32 RW, 1000 member+N(0,0.05^2) queries, exact 1-NN (line); 'sweep': k = 10"),
    3: dict(n=10_000_000, len=128, nq=1000, k=1, queries="fresh", call=64, desc="C3: 1e7 x 128 fp32 RW, 1000 fresh RW queries in calls of 64, exact 1-NN"),
    4: dict(n=100_000_000, len=256, nq=100, k=1, queries="fresh", desc="C4: 1e8 x 256 fp32 RW (102.4 GB raw + 1.6 GB SAX in HBM), 100 fresh RW queries, exact 1-NN"),
    5: dict(n=20_000_000, len=256, nq=200, k=1, queries="noise0.05", desc="C5: 2e7 x 256 fp32 RW, 200 member+N(0,0.05^2) queries, exact 1-NN (line); 'sweep': 5 sets x 200 queries, sigma in {0.01..0.2}, k = 1 and 100"),
}
W, CARD = 16, 256
ALU_CLOCK_GHZ = 1.965  # B200 clocks.max.sm (B200_PROFILING.md)


def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """nvidia-smi clocks + throttle reasons sampled every 200 ms while running."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._t = threading.Thread(target=self._run, daemon=True)

    def _run(self):
        while not self._stop.is_set():
            try:
                out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                      "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                     timeout=5).stdout.strip()
                if out:
                    self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows)}


def rank_seeds(config: int, rank: int):
    """(dataset seed, query seed) of a rank: weak scaling -- every rank owns a distinct
    collection and query set of the config's size (queries are independent problems)."""
    import datagen
    ds, qs = datagen.config_seeds(config)
    return ds + 7919 * rank, qs + 7919 * rank


def reduce_max_ms(ms: float, device, world_size: int) -> float:
    """Max over ranks of a device-timed duration (the slowest rank defines the step)."""
    import torch
    t = torch.tensor([float(ms)], dtype=torch.float64, device=device)
    if world_size > 1:
        import torch.distributed as dist
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def weak_throughput(nq_per_rank: int, world_size: int, max_ms: float) -> float:
    """Whole-job queries/s: every rank answered nq_per_rank queries within max_ms."""
    return nq_per_rank * world_size / (max_ms / 1e3)


def seed_series(n: int, use_index: bool, index_seeds: int, k: int) -> int:
    """Series whose true distance the BSF seed computes per query (plan_seed in csrc/knn.cu):
    index path -- the index_seeds (default 1024) series around the query's leaf; flat path --
    the LB-best series of each of 16 warps x seed_grid CTAs over a prefix sample of n/16."""
    if use_index:
        return max(k, min(4096, index_seeds or 1024))
    ns = min(n, max(n // 16, min(n, 65536)))
    ns = min(n, (ns + 15) // 16 * 16)
    return min(148, (ns + 2047) // 2048) * 16


def refined_sum_of(stats) -> float:
    return float(stats["refined"].double().sum())


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy R+W)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str, config: int):
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    return d.get(f"C{config}", {}).get(kernel)


# --------------------------------------------------------------------------- CPU oracle arm
def oracle_sample(raw_dev, queries_dev, k, n_sample, nq_sample):
    """Time the oracle's LB-pruned exact search (its own SAX) on the first n_sample series
    for nq_sample queries; returns (seconds per query on the sample, threads)."""
    import numpy as np
    import oracle
    x = raw_dev[:n_sample].cpu().numpy()
    q = queries_dev[:nq_sample].cpu().numpy()
    sax = oracle.summarize(x, W, CARD)
    t0 = time.perf_counter()
    oracle.knn_pruned(x, sax, q, k, W, CARD)
    dt = time.perf_counter() - t0
    del x, sax
    _ = np
    return dt / nq_sample


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch
    from datagen import gpu as dg
    cfg = CONFIGS[args.config]
    n, length, nq, k = cfg["n"], cfg["len"], cfg["nq"], cfg["k"]
    dev = torch.device("cuda:0") if torch.cuda.is_available() else None
    n_sample = min(n, args.ref_sample)
    log(f"reference arm: oracle on {n_sample} of {n} series")
    if dev is not None:
        ds, qs = __import__("datagen").config_seeds(args.config)
        raw = dg.walks(n_sample, length, ds, device=dev)
        queries = dg.walks(max(2, args.ref_queries), length, qs, device=dev)
    else:
        import datagen
        ds, qs = datagen.config_seeds(args.config)
        raw = torch.from_numpy(datagen.random_walks(n_sample, length, ds))
        queries = torch.from_numpy(datagen.random_walks(max(2, args.ref_queries), length, qs))
    per_q = []
    for i in range(args.warmup + args.steps):
        t = oracle_sample(raw, queries, k, n_sample, args.ref_queries)
        if i >= args.warmup:
            per_q.append(t * (n / n_sample))  # scaled to the full collection (linear in n)
    sec_per_query = statistics.mean(per_q)
    value = 1.0 / sec_per_query
    sample = (f"oracle_knn_pruned (single thread, fp64) over the first {n_sample} series of {cfg['desc']}, "
              f"{args.ref_queries} queries per step, time scaled x{n / n_sample:.0f} to n={n}")
    line = {"impl": "reference", "metric": "exact 1-NN queries/sec", "value": value, "unit": "queries/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec_per_query * nq * 1e3, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": cfg["desc"], "n": n, "len": length, "w": W, "card": CARD, "nq": nq, "k": k},
            "cpu_baseline": {"value": value, "unit": "queries/s", "cores": 1, "kind": "oracle", "sample": sample},
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2009_00166_b200 as P
    from datagen import gpu as dg
    import datagen

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = CONFIGS[args.config]
    n, length, nq, k = cfg["n"], cfg["len"], cfg["nq"], cfg["k"]
    if args.n:
        n = args.n
    if args.nq:
        nq = args.nq
    call_q = cfg.get("call", nq)  # queries per paris_knn_exact call (C3: batches of 64)
    ds, qs = rank_seeds(args.config, rank)

    t0 = time.time()
    raw = dg.walks(n, length, ds, device=dev)
    if cfg["queries"] == "fresh":
        queries = dg.walks(nq, length, qs, device=dev)
    else:
        queries, _ = dg.noisy_members(raw, nq, float(cfg["queries"][5:]), qs)
    sax = torch.empty((W, n), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    log(f"rank {rank}: generated n={n} len={length} nq={nq} in {time.time() - t0:.1f}s")
    h2d_gbs = None
    # the bf16 copy of raw for the index path's refinement pre-filter (paris_raw_bf16), built once
    raw16, raw16_ms = None, None
    if not args.no_raw16 and (args.path == "index" or args.both):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        raw16 = P.raw_bf16(raw)
        e1.record()
        torch.cuda.synchronize()
        raw16_ms = e0.elapsed_time(e1)
    if args.raw_host:
        # f3: the raw collection lives in pinned host memory (not in HBM); summarize streams
        # it through the double-buffered H2D pipeline, the refinement reads candidates' rows
        # through the host mapping.  Only SAX (+ index) stays in HBM.
        t1 = time.time()
        raw_h = torch.empty((n, length), dtype=torch.float32, pin_memory=True)
        step_rows = 1 << 20
        for r0 in range(0, n, step_rows):
            raw_h[r0:r0 + step_rows].copy_(raw[r0:r0 + step_rows])
        torch.cuda.synchronize()
        del raw
        torch.cuda.empty_cache()
        raw = raw_h
        # the PCIe roofline: a plain pinned -> device copy of 1 GB (cudaMemcpyAsync)
        tmp = torch.empty(1 << 28, dtype=torch.float32, device=dev)
        src = raw.view(-1)[:1 << 28]
        tmp.copy_(src, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            tmp.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d_gbs = 3 * 4.0 * (1 << 28) / (e0.elapsed_time(e1) / 1e3) / 1e9
        del tmp
        log(f"rank {rank}: raw moved to pinned host memory in {time.time() - t1:.1f}s; H2D copy {h2d_gbs:.1f} GB/s")
    st = torch.cuda.current_stream()

    # ---- summarize (rows a1-a2): warmup + timed
    for _ in range(args.warmup):
        P.summarize(raw, W, CARD, out=sax)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        P.summarize(raw, W, CARD, out=sax)
    e1.record(st)
    torch.cuda.synchronize()
    sum_ms = e0.elapsed_time(e1) / args.steps

    # ---- index (f1): iSAX-ordered SAX + block envelopes, built once (timed on its own)
    index = None
    index_ms = None
    if args.path == "index" or args.both:
        index = P.index_build(sax, W, CARD)
        torch.cuda.synchronize()
        e0.record(st)
        index = P.index_build(sax, W, CARD)
        e1.record(st)
        torch.cuda.synchronize()
        index_ms = e0.elapsed_time(e1)
    peak, peak_src = measured_peaks()
    # read-only streaming peak: the library's 16-byte read probe over >= 8 GB
    read_peak = None
    if not args.raw_host:
        probe = raw if raw.numel() * 4 >= (8 << 30) else torch.empty(8 << 30, dtype=torch.uint8, device=dev)
        P.debug_read_probe(probe)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            P.debug_read_probe(probe)
        e1.record()
        torch.cuda.synchronize()
        read_peak = 3.0 * probe.numel() * probe.element_size() / (e0.elapsed_time(e1) / 1e3) / 1e9
        del probe

    def measure_path(path: str, full: bool):
        """Warm up, time K steps of `path` (device events, max over ranks), then the same K
        steps with per-launch events for the kernel split and the roofline; with full=True
        also the end-to-end variant through host buffers and the clock record."""
        use_index = path == "index"
        use_nb = path == "nb"
        b_path = args.batch or (64 if use_index else 16)  # the library's default queries per pass
        kcfg = P.KnnConfig(batch=b_path, index_seeds=args.index_seeds, sorted_refine=args.sorted_refine)
        nbatches = sum((min(call_q, nq - c0) + b_path - 1) // b_path for c0 in range(0, nq, call_q))
        q_per_pass = nq / nbatches

        def knn(qsrc, **kw):
            if use_index:
                return P.knn_index(raw, index, qsrc, k=k, raw16=raw16, **kw)
            if use_nb:
                return P.knn_nb(raw, sax, qsrc, w=W, card=CARD, **kw)
            return P.knn_exact(raw, sax, qsrc, k=k, w=W, card=CARD, **kw)

        out_idx = torch.empty((nq, k), dtype=torch.int64, device=dev)
        out_dist = torch.empty((nq, k), dtype=torch.float32, device=dev)

        def step(qsrc, oi, od, cfg_=None):
            cfg_ = cfg_ or kcfg
            for c0 in range(0, nq, call_q):
                c1 = min(nq, c0 + call_q)
                knn(qsrc[c0:c1], out_idx=oi[c0:c1], out_dist=od[c0:c1], config=cfg_)

        _, _, stats = knn(queries, out_idx=out_idx, out_dist=out_dist, config=kcfg, stats=True)
        for _ in range(max(0, args.warmup - 1)):
            step(queries, out_idx, out_dist)
        torch.cuda.synchronize()
        r = {"path": path, "stats": stats, "knn": knn, "out_idx": out_idx}
        # timed region
        launches0 = P.launch_count()
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clocks:
            e0.record(st)
            for _ in range(args.steps):
                step(queries, out_idx, out_dist)
            e1.record(st)
            torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        r["launches"] = P.launch_count() - launches0
        r["clocks"] = clocks.summary()
        r["step_ms"] = reduce_max_ms(e0.elapsed_time(e1) / args.steps, dev, ws)
        r["value"] = weak_throughput(nq, ws, r["step_ms"])
        # the same K steps with libparis' per-launch CUDA events (launching stream)
        P.profile_reset()
        P.profile_enable(True)
        for _ in range(args.steps):
            step(queries, out_idx, out_dist)
        torch.cuda.synchronize()
        P.profile_enable(False)
        prof = P.profile_read()
        if full:
            # e2e through the same ABI calls with HOST (pinned) buffers
            hq = queries.cpu().pin_memory()
            hidx = torch.empty((nq, k), dtype=torch.int64).pin_memory()
            hdist = torch.empty((nq, k), dtype=torch.float32).pin_memory()
            step(hq, hidx, hdist)
            torch.cuda.synchronize()
            e0.record(st)
            for _ in range(args.steps):
                step(hq, hidx, hdist)
            e1.record(st)
            torch.cuda.synchronize()
            r["e2e_value"] = weak_throughput(nq, ws, reduce_max_ms(e0.elapsed_time(e1) / args.steps, dev, ws))
            assert torch.equal(hidx, out_idx.cpu()), "host-buffer path disagrees with device path"
        cand = stats["candidates"].numpy().astype(np.float64)
        refined = stats["refined"].numpy().astype(np.float64)
        kern = {}
        for name, (cnt, ms) in prof.items():
            kern[name] = {"launches": cnt, "ms_per_step": ms / args.steps, "share": None}
        tot = sum(v["ms_per_step"] for v in kern.values()) or 1.0
        for v in kern.values():
            v["share"] = v["ms_per_step"] / tot
        alg = {
            # SAX bytes per pass + 8 B per candidate written
            "lb_pass": (nbatches * n * W + 8.0 * cand.sum()) / nbatches,
            # raw bytes per refined series (K6): fp32 rows + the bf16 rows of the pre-filter
            "refine": (4.0 * length * refined.sum()
                       + 2.0 * length * stats["raw16_rows"].numpy().astype(np.float64).sum()) / nbatches,
            # nb-ParIS+ workers: the SAX array + the raw series they read
            "nb_distcomp": (nbatches * n * W + 4.0 * length * refined.sum()) / nbatches,
        }
        # per-batch algorithmic amounts against the kernel's device time per batch (the k = 1
        # refine is two launches per batch -- two LB-ordered waves -- so time is summed per batch)
        for name, v in kern.items():
            v["launch_ms"] = v["ms_per_step"] * args.steps / prof[name][0]
            v["ms_per_batch"] = v["ms_per_step"] / nbatches
            if name in alg:
                v["achieved_gbs"] = alg[name] / (v["ms_per_batch"] / 1e3) / 1e9
        dom = max(kern, key=lambda s_: kern[s_]["ms_per_step"]) if kern else None
        roof = None
        if dom:
            per_launch_ms = kern[dom]["ms_per_batch"]
            pk = 148 * 64 * 2 * ALU_CLOCK_GHZ * 1e9 / 1e12
            alu_src = f"derived: 148 SM x 64 FMA lanes/clk x 2 (f16x2) x {ALU_CLOCK_GHZ} GHz"
            if dom == "lb_pass" and use_index:
                # index path: the algorithmic work is the (block, query) pairs whose envelope
                # bound passed (stats lb_blocks) x PARIS_INDEX_BLOCK series x w segments x 3 FMA-pipe half-ops
                blocks = stats["lb_blocks"].numpy().astype(np.float64).sum()
                ops = 3.0 * W * P.PARIS_INDEX_BLOCK * blocks / nbatches
                ach = ops / (per_launch_ms / 1e3) / 1e12
                roof = {"kernel": dom, "bound": "alu", "achieved": ach, "peak": pk,
                        "unit": "Tops/s (fp16x2 half-ops)", "frac": ach / pk,
                        "traffic": ncu_traffic(dom + "_index", args.config),
                        "algorithmic_ops_per_batch": ops, "ms_per_batch": per_launch_ms, "peak_source": alu_src,
                        "active_block_frac": blocks / (nq * (n / P.PARIS_INDEX_BLOCK)),
                        "hbm_achieved_gbs": alg[dom] / (per_launch_ms / 1e3) / 1e9, "hbm_peak_gbs": peak,
                        "queries_per_pass": q_per_pass}
            elif dom == "lb_pass" and q_per_pass > 1.5:
                # batched fp16x2 LB: bound by the FMA pipe, not HBM: 3 half-precision
                # FMA-pipe ops per (series, segment, query)
                ops = 3.0 * n * W * q_per_pass
                ach = ops / (per_launch_ms / 1e3) / 1e12
                roof = {"kernel": dom, "bound": "alu", "achieved": ach, "peak": pk,
                        "unit": "Tops/s (fp16x2 half-ops)", "frac": ach / pk,
                        "traffic": ncu_traffic(dom, args.config),
                        "algorithmic_ops_per_batch": ops, "ms_per_batch": per_launch_ms, "peak_source": alu_src,
                        "hbm_achieved_gbs": alg[dom] / (per_launch_ms / 1e3) / 1e9, "hbm_peak_gbs": peak,
                        "queries_per_pass": q_per_pass}
            elif args.raw_host and dom in ("refine", "nb_distcomp", "seed_ed"):
                # f3: the seeds' and candidates' raw rows cross PCIe (zero-copy reads of pinned host memory)
                if dom == "seed_ed":
                    byts = 4.0 * length * seed_series(n, use_index, args.index_seeds, k) * q_per_pass
                else:
                    byts = 4.0 * length * refined_sum_of(stats) / nbatches
                ach = byts / (per_launch_ms / 1e3) / 1e9
                roof = {"kernel": dom, "bound": "pcie", "achieved": ach, "peak": h2d_gbs, "unit": "GB/s",
                        "frac": ach / h2d_gbs, "traffic": None, "algorithmic_bytes_per_batch": byts,
                        "ms_per_batch": per_launch_ms,
                        "peak_source": "measured in this run: pinned host -> device cudaMemcpyAsync, 1 GB x3"}
            elif dom in alg:
                ach = alg[dom] / (per_launch_ms / 1e3) / 1e9
                roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                        "frac": ach / peak, "traffic": ncu_traffic(dom + ("_index" if use_index else ""), args.config),
                        "algorithmic_bytes_per_batch": alg[dom], "ms_per_batch": per_launch_ms,
                        "peak_source": peak_src}
        r.update(kern=kern, roof=roof, cand=cand, refined=refined, batch=b_path)
        if use_nb:
            r["bsf_updates_mean"] = float(stats["bsf_updates"].numpy().astype(np.float64).mean())
        return r

    primary = measure_path(args.path, True)
    secondary = None
    if args.both:
        secondary = measure_path("flat" if args.path in ("index", "nb") else "index", False)

    def timed_index(qsrc, kk):
        """q/s and pruning of the index path on a query set (events, max over ranks)."""
        kc = P.KnnConfig(batch=args.batch or 64, index_seeds=args.index_seeds)
        _, _, stq = P.knn_index(raw, index, qsrc, k=kk, config=kc, stats=True, raw16=raw16)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            for c0 in range(0, qsrc.shape[0], call_q):
                P.knn_index(raw, index, qsrc[c0:c0 + call_q], k=kk, config=kc, raw16=raw16)
        e1.record(st)
        torch.cuda.synchronize()
        ms = reduce_max_ms(e0.elapsed_time(e1) / args.steps, dev, ws)
        ref = stq["refined"].numpy().astype(np.float64)
        return {"k": kk, "queries": int(qsrc.shape[0]), "value": weak_throughput(int(qsrc.shape[0]), ws, ms),
                "unit": "queries/s", "ms_per_step": ms,
                "candidates_mean": float(stq["candidates"].numpy().astype(np.float64).mean()),
                "refined_mean": float(ref.mean()), "pruning_ratio": float(1.0 - ref.mean() / n),
                "raw16_rows_mean": float(stq["raw16_rows"].numpy().astype(np.float64).mean())}

    sweep = None
    if index is not None and not args.no_sweep and not args.raw_host:
        if args.config == 2:  # BASELINE config 2: exact 1-NN and k = 10
            sweep = [dict(timed_index(queries, 10), sigma=0.05)]
        elif args.config == 5:  # config 5: 5 sets x 200 member + N(0, sigma^2) queries, k = 1 and 100
            sweep = []
            for si, sig in enumerate((0.01, 0.02, 0.05, 0.1, 0.2)):
                qset, _ = dg.noisy_members(raw, nq, sig, qs + 101 * (si + 1))
                for kk in (1, 100):
                    sweep.append(dict(timed_index(qset, kk), sigma=sig))

    def knn_flat(qsrc, **kw):
        return P.knn_exact(raw, sax, qsrc, k=k, w=W, card=CARD, **kw)
    stats, kern, roof = primary["stats"], primary["kern"], primary["roof"]
    cand, refined = primary["cand"], primary["refined"]
    value, step_ms_max, launches, clocks = primary["value"], primary["step_ms"], primary["launches"], primary["clocks"]
    e2e_value = primary["e2e_value"]

    # ---- flat LB pass at one query per SAX read: the HBM-roofline configuration of K4 (SURVEY §7 hard part 1)
    lb1 = None
    if not args.no_b1:
        nq1 = min(nq, 8)
        cfg1 = P.KnnConfig(batch=1)
        knn_flat(queries[:nq1], config=cfg1)
        torch.cuda.synchronize()
        P.profile_reset()
        P.profile_enable(True)
        _, _, st1 = knn_flat(queries[:nq1], config=cfg1, stats=True)
        P.profile_enable(False)
        pr1 = P.profile_read()
        if "lb_pass" in pr1:
            c1, ms1 = pr1["lb_pass"]
            by1 = n * W + 8.0 * float(st1["candidates"].double().mean())
            a1 = by1 / (ms1 / c1 / 1e3) / 1e9
            lb1 = {"kernel": "lb_pass", "bound": "hbm", "queries_per_pass": 1, "launch_ms": ms1 / c1,
                   "algorithmic_bytes_per_launch": by1, "achieved": a1, "peak": peak, "unit": "GB/s",
                   "frac": a1 / peak, "queries": nq1}
        if "refine" in pr1:
            c1, ms1 = pr1["refine"]  # two launches (waves) per query
            by1 = 4.0 * length * float(st1["refined"].double().mean())
            lb1 = lb1 or {}
            lb1["refine_batch1"] = {"ms_per_query": ms1 / nq1, "algorithmic_bytes_per_query": by1,
                                    "achieved": by1 / (ms1 / nq1 / 1e3) / 1e9, "peak": peak, "unit": "GB/s"}
    sum_bytes = n * (4.0 * length + W)
    summarize = {"series_per_s": n / (sum_ms / 1e3), "ms": sum_ms, "unit": "series/s",
                 "roofline": {"kernel": "summarize", "bound": "hbm", "achieved": sum_bytes / (sum_ms / 1e3) / 1e9,
                              "peak": peak, "unit": "GB/s", "frac": sum_bytes / (sum_ms / 1e3) / 1e9 / peak,
                              "traffic": ncu_traffic("summarize", args.config),
                              "algorithmic_bytes_per_launch": sum_bytes}}
    if args.raw_host:
        # host raw: the whole call (chunked H2D copies overlapped with the kernel) is bound by PCIe
        h2d = n * 4.0 * length
        summarize["roofline"] = {"kernel": "summarize (host raw, double-buffered H2D)", "bound": "pcie",
                                 "achieved": h2d / (sum_ms / 1e3) / 1e9, "peak": h2d_gbs, "unit": "GB/s",
                                 "frac": h2d / (sum_ms / 1e3) / 1e9 / h2d_gbs, "traffic": None,
                                 "algorithmic_bytes_per_launch": h2d,
                                 "peak_source": "measured in this run: pinned host -> device cudaMemcpyAsync"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        n_sample = min(n, args.ref_sample)
        t_q = oracle_sample(raw, queries, k, n_sample, args.ref_queries)
        cpu = {"value": 1.0 / (t_q * n / n_sample), "unit": "queries/s", "cores": 1, "kind": "oracle",
               "sample": f"oracle_knn_pruned (1 thread, fp64) over the first {n_sample} series, "
                         f"{args.ref_queries} queries, time scaled x{n / n_sample:.0f} to n={n}"}

    if rank == 0:
        line = {
            "metric": "exact 1-NN queries/sec", "value": value, "unit": "queries/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
            "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f32",
            "data": "synthetic (seeded Philox random walks, z-normalized; no dataset on the box)",
            "config": {"workload": cfg["desc"], "n": n, "len": length, "w": W, "card": CARD, "nq": nq, "k": k,
                       "batch": primary["batch"], "path": args.path, "index_build_ms": index_ms,
                       "raw_bf16": None if raw16 is None else {"build_ms": raw16_ms, "bytes": raw16.numel() * 2}, "parallelism": f"weak x{ws} (independent collections + queries per GPU)",
                       "l2": "inputs larger than L2 (no flush)",
                       "raw": "pinned host memory (f3)" if args.raw_host else "HBM"},
            "roofline": dict(roof, read_peak_gbs=read_peak,
                             frac_of_read_peak=(roof["achieved"] / read_peak
                                                if read_peak and roof and roof.get("unit") == "GB/s" else None))
                        if roof else roof,
            "lb_batch1": lb1,
            "other_path": None if secondary is None else {
                "path": secondary["path"], "value": secondary["value"], "ms_per_step": secondary["step_ms"],
                "roofline": secondary["roof"], "kernels": secondary["kern"],
                "candidates_mean": float(secondary["cand"].mean()), "refined_mean": float(secondary["refined"].mean())},
            "cpu_baseline": cpu,
            "sweep": sweep,
            "e2e": {"value": e2e_value, "unit": "queries/s", "h2d_bytes_per_step": nq * length * 4,
                    "d2h_bytes_per_step": nq * k * 12},
            "gpu_launches": launches,
            "clocks": clocks,
            "summarize": summarize,
            "kernels": kern,
            "pruning": {"candidates_mean": float(cand.mean()), "candidates_p50": float(np.median(cand)),
                        "candidates_max": float(cand.max()), "refined_mean": float(refined.mean()),
                        "refined_max": float(refined.max()),
                        "pruning_ratio": float(1.0 - refined.mean() / n),
                        "tau_seed_mean": float(stats["tau_seed"].mean()),
                        "lb_blocks_frac_p50": float(np.median(stats["lb_blocks"].numpy())) / max(1.0, n / P.PARIS_INDEX_BLOCK),
                        "lb_blocks_frac_max": float(stats["lb_blocks"].numpy().max()) / max(1.0, n / P.PARIS_INDEX_BLOCK),
                        "lb_blocks_frac_mean": float(stats["lb_blocks"].numpy().mean()) / max(1.0, n / P.PARIS_INDEX_BLOCK),
                        "lb_blocks_top5_share": float(np.sort(stats["lb_blocks"].numpy())[-5:].sum()
                                                      / max(1, stats["lb_blocks"].numpy().sum())),
                        "refined_top5_share": float(np.sort(refined)[-5:].sum() / max(1.0, refined.sum())),
                        "bsf_updates_mean": primary.get("bsf_updates_mean"),
                        "raw16_rows_mean": float(stats["raw16_rows"].numpy().astype(np.float64).mean())},
        }
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def run_gpu_sharded(args):
    """--shard: ONE collection of the config's size split by id range across the ranks
    (strong scaling); every query batch is searched per shard and merged exactly with one
    all-gather of the per-rank rows + paris_merge_topk."""
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2009_00166_b200 as P
    from paper_2009_00166_b200 import parallel as par
    from datagen import gpu as dg
    import datagen

    ws, rank, local = dist_env()
    if ws > 1:
        dist.init_process_group("nccl")
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    cfg = CONFIGS[args.config]
    n, length, nq, k = cfg["n"], cfg["len"], cfg["nq"], cfg["k"]
    if args.n:
        n = args.n
    if args.nq:
        nq = args.nq
    call_q = cfg.get("call", nq)
    ds, qs = datagen.config_seeds(args.config)
    lo, hi = par.shard_range(n, rank, ws)
    raw = dg.walks(hi - lo, length, ds, first_id=lo, device=dev)        # this rank's ids [lo, hi)
    if cfg["queries"] == "fresh":
        queries = dg.walks(nq, length, qs, device=dev)
    else:
        full_src = torch.empty(0)  # member queries need their source rows: generate them by id
        src = datagen.member_ids(nq, n, qs)
        base = torch.stack([dg.walks(1, length, ds, first_id=int(s_), device=dev)[0] for s_ in src])
        queries, _ = dg.noisy_members(base, nq, float(cfg["queries"][5:]), qs)
        del full_src
    sax = P.summarize(raw, W, CARD)
    index = P.index_build(sax, W, CARD)
    local_fn = par.local_index_search(raw, index, config=P.KnnConfig(index_seeds=args.index_seeds))
    torch.cuda.synchronize()

    def step():
        outs = []
        for c0 in range(0, nq, call_q):
            outs.append(par.knn_sharded(queries[c0:c0 + call_q], k, lo, local_fn))
        return outs

    for _ in range(max(3, args.warmup)):
        step()
    torch.cuda.synchronize()
    st = torch.cuda.current_stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    if ws > 1:
        dist.barrier()
    torch.cuda.synchronize()
    with ClockSampler(local) as clocks:
        e0.record(st)
        for _ in range(args.steps):
            step()
        e1.record(st)
        torch.cuda.synchronize()
    if ws > 1:
        dist.barrier()
    ms = reduce_max_ms(e0.elapsed_time(e1) / args.steps, dev, ws)
    value = nq / (ms / 1e3)
    if rank == 0:
        line = {"metric": "exact 1-NN queries/sec", "value": value, "unit": "queries/s", "n_gpus": ws,
                "steps": args.steps, "warmup": max(3, args.warmup), "ms_per_step": ms, "higher_is_better": True,
                "scaling": "strong", "vs_baseline": None, "dtype": "f32",
                "data": "synthetic (seeded Philox random walks, z-normalized; no dataset on the box)",
                "config": {"workload": cfg["desc"], "n": n, "len": length, "w": W, "card": CARD, "nq": nq, "k": k,
                           "path": "index, sharded by id range + all-gather + paris_merge_topk",
                           "parallelism": f"shard x{ws}", "l2": "inputs larger than L2 (no flush)"},
                "clocks": clocks.summary()}
        print(json.dumps(line), flush=True)
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="paris", choices=["paris", "reference"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--index-seeds", type=int, default=0, help="index path: seed series around the leaf")
    ap.add_argument("--both", type=int, default=1, help="also time the other query path (reported as a sub-object)")
    ap.add_argument("--path", default="index", choices=["flat", "index", "nb"],
                    help="flat: paris_knn_exact over the SAX array (ParIS+ Alg9); index: paris_knn_index over "
                         "the iSAX-ordered array with block envelopes (SURVEY f1)")
    ap.add_argument("--n", type=int, default=0, help="override n (debug only)")
    ap.add_argument("--nq", type=int, default=0, help="override query count (debug only)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--shard", action="store_true",
                    help="one collection split across the ranks (strong scaling, exact merge) instead of one "
                         "collection per rank (weak scaling)")
    ap.add_argument("--no-b1", action="store_true", help="skip the batch-1 LB roofline measurement")
    ap.add_argument("--sorted-refine", action="store_true",
                    help="k = 1: refine bucket-sorted lists (K5 scatter) instead of the unsorted waves (A/B)")
    ap.add_argument("--raw16", action="store_true", help="(default) index path with the bf16 refinement "
                    "pre-filter (paris_raw_bf16 + paris_knn_index_x)")
    ap.add_argument("--no-raw16", action="store_true", help="index path without the bf16 pre-filter")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C2 k=10 / C5 sigma x k sweeps")
    ap.add_argument("--raw-host", action="store_true",
                    help="f3: keep the raw collection in pinned host memory (SAX/index in HBM)")
    ap.add_argument("--ref-sample", type=int, default=2_000_000)
    ap.add_argument("--ref-queries", type=int, default=4)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "paris" else args.warmup
    if args.impl == "reference":
        return run_reference(args)
    if args.shard:
        return run_gpu_sharded(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
