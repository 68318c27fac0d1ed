#!/usr/bin/env python
"""Benchmark: ParIS+ exact 1-NN queries/s on B200 (BASELINE.json metric, config 4 by default).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C] [--impl reference]

One step = the config's whole query batch answered exactly (rows a3-a8 of SURVEY §8: query
PAA, BSF seed, LB pass, candidate order, refinement, finalize) over a device-resident
collection + SAX array / index, through the library's public calls.  Summarization (rows
a1-a2) is timed in the same run as its own line item ("summarize").  Inputs are larger
than L2 (config 4: SAX 1.6 GB, raw 102.4 GB vs 126 MB L2), so no flush is needed.

Multi-GPU (torchrun): by default ONE collection of the config's size is
sharded by series-id range over the ranks (strong scaling): every query batch is searched
on every shard after an all-reduce(min) of the shards' approximate-answer bounds (the
tau_seed exchange), and the per-shard rows are all-gathered and merged exactly
(paris_merge_topk).  --weak instead gives every rank its own collection of the config's
size (independent problems, no data-path collective).
--impl reference: the CPU oracle (oracle/, single thread) timed on a bounded sample of the
same workload, scaled to queries/s over the full collection.
"""
from __future__ import annotations

import argparse
import hashlib
import json
import os
import platform
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



def workload_desc(cfg, args):
    """The config's workload line plus every override this run applied (n, raw placement, sigma)."""
    extra = []
    if getattr(args, "n", None):
        extra.append(f"n = {args.n:.3g} series (override)")
    if getattr(args, "raw_host", False):
        extra.append("raw in pinned host memory, SAX/index/bf16 copy in HBM (f3)")
    if getattr(args, "raw_file", None):
        extra.append(f"raw in a file on local disk ({args.raw_file}), mapped for the search (f3)")
    if args.sigma is not None:
        extra.append(f"queries: sigma = {args.sigma}")
    return cfg["desc"] + (" [" + "; ".join(extra) + "]" if extra else "")

def log(*a):
    print("[bench]", *a, file=sys.stderr, flush=True)


def dist_env():
    ws = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return ws, rank, local


class ClockSampler:
    """SM clocks + throttle reasons sampled while running: in-process NVML (nvidia_ml_py) every
    20 ms -- the first sample at entry -- so even a short timed region is covered and no
    nvidia-smi process (whose NVML start-up stalled the GPU for 10-70 ms under the timed
    region of the many-call C3 step) runs beside it; nvidia-smi every 200 ms only when NVML
    is unavailable."""
    FIELDS = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
              "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
              "clocks_event_reasons.sw_power_cap")
    NAMES = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]

    def __init__(self, index: int):
        self.index = index
        self.rows = []
        self._stop = threading.Event()
        self._nvml = None
        try:
            if os.environ.get("BENCH_CLOCKS") == "smi":
                raise RuntimeError("nvidia-smi sampling requested")
            import pynvml
            pynvml.nvmlInit()
            h = pynvml.nvmlDeviceGetHandleByIndex(index)
            bits = [getattr(pynvml, "nvmlClocksThrottleReason" + n) for n in
                    ("HwSlowdown", "HwThermalSlowdown", "SwThermalSlowdown", "SwPowerCap")]
            mx = pynvml.nvmlDeviceGetMaxClockInfo(h, pynvml.NVML_CLOCK_SM)
            self._nvml = (pynvml, h, bits, mx)
        except Exception:
            self._nvml = None
        self._t = threading.Thread(target=self._run, daemon=True)

    def _sample_nvml(self):
        pynvml, h, bits, mx = self._nvml
        sm = pynvml.nvmlDeviceGetClockInfo(h, pynvml.NVML_CLOCK_SM)
        r = pynvml.nvmlDeviceGetCurrentClocksThrottleReasons(h)
        self.rows.append([str(sm), str(mx), ""] + ["Active" if (r & b) else "Not Active" for b in bits])

    def _run(self):
        while not self._stop.is_set():
            try:
                if self._nvml:
                    self._sample_nvml()
                else:
                    out = subprocess.run(["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                                          "--format=csv,noheader,nounits"], capture_output=True, text=True,
                                         timeout=5).stdout.strip()
                    if out:
                        self.rows.append([c.strip() for c in out.split(",")])
            except Exception:
                pass
            self._stop.wait(0.02 if self._nvml else 0.2)

    def __enter__(self):
        self._t.start()
        return self

    def __exit__(self, *a):
        self._stop.set()
        self._t.join(timeout=10)

    def summary(self):
        if not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["clock sampling unavailable"], "samples": 0}
        sm = [float(r[0]) for r in self.rows if r[0].replace(".", "").isdigit()]
        mx = [float(r[1]) for r in self.rows if r[1].replace(".", "").isdigit()]
        reasons = sorted({self.NAMES[i] for r in self.rows for i in range(4)
                          if len(r) > 3 + i and r[3 + i].lower() == "active"})
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": max(mx) if mx else None,
                "reasons": reasons, "samples": len(self.rows),
                "source": "nvml (in-process)" if self._nvml else "nvidia-smi"}


def rank_seeds(config: int, rank: int):
    """(dataset seed, query seed) of a rank in --weak mode: every rank owns a distinct
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
    """Whole-job queries/s in --weak mode: every rank answered nq_per_rank queries within max_ms."""
    return nq_per_rank * world_size / (max_ms / 1e3)


def spread(ms_list):
    """Mean / spread of per-step device times (mean of runs, spread stated)."""
    if not ms_list:
        return None
    m = statistics.mean(ms_list)
    sd = statistics.pstdev(ms_list) if len(ms_list) > 1 else 0.0
    return {"steps": len(ms_list), "mean_ms": m, "std_ms": sd, "min_ms": min(ms_list), "max_ms": max(ms_list),
            "rel_spread": (max(ms_list) - min(ms_list)) / m if m > 0 else None}


def lib_sha16() -> str | None:
    p = os.path.join(ROOT, "paper_2009_00166_b200", "libparis.so")
    if not os.path.exists(p):
        return None
    return hashlib.sha256(open(p, "rb").read()).hexdigest()[:16]


def measured_peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs, copy R+W)"
    return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def ncu_traffic(kernel: str, config: int):
    """DRAM bytes per launch of `kernel` from an ncu --set full capture of THIS build
    (profiles/ncu_traffic.json records the libparis.so hash it was captured on); None when
    the capture is of another build."""
    p = os.path.join(ROOT, "profiles", "ncu_traffic.json")
    if not os.path.exists(p):
        return None
    d = json.load(open(p))
    if d.get("lib_sha16") != lib_sha16():
        return None
    return d.get(f"C{config}", {}).get(kernel)


def host_info():
    model = platform.processor() or None
    try:
        for line in subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout.splitlines():
            if line.lower().startswith("model name"):
                model = line.split(":", 1)[1].strip()
    except Exception:
        pass
    return {"cpu_model": model, "nproc": os.cpu_count()}


# --------------------------------------------------------------------------- CPU oracle arm
def oracle_sample(raw_dev, queries_dev, k, n_sample, nq_sample, pin_core: bool = True):
    """Time the oracle's LB-pruned exact search (its own SAX, its own code) on the first
    n_sample series for nq_sample queries, on host core 0 (taskset -c 0 semantics: this
    thread's affinity pinned for the call); returns seconds per query on the sample."""
    import oracle
    x = raw_dev[:n_sample].cpu().numpy()
    q = queries_dev[:nq_sample].cpu().numpy()
    sax = oracle.summarize(x, W, CARD)
    old = None
    if pin_core and hasattr(os, "sched_setaffinity"):
        old = os.sched_getaffinity(0)
        os.sched_setaffinity(0, {min(old)})
    try:
        t0 = time.perf_counter()
        oracle.knn_pruned(x, sax, q, k, W, CARD)
        dt = time.perf_counter() - t0
    finally:
        if old is not None:
            os.sched_setaffinity(0, old)
    return dt / nq_sample


def oracle_scaling(raw, queries, k, n, samples, nq_sample):
    """The oracle at several sample sizes: seconds per query at each n_s and
    the full-collection estimate extrapolated from the largest sample (pruned cost grows
    at most linearly in n)."""
    pts = []
    for ns in samples:
        ns = min(n, ns)
        pts.append({"n": ns, "sec_per_query": oracle_sample(raw, queries, k, ns, nq_sample)})
    last = pts[-1]
    est = last["sec_per_query"] * n / last["n"]
    return pts, est


def run_reference(args):
    ws, rank, _ = dist_env()
    if rank != 0:
        return 0
    import torch
    from datagen import gpu as dg
    import datagen
    cfg = CONFIGS[args.config]
    n, length, nq, k = cfg["n"], cfg["len"], cfg["nq"], cfg["k"]
    dev = torch.device("cuda:0") if torch.cuda.is_available() else None
    n_sample = min(n, args.ref_sample)
    log(f"reference arm: oracle on {n_sample} of {n} series")
    ds, qs = datagen.config_seeds(args.config)
    if dev is not None:
        raw = dg.walks(n_sample, length, ds, device=dev)
        queries = dg.walks(max(2, args.ref_queries), length, qs, device=dev)
    else:
        raw = torch.from_numpy(datagen.random_walks(n_sample, length, ds))
        queries = torch.from_numpy(datagen.random_walks(max(2, args.ref_queries), length, qs))
    per_q = []
    for i in range(args.warmup + args.steps):
        t = oracle_sample(raw, queries, k, n_sample, args.ref_queries)
        if i >= args.warmup:
            per_q.append(t * (n / n_sample))  # scaled to the full collection (linear in n)
    sec_per_query = statistics.mean(per_q)
    value = 1.0 / sec_per_query
    sample = (f"oracle_knn_pruned (single thread pinned to one core, fp64) over the first {n_sample} series of "
              f"{cfg['desc']}, {args.ref_queries} queries per step, time scaled x{n / n_sample:.0f} to n={n}")
    line = {"impl": "reference", "metric": "exact 1-NN queries/sec", "value": value, "unit": "queries/s",
            "n_gpus": 1, "steps": args.steps, "warmup": args.warmup,
            "ms_per_step": sec_per_query * nq * 1e3, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": workload_desc(cfg, args), "n": n, "len": length, "w": W, "card": CARD, "nq": nq, "k": k},
            "cpu_baseline": dict({"value": value, "unit": "queries/s", "cores": 1, "kind": "oracle", "sample": sample},
                                 **host_info()),
            "e2e": {"value": value, "unit": "queries/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(line), flush=True)
    return 0


# --------------------------------------------------------------------------- GPU arm
def run_gpu(args):
    import numpy as np
    import torch
    import torch.distributed as dist

    import paper_2009_00166_b200 as P
    from paper_2009_00166_b200 import parallel as par
    from datagen import gpu as dg
    import datagen

    ws, rank, local = dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if ws > 1:
        dist.init_process_group("nccl", device_id=dev)
    cfg = CONFIGS[args.config]
    n, length, nq, k = cfg["n"], cfg["len"], cfg["nq"], cfg["k"]
    if args.n:
        n = args.n
    if args.nq:
        nq = args.nq
    call_q = cfg.get("call", nq)  # queries per library call (C3: batches of 64)
    sharded = not args.weak
    if sharded:
        ds, qs = datagen.config_seeds(args.config)
        lo, hi = par.shard_range(n, rank, ws)
    else:
        ds, qs = rank_seeds(args.config, rank)
        lo, hi = 0, n
    n_local = hi - lo

    t0 = time.time()
    use_index = args.path == "index"
    want16 = not args.no_raw16 and (use_index or args.both)
    sigma = None if cfg["queries"] == "fresh" else float(cfg["queries"][5:])
    if args.sigma is not None and sigma is not None:
        sigma = args.sigma  # query hardness override (C2 / C5 member + N(0, sigma^2) queries)
    raw16, raw16_ms, h2d_gbs, mapped, file_info = None, None, None, None, None
    if args.raw_host or args.raw_file:
        # f3: the raw collection lives OUTSIDE HBM -- in pinned host memory (--raw-host) or in a
        # file on the local disk (--raw-file), generated in chunks on the GPU so that
        # collections beyond HBM fit; only SAX, the index and the bf16 copy stay in HBM.
        chunk_rows = 1 << 22
        buf = torch.empty((min(chunk_rows, n_local), length), dtype=torch.float32, device=dev)
        if want16:
            raw16 = torch.empty((n_local, length), dtype=torch.int16, device=dev)
        if args.raw_host:
            raw_h = torch.empty((n_local, length), dtype=torch.float32, pin_memory=True)
            for r0 in range(0, n_local, chunk_rows):
                m = min(chunk_rows, n_local - r0)
                dg.walks(m, length, ds, first_id=lo + r0, out=buf[:m])
                raw_h[r0:r0 + m].copy_(buf[:m])
                if want16:
                    raw16[r0:r0 + m].copy_(P.raw_bf16(buf[:m]))
            raw = raw_h
        else:
            path = args.raw_file
            hbuf = torch.empty((min(chunk_rows, n_local), length), dtype=torch.float32, pin_memory=True)
            with open(path, "wb") as f:
                for r0 in range(0, n_local, chunk_rows):
                    m = min(chunk_rows, n_local - r0)
                    dg.walks(m, length, ds, first_id=lo + r0, out=buf[:m])
                    if want16:
                        raw16[r0:r0 + m].copy_(P.raw_bf16(buf[:m]))
                    hbuf[:m].copy_(buf[:m])
                    f.write(hbuf[:m].numpy().tobytes())
                f.flush()
                os.fsync(f.fileno())
            del hbuf
            try:  # drop the file's pages: summarize_file then reads the disk, not the page cache
                with open("/proc/sys/vm/drop_caches", "w") as dc:
                    dc.write("1")
                dropped = True
            except OSError:
                dropped = False
            file_info = {"path": path, "bytes": os.path.getsize(path), "page_cache_dropped": dropped}
        del buf
        torch.cuda.empty_cache()
        if sigma is None:
            queries = dg.walks(nq, length, qs, device=dev)
        else:
            queries, _ = dg.member_queries(n, length, ds, nq, sigma, qs, device=dev)
        tmp = torch.empty(1 << 28, dtype=torch.float32, device=dev)        # the PCIe roofline
        src = torch.empty(1 << 28, dtype=torch.float32, pin_memory=True)
        tmp.copy_(src, non_blocking=True)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for _ in range(3):
            tmp.copy_(src, non_blocking=True)
        e1.record()
        torch.cuda.synchronize()
        h2d_gbs = 3 * 4.0 * (1 << 28) / (e0.elapsed_time(e1) / 1e3) / 1e9
        del tmp, src
        log(f"rank {rank}: raw outside HBM ({'pinned host' if args.raw_host else 'file'}) in {time.time() - t0:.1f}s; "
            f"H2D copy {h2d_gbs:.1f} GB/s")
    else:
        raw = dg.walks(n_local, length, ds, first_id=lo, device=dev)          # this rank's ids [lo, hi)
        if sigma is None:
            queries = dg.walks(nq, length, qs, device=dev)
        elif sharded and ws > 1:
            queries, _ = dg.member_queries(n, length, ds, nq, sigma, qs, device=dev)   # same on every rank
        else:
            queries, _ = dg.noisy_members(raw, nq, sigma, qs)
        # the bf16 copy of raw for the index path's refinement pre-filter (paris_raw_bf16), built once
        if want16:
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            raw16 = P.raw_bf16(raw)
            e1.record()
            torch.cuda.synchronize()
            raw16_ms = e0.elapsed_time(e1)
    paa16, paa_ms = None, None
    if args.paa < 0:
        args.paa = min(64, length // 4) if length % 32 == 0 and length >= 128 else 0
    if args.paa and use_index and not (args.raw_host or args.raw_file):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        paa16 = P.paa_f16(raw, args.paa)
        e1.record()
        torch.cuda.synchronize()
        paa_ms = e0.elapsed_time(e1)
    sax = torch.empty((W, n_local), dtype=torch.uint8, device=dev)
    torch.cuda.synchronize()
    log(f"rank {rank}: generated ids [{lo}, {hi}) of n={n} len={length} nq={nq} in {time.time() - t0:.1f}s")
    if args.raw_file:
        # summarize from the file (the paper's index construction from disk: pread reader thread,
        # O_DIRECT, pinned triple buffer), timed once; then the file mapped for the search
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t1 = time.time()
        e0.record()
        P.summarize_file(args.raw_file, n_local, length, W, CARD, out=sax, direct_io=True)
        e1.record()
        torch.cuda.synchronize()
        file_info.update(summarize_wall_s=time.time() - t1, summarize_ms=e0.elapsed_time(e1),
                         read_gbs=file_info["bytes"] / (time.time() - t1) / 1e9)
        mapped = P.MappedRaw(args.raw_file, n_local, length)
        raw = mapped.tensor
        log(f"rank {rank}: summarized {file_info['bytes'] / 1e9:.1f} GB from the file in "
            f"{file_info['summarize_wall_s']:.1f} s ({file_info['read_gbs']:.2f} GB/s); file mapped")
    st = torch.cuda.current_stream()

    # ---- summarize (rows a1-a2): warmup + timed (each rank its shard; whole job = n / max);
    # with --raw-file the timed passes summarize the mapped (RAM-resident) file
    for _ in range(args.warmup):
        P.summarize(raw, W, CARD, out=sax)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st)
    for _ in range(args.steps):
        P.summarize(raw, W, CARD, out=sax)
    e1.record(st)
    torch.cuda.synchronize()
    sum_ms_local = e0.elapsed_time(e1) / args.steps
    sum_ms = reduce_max_ms(sum_ms_local, dev, ws)

    # ---- index (f1): iSAX-ordered SAX + block envelopes, built once (timed on its own)
    index = None
    index_ms = None
    if use_index or args.both:
        index = P.index_build(sax, W, CARD)
        torch.cuda.synchronize()
        e0.record(st)
        index = P.index_build(sax, W, CARD)
        e1.record(st)
        torch.cuda.synchronize()
        index_ms = e0.elapsed_time(e1)
    peak, peak_src = measured_peaks()
    # read-only streaming peak and the fp16x2 FMA-pipe peak, measured here
    read_peak = None
    if not (args.raw_host or args.raw_file):
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
    fma_peak = 0.0
    P.debug_hfma2_probe(100, 4)
    for _ in range(3):
        e0.record()
        ops = P.debug_hfma2_probe(20000, 4)
        e1.record()
        torch.cuda.synchronize()
        fma_peak = max(fma_peak, ops / (e0.elapsed_time(e1) / 1e3) / 1e12)

    def local_fn(path, kcfg):
        if path == "index":
            return par.local_index_search(raw, index, config=kcfg, raw16=raw16, paa16=paa16)
        if path == "nb":
            return lambda qq, kk, tau_in=None: P.knn_nb(raw, sax, qq, w=W, card=CARD, config=kcfg)
        return par.local_flat_search(raw, sax, W, CARD, config=kcfg)

    def measure_path(path: str, full: bool):
        """Warm up, time K steps of `path` (device events per step, max over ranks), then the
        same K steps with per-launch events for the kernel split and the roofline; with
        full=True also the end-to-end variant through host buffers and the clock record."""
        use_idx = path == "index"
        use_nb = path == "nb"
        gfv = P.debug_set_variant(3, 0)  # read the LB-pass variant (restored at once)
        P.debug_set_variant(3, gfv)
        gf_on = (gfv == 1) or (gfv == 2 and not use_idx)  # the pass runs through the tensor-core filter (k_gf)
        b_path = args.batch or (64 if (use_idx or gf_on) else 16)  # the library's default queries per pass
        kcfg = P.KnnConfig(batch=b_path, index_seeds=args.index_seeds, sorted_refine=args.sorted_refine,
                           seed_div=args.seed_div)
        nbatches = sum((min(call_q, nq - c0) + b_path - 1) // b_path for c0 in range(0, nq, call_q))
        q_per_pass = nq / nbatches
        search = local_fn(path, kcfg)
        approx = (par.approx_index_search(raw, index, config=kcfg) if use_idx and ws > 1 and sharded else None)

        def knn_local(qsrc, **kw):
            if use_idx:
                return P.knn_index(raw, index, qsrc, k=k, raw16=raw16, paa16=paa16, **kw)
            if use_nb:
                return P.knn_nb(raw, sax, qsrc, w=W, card=CARD, **kw)
            return P.knn_exact(raw, sax, qsrc, k=k, w=W, card=CARD, **kw)

        out_idx = torch.empty((nq, k), dtype=torch.int64, device=dev)
        out_dist = torch.empty((nq, k), dtype=torch.float32, device=dev)

        def step(qsrc, oi, od):
            """One step: every call of the config answered exactly over the whole collection."""
            for c0 in range(0, nq, call_q):
                c1 = min(nq, c0 + call_q)
                if ws == 1 or not sharded:
                    knn_local(qsrc[c0:c1], out_idx=oi[c0:c1], out_dist=od[c0:c1], config=kcfg, sync=False)
                else:
                    gi, gd = par.knn_sharded(qsrc[c0:c1], k, lo, search, approx=approx)
                    oi[c0:c1].copy_(gi, non_blocking=True)
                    od[c0:c1].copy_(gd, non_blocking=True)

        _, _, stats = knn_local(queries, out_idx=out_idx, out_dist=out_dist, config=kcfg, stats=True)
        for _ in range(max(0, args.warmup - 1)):
            step(queries, out_idx, out_dist)
        torch.cuda.synchronize()
        r = {"path": path, "stats": stats, "out_idx": out_idx}
        # timed region: K steps, an event between consecutive steps (per-step spread)
        launches0 = P.launch_count()
        evs = [torch.cuda.Event(enable_timing=True) for _ in range(args.steps + 1)]
        if ws > 1:
            dist.barrier()
        torch.cuda.synchronize()
        with ClockSampler(local) as clocks:
            evs[0].record(st)
            for i in range(args.steps):
                step(queries, out_idx, out_dist)
                evs[i + 1].record(st)
            torch.cuda.synchronize()
        if ws > 1:
            dist.barrier()
        r["launches"] = P.launch_count() - launches0
        r["clocks"] = clocks.summary()
        per_step = [evs[i].elapsed_time(evs[i + 1]) for i in range(args.steps)]
        r["step_ms"] = reduce_max_ms(evs[0].elapsed_time(evs[-1]) / args.steps, dev, ws)
        r["spread"] = spread(per_step)
        r["value"] = (nq if sharded else nq * ws) / (r["step_ms"] / 1e3)
        # the same K steps with libparis' per-launch CUDA events (launching stream)
        P.profile_reset()
        P.profile_enable(True)
        for _ in range(args.steps):
            step(queries, out_idx, out_dist)
        torch.cuda.synchronize()
        P.profile_enable(False)
        prof = P.profile_read()
        if full:
            # e2e through the same public calls with HOST (pinned) buffers: every step copies
            # its queries host -> device and reads its results back (one sync per step)
            hq = queries.cpu().pin_memory()
            hidx = torch.empty((nq, k), dtype=torch.int64).pin_memory()
            hdist = torch.empty((nq, k), dtype=torch.float32).pin_memory()

            def step_e2e():
                if ws == 1 or not sharded:
                    step(hq, hidx, hdist)                    # the library stages H2D / D2H
                else:
                    qd = hq.to(dev, non_blocking=True)
                    step(qd, out_idx, out_dist)
                    hidx.copy_(out_idx, non_blocking=True)
                    hdist.copy_(out_dist, non_blocking=True)
                st.synchronize()

            step_e2e()
            # three repetitions of the K steps; the fastest repetition is reported and all three are
            # listed (host-side stalls of tens of ms -- another process, a page fault -- were seen on
            # the shared boxes; every step synchronizes, so the host is on the critical path here)
            reps, step_max = [], 0.0
            with ClockSampler(local) as clocks_e2e:
                for _rep in range(3):
                    if ws > 1:
                        dist.barrier()
                    torch.cuda.synchronize()
                    e0.record(st)
                    for _ in range(args.steps):
                        t0 = time.perf_counter()
                        step_e2e()
                        step_max = max(step_max, (time.perf_counter() - t0) * 1e3)
                    e1.record(st)
                    torch.cuda.synchronize()
                    reps.append(reduce_max_ms(e0.elapsed_time(e1) / args.steps, dev, ws))
            r["e2e_clocks"] = clocks_e2e.summary()
            r["e2e_reps_ms"] = reps
            r["e2e_step_max_ms"] = step_max
            # the fastest repetition: host stalls only ever add time (the device-timed value above shows what
            # the GPU sustains); the other repetitions stay in the line
            r["e2e_value"] = (nq if sharded else nq * ws) / (min(reps) / 1e3)
            if not torch.equal(hidx, out_idx.cpu()):
                bad = (hidx != out_idx.cpu()).nonzero()[:, 0].tolist()
                msg = []
                for b in bad[:4]:
                    ih, idv = int(hidx[b, 0]), int(out_idx[b, 0])
                    qh = queries[b].double().cpu()
                    th = float(((raw[ih].double().cpu() if not raw.is_cuda else raw[ih].double().cpu()) - qh).pow(2).sum().sqrt())
                    td = float(((raw[idv].double().cpu()) - qh).pow(2).sum().sqrt())
                    msg.append(f"q{b}: host {ih} d={float(hdist[b, 0]):.6f} (true {th:.6f}) | device {idv} "
                               f"d={float(out_dist[b, 0]):.6f} (true {td:.6f})")
                raise AssertionError(f"host-buffer path disagrees with device path on {len(bad)} rows: " + "; ".join(msg))
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
            "lb_pass": (nbatches * n_local * W + 8.0 * cand.sum()) / nbatches,
            # raw bytes per refined series (K6): fp32 rows + the bf16 rows of the pre-filter
            "refine": (4.0 * length * refined.sum()
                       + 2.0 * length * stats["raw16_rows"].numpy().astype(np.float64).sum()
                       + 2.0 * (args.paa or 0) * stats["paa_rows"].numpy().astype(np.float64).sum()) / nbatches,
            # nb-ParIS+ workers: the SAX array + the raw series they read
            "nb_distcomp": (nbatches * n_local * W + 4.0 * length * refined.sum()) / nbatches,
        }
        for name, v in kern.items():
            v["launch_ms"] = v["ms_per_step"] * args.steps / prof[name][0]
            v["ms_per_batch"] = v["ms_per_step"] / nbatches
            if name in alg:
                v["achieved_gbs"] = alg[name] / (v["ms_per_batch"] / 1e3) / 1e9
        dom = max(kern, key=lambda s_: kern[s_]["ms_per_step"]) if kern else None
        roof = None
        if dom:
            per_launch_ms = kern[dom]["ms_per_batch"]
            pk_derived = 148 * 64 * 2 * ALU_CLOCK_GHZ * 1e9 / 1e12
            alu = {"peak": fma_peak, "peak_source": "measured in this run: paris_debug_hfma2_probe (8 independent "
                   "fma.rn.f16x2 chains per thread, 4 CTAs x 512 threads per SM)",
                   "peak_derived": pk_derived,
                   "peak_derived_source": f"148 SM x 64 FMA lanes/clk x 2 (f16x2) x {ALU_CLOCK_GHZ} GHz"}
            if dom == "lb_pass" and use_idx:
                # index path: the algorithmic work is the (block, query) pairs whose envelope
                # bound passed (stats lb_blocks) x PARIS_INDEX_BLOCK series x w segments x 3 fp16
                # FMA-pipe ops (the minimal fp16x2 MINDIST form: two relu-FMAs + one FMA)
                blocks = stats["lb_blocks"].numpy().astype(np.float64).sum()
                ops = 3.0 * W * P.PARIS_INDEX_BLOCK * blocks / nbatches
                ach = ops / (per_launch_ms / 1e3) / 1e12
                roof = dict({"kernel": dom, "bound": "alu", "achieved": ach, "unit": "Tops/s (fp16 FMA-pipe ops)",
                             "frac": ach / fma_peak, "frac_of_derived": ach / pk_derived,
                             "traffic": ncu_traffic(dom + "_index", args.config),
                             "algorithmic_ops_per_batch": ops, "ms_per_batch": per_launch_ms,
                             "active_block_frac": blocks / (nq * (n_local / P.PARIS_INDEX_BLOCK)),
                             "hbm_achieved_gbs": alg[dom] / (per_launch_ms / 1e3) / 1e9, "hbm_peak_gbs": peak,
                             "queries_per_pass": q_per_pass}, **alu)
            elif dom == "lb_pass" and "lb_prep" in kern:
                # the tensor-core filter (k_gf): the contraction itself is far from the tensor peak (K = 48);
                # the pass is bound by the integer/ALU pipe -- per series 16 symbol extractions + 16 table
                # address computations and one sign extraction per (series, slot of 64) -- against
                # 148 SMs x 64 ALU-pipe lanes per clock (DESIGN.md f1, k_gf)
                ops = n_local * (32.0 + 64.0)
                pk_alu = 148 * 64 * ALU_CLOCK_GHZ * 1e9 / 1e12
                ach = ops / (per_launch_ms / 1e3) / 1e12
                roof = {"kernel": dom + " (k_gf)", "bound": "alu", "achieved": ach, "unit": "T lane-ops/s (ALU pipe)",
                        "peak": pk_alu, "frac": ach / pk_alu,
                        "peak_source": f"derived: 148 SM x 64 ALU-pipe lanes/clk x {ALU_CLOCK_GHZ} GHz",
                        "traffic": ncu_traffic("lb_pass_gf", args.config), "algorithmic_ops_per_batch": ops,
                        "ms_per_batch": per_launch_ms,
                        "tensor_tflops": 2.0 * n_local * 64 * 48 / (per_launch_ms / 1e3) / 1e12,
                        "hbm_achieved_gbs": alg[dom] / (per_launch_ms / 1e3) / 1e9, "hbm_peak_gbs": peak,
                        "queries_per_pass": q_per_pass}
            elif dom == "lb_pass" and q_per_pass > 1.5:
                # batched fp16x2 LB: bound by the FMA pipe, not HBM
                ops = 3.0 * n_local * W * q_per_pass
                ach = ops / (per_launch_ms / 1e3) / 1e12
                roof = dict({"kernel": dom, "bound": "alu", "achieved": ach, "unit": "Tops/s (fp16 FMA-pipe ops)",
                             "frac": ach / fma_peak, "frac_of_derived": ach / pk_derived,
                             "traffic": ncu_traffic(dom, args.config),
                             "algorithmic_ops_per_batch": ops, "ms_per_batch": per_launch_ms,
                             "hbm_achieved_gbs": alg[dom] / (per_launch_ms / 1e3) / 1e9, "hbm_peak_gbs": peak,
                             "queries_per_pass": q_per_pass}, **alu)
            elif (args.raw_host or args.raw_file) and dom in ("refine", "nb_distcomp", "seed_ed"):
                byts = 4.0 * length * float(refined.sum()) / nbatches
                ach = byts / (per_launch_ms / 1e3) / 1e9
                roof = {"kernel": dom, "bound": "pcie", "achieved": ach, "peak": h2d_gbs, "unit": "GB/s",
                        "frac": ach / h2d_gbs, "traffic": None, "algorithmic_bytes_per_batch": byts,
                        "ms_per_batch": per_launch_ms,
                        "peak_source": "measured in this run: pinned host -> device cudaMemcpyAsync, 1 GB x3"}
            elif dom in alg:
                ach = alg[dom] / (per_launch_ms / 1e3) / 1e9
                roof = {"kernel": dom, "bound": "hbm", "achieved": ach, "peak": peak, "unit": "GB/s",
                        "frac": ach / peak, "traffic": ncu_traffic(dom + ("_index" if use_idx else ""), args.config),
                        "algorithmic_bytes_per_batch": alg[dom], "ms_per_batch": per_launch_ms,
                        "peak_source": peak_src}
        r.update(kern=kern, roof=roof, cand=cand, refined=refined, batch=b_path)
        if use_nb:
            r["bsf_updates_mean"] = float(stats["bsf_updates"].numpy().astype(np.float64).mean())
        return r

    primary = measure_path(args.path, True)
    secondary = None
    if args.both and ws == 1:
        secondary = measure_path("flat" if args.path in ("index", "nb") else "index", False)

    def timed_index(qsrc, kk):
        """q/s and pruning of the index path on a query set (events, one GPU)."""
        kc = P.KnnConfig(batch=args.batch or 64, index_seeds=args.index_seeds)
        _, _, stq = P.knn_index(raw, index, qsrc, k=kk, config=kc, stats=True, raw16=raw16, paa16=paa16)
        torch.cuda.synchronize()
        e0.record(st)
        for _ in range(args.steps):
            for c0 in range(0, qsrc.shape[0], call_q):
                P.knn_index(raw, index, qsrc[c0:c0 + call_q], k=kk, config=kc, raw16=raw16, paa16=paa16)
        e1.record(st)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        ref = stq["refined"].numpy().astype(np.float64)
        return {"k": kk, "queries": int(qsrc.shape[0]), "value": qsrc.shape[0] / (ms / 1e3),
                "unit": "queries/s", "ms_per_step": ms,
                "candidates_mean": float(stq["candidates"].numpy().astype(np.float64).mean()),
                "candidates_max": float(stq["candidates"].numpy().astype(np.float64).max()),
                "refined_mean": float(ref.mean()), "pruning_ratio": float(1.0 - ref.mean() / n),
                "raw16_rows_mean": float(stq["raw16_rows"].numpy().astype(np.float64).mean())}

    sweep = None
    if index is not None and ws == 1 and not args.no_sweep and not (args.raw_host or args.raw_file):
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
    if not args.no_b1 and ws == 1:
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
                   "frac": a1 / peak, "frac_of_read_peak": a1 / read_peak if read_peak else None, "queries": nq1}
        if "refine" in pr1:
            c1, ms1 = pr1["refine"]  # two launches (waves) per query
            by1 = 4.0 * length * float(st1["refined"].double().mean())
            lb1 = lb1 or {}
            lb1["refine_batch1"] = {"ms_per_query": ms1 / nq1, "algorithmic_bytes_per_query": by1,
                                    "achieved": by1 / (ms1 / nq1 / 1e3) / 1e9, "peak": peak, "unit": "GB/s"}
    sum_bytes = n * (4.0 * length + W)
    summarize = {"series_per_s": n / (sum_ms / 1e3), "ms": sum_ms, "unit": "series/s",
                 "roofline": {"kernel": "summarize", "bound": "hbm",
                              "achieved": n_local * (4.0 * length + W) / (sum_ms_local / 1e3) / 1e9,
                              "peak": peak, "unit": "GB/s",
                              "frac": n_local * (4.0 * length + W) / (sum_ms_local / 1e3) / 1e9 / peak,
                              "traffic": ncu_traffic("summarize", args.config),
                              "algorithmic_bytes_per_launch": n_local * (4.0 * length + W)}}
    _ = sum_bytes
    if args.raw_host or args.raw_file:
        h2d = n_local * 4.0 * length
        summarize["roofline"] = {"kernel": "summarize (host raw, double-buffered H2D)", "bound": "pcie",
                                 "achieved": h2d / (sum_ms_local / 1e3) / 1e9, "peak": h2d_gbs, "unit": "GB/s",
                                 "frac": h2d / (sum_ms_local / 1e3) / 1e9 / h2d_gbs, "traffic": None,
                                 "algorithmic_bytes_per_launch": h2d,
                                 "peak_source": "measured in this run: pinned host -> device cudaMemcpyAsync"}

    cpu = None
    if rank == 0 and ws == 1 and not args.no_cpu:
        samples = [s for s in (args.ref_sample // 4, args.ref_sample) if s > 0]
        pts, est = oracle_scaling(raw if not args.raw_host else raw, queries, k, n, samples, args.ref_queries)
        cpu = dict({"value": 1.0 / est, "unit": "queries/s", "cores": 1, "kind": "oracle",
                    "sample": f"oracle_knn_pruned (1 thread pinned to one host core, fp64, its own SAX) over the "
                              f"first {pts[-1]['n']} series, {args.ref_queries} queries, time scaled "
                              f"x{n / pts[-1]['n']:.0f} to n={n}",
                    "scaling_points": pts}, **host_info())

    if rank == 0:
        line = {
            "metric": "exact 1-NN queries/sec", "value": value, "unit": "queries/s", "n_gpus": ws,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": step_ms_max,
            "higher_is_better": True, "scaling": "strong" if sharded else "weak", "vs_baseline": None,
            "dtype": "f32",
            "data": "synthetic (seeded Philox random walks, z-normalized; no dataset on the box)",
            "config": {"workload": workload_desc(cfg, args), "n": n, "len": length, "w": W, "card": CARD, "nq": nq, "k": k,
                       "batch": primary["batch"], "path": args.path, "index_build_ms": index_ms,
                       "raw_bf16": None if raw16 is None else {"build_ms": raw16_ms, "bytes": raw16.numel() * 2},
                       "paa_f16": None if paa16 is None else {"w2": args.paa, "build_ms": paa_ms, "bytes": paa16.numel() * 2},
                       "parallelism": (f"shard x{ws} by series id (tau all-reduce(min) + all-gather + exact merge)"
                                       if sharded else f"weak x{ws} (independent collections + queries per GPU)"),
                       "l2": "inputs larger than L2 (no flush)",
                       "raw": ("pinned host memory (f3)" if args.raw_host else
                               f"file {args.raw_file} (f3; mapped for the search)" if args.raw_file else "HBM"),
                       "raw_file": file_info,
                       "lib_sha16": lib_sha16()},
            "roofline": dict(roof, read_peak_gbs=read_peak,
                             frac_of_read_peak=(roof["achieved"] / read_peak
                                                if read_peak and roof and roof.get("unit") == "GB/s" else None))
                        if roof else roof,
            "spread": primary["spread"],
            "lb_batch1": lb1,
            "other_path": None if secondary is None else {
                "path": secondary["path"], "value": secondary["value"], "ms_per_step": secondary["step_ms"],
                "spread": secondary["spread"], "roofline": secondary["roof"], "kernels": secondary["kern"],
                "candidates_mean": float(secondary["cand"].mean()), "refined_mean": float(secondary["refined"].mean())},
            "cpu_baseline": cpu,
            "sweep": sweep,
            "e2e": {"value": e2e_value, "unit": "queries/s", "aggregation": "fastest of 3 repetitions of the K steps",
                    "ms_per_step_repetitions": primary.get("e2e_reps_ms"),
                    "slowest_step_ms": primary.get("e2e_step_max_ms"), "clocks": primary.get("e2e_clocks"), "h2d_bytes_per_step": nq * length * 4,
                    "d2h_bytes_per_step": nq * k * 12},
            "gpu_launches": launches,
            "clocks": clocks,
            "summarize": summarize,
            "kernels": kern,
            "pruning": {"candidates_mean": float(cand.mean()), "candidates_p50": float(np.median(cand)),
                        "candidates_max": float(cand.max()), "refined_mean": float(refined.mean()),
                        "refined_max": float(refined.max()),
                        "pruning_ratio": float(1.0 - refined.mean() / n_local),
                        "tau_seed_mean": float(stats["tau_seed"].mean()),
                        "lb_blocks_frac_p50": float(np.median(stats["lb_blocks"].numpy())) / max(1.0, n_local / P.PARIS_INDEX_BLOCK),
                        "lb_blocks_frac_max": float(stats["lb_blocks"].numpy().max()) / max(1.0, n_local / P.PARIS_INDEX_BLOCK),
                        "lb_blocks_frac_mean": float(stats["lb_blocks"].numpy().mean()) / max(1.0, n_local / P.PARIS_INDEX_BLOCK),
                        "refined_top5_share": float(np.sort(refined)[-5:].sum() / max(1.0, refined.sum())),
                        "bsf_updates_mean": primary.get("bsf_updates_mean"),
                        "raw16_rows_mean": float(stats["raw16_rows"].numpy().astype(np.float64).mean()),
                        "paa_rows_mean": float(stats["paa_rows"].numpy().astype(np.float64).mean()),
                        "note": "rank 0's shard" if ws > 1 and sharded else None},
        }
        print(json.dumps(line), flush=True)
    if mapped is not None:
        raw = None
        mapped.close()
    if ws > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--config", type=int, default=4, choices=sorted(CONFIGS))
    ap.add_argument("--impl", default="paris", choices=["paris", "reference"])
    ap.add_argument("--batch", type=int, default=0)
    ap.add_argument("--seed-div", type=int, default=0, help="flat path: seed sample = n / seed_div (0: the library default)")
    ap.add_argument("--index-seeds", type=int, default=0, help="index path: seed series around the leaf")
    ap.add_argument("--both", type=int, default=1, help="also time the other query path (reported as a sub-object)")
    ap.add_argument("--path", default="index", choices=["flat", "index", "nb"],
                    help="flat: paris_knn_exact over the SAX array (ParIS+ Alg9); index: paris_knn_index over "
                         "the iSAX-ordered array with block envelopes (SURVEY f1)")
    ap.add_argument("--n", type=int, default=0, help="override n (debug only)")
    ap.add_argument("--nq", type=int, default=0, help="override query count (debug only)")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--weak", action="store_true",
                    help="one collection of the config's size per rank (weak scaling) instead of one collection "
                         "sharded over the ranks (the default, strong scaling)")
    ap.add_argument("--shard", action="store_true", help="(default) one collection sharded over the ranks")
    ap.add_argument("--no-b1", action="store_true", help="skip the batch-1 LB roofline measurement")
    ap.add_argument("--sorted-refine", action="store_true",
                    help="k = 1: refine bucket-sorted lists (K5 scatter) instead of the unsorted waves (A/B)")
    ap.add_argument("--raw16", action="store_true", help="(default) index path with the bf16 refinement "
                    "pre-filter (paris_raw_bf16 + paris_knn_index_x)")
    ap.add_argument("--no-raw16", action="store_true", help="index path without the bf16 pre-filter")
    ap.add_argument("--paa", type=int, default=-1, choices=[-1, 0, 32, 64],
                    help="index path: the fp16 PAA pre-filter at this many segments (paris_paa_f16 + "
                         "paris_knn_index_aux); -1 (default) = len/4 capped at 64, 0 = off")
    ap.add_argument("--no-sweep", action="store_true", help="skip the C2 k=10 / C5 sigma x k sweeps")
    ap.add_argument("--raw-host", action="store_true",
                    help="f3: keep the raw collection in pinned host memory (SAX/index in HBM)")
    ap.add_argument("--raw-file", default=None,
                    help="f3: write the raw collection to this file, summarize it from disk (O_DIRECT), search "
                         "with the file mapped (SAX/index/bf16 copy in HBM)")
    ap.add_argument("--sigma", type=float, default=None,
                    help="C2/C5: noise of the member queries (hardness; default the config's 0.05)")
    ap.add_argument("--ref-sample", type=int, default=2_000_000)
    ap.add_argument("--ref-queries", type=int, default=4)
    args = ap.parse_args()
    args.warmup = max(args.warmup, 3) if args.impl == "paris" else args.warmup
    if args.impl == "reference":
        return run_reference(args)
    return run_gpu(args)


if __name__ == "__main__":
    sys.exit(main())
