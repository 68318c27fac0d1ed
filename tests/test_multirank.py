"""N > 1 host logic of bench.py on CPU (gloo, world_size 2): weak scaling = distinct
collections per rank, step time = max over ranks, whole-job throughput."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import bench


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        local_ms = [12.5, 20.0][rank]
        mx = bench.reduce_max_ms(local_ms, "cpu", world)
        v = bench.weak_throughput(100, world, mx)
        seeds = bench.rank_seeds(4, rank)
        gathered = [None] * world
        dist.all_gather_object(gathered, seeds)
        q.put((rank, mx, v, gathered))
    finally:
        dist.destroy_process_group()


def test_two_rank_timing_and_seeds():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = [q.get(timeout=120) for _ in range(2)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, mx, v, gathered in res:
        assert mx == 20.0                       # the slowest rank defines the step
        assert v == pytest.approx(100 * 2 / 0.020)
        assert gathered[0] != gathered[1]       # distinct collections / query sets per rank
        assert gathered[0] == bench.rank_seeds(4, 0)


def test_single_rank_is_identity():
    assert bench.reduce_max_ms(7.0, "cpu", 1) == 7.0
    assert bench.weak_throughput(100, 1, 10.0) == pytest.approx(10000.0)


# ---------------------------------------------------------------- sharded exact k-NN (f4)
def _ref_merge(dst, idx):
    """Test-side merge (the product uses paris_merge_topk on the GPU)."""
    R, nq, k = dst.shape
    d = dst.permute(1, 0, 2).reshape(nq, R * k).numpy().astype(np.float64)
    i = idx.permute(1, 0, 2).reshape(nq, R * k).numpy()
    d = np.where(i < 0, np.inf, d)
    out_i = np.empty((nq, k), np.int64)
    out_d = np.empty((nq, k), np.float32)
    for q in range(nq):
        order = np.lexsort((i[q], d[q]))[:k]
        out_i[q], out_d[q] = i[q][order], d[q][order]
    return torch.from_numpy(out_i), torch.from_numpy(out_d)


def _shard_worker(rank, world, port, q, n, k, use_tau=False):
    import datagen
    import oracle
    from paper_2009_00166_b200 import parallel as par
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        lo, hi = par.shard_range(n, rank, world)
        shard = datagen.random_walks(hi - lo, 128, 77, first_id=lo)     # this rank's ids [lo, hi)
        queries = datagen.random_walks(5, 128, 78)
        seen = {}

        def local(qs, kk, tau_in=None):                                # test-side stand-in for the GPU search:
            ri, rd2 = oracle.knn_bruteforce(shard, qs.numpy(), kk)     # the library's tau_in semantics --
            d = np.sqrt(rd2).astype(np.float32)                        # rows beyond the bound come back -1
            if tau_in is not None:
                seen["tau"] = tau_in.numpy().copy()
                out = d > tau_in.numpy()[:, None]
                ri = np.where(out, -1, ri)
                d = np.where(out, np.float32(np.inf), d)
            return torch.from_numpy(ri), torch.from_numpy(d)

        def approx(qs, kk):                                             # a shard's approximate answer: the k-th
            seeds = shard[: 40 + 30 * rank]                             # best of a few of its series (a real bound)
            _, rd2 = oracle.knn_bruteforce(seeds, qs.numpy(), kk)
            tau = torch.from_numpy(np.sqrt(rd2[:, kk - 1]).astype(np.float32))
            seen["own"] = tau.numpy().copy()
            return tau

        gi, gd = par.knn_sharded(torch.from_numpy(queries), k, lo, local, merge=_ref_merge,
                                 approx=approx if use_tau else None)
        q.put((rank, gi.numpy(), gd.numpy(), seen))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("k,use_tau", [(1, False), (7, False), (1, True), (7, True)])
def test_two_rank_sharded_knn_is_exact(k, use_tau):
    """Sharded exact k-NN over gloo (world size 2): with use_tau, the tau_seed exchange --
    every shard's approximate k-th distance, all-reduced with min, bounds every shard's
    search (rows beyond it come back empty) -- must leave the merged answer exact, and both
    ranks must have searched with the same bound, the minimum of their own."""
    import datagen
    import oracle
    from paper_2009_00166_b200 import parallel as par
    n = 3000 + 5
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_shard_worker, args=(r, 2, port, q, n, k, use_tau)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted([q.get(timeout=180) for _ in range(2)], key=lambda t: t[0])
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    full = np.concatenate([datagen.random_walks(hi - lo, 128, 77, first_id=lo)
                           for lo, hi in (par.shard_range(n, r, 2) for r in range(2))])
    assert np.array_equal(full, datagen.random_walks(n, 128, 77))   # shards tile the collection
    ri, rd2 = oracle.knn_bruteforce(full, datagen.random_walks(5, 128, 78), k)
    for _, gi, gd, _ in res:                                        # same answer on every rank
        np.testing.assert_array_equal(gi, ri)
        np.testing.assert_allclose(gd, np.sqrt(rd2), rtol=1e-6)
    if use_tau:
        own = np.minimum(res[0][3]["own"], res[1][3]["own"])
        for _, _, _, seen in res:
            np.testing.assert_array_equal(seen["tau"], own)         # all-reduce(min) of the shards' bounds
        assert not np.array_equal(res[0][3]["own"], res[1][3]["own"])


def test_shard_ranges_partition():
    from paper_2009_00166_b200 import parallel as par
    for n in (1, 15, 16, 1000, 100_003):
        for world in (1, 2, 3, 8):
            rs = [par.shard_range(n, r, world) for r in range(world)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            for (a, b), (c, d) in zip(rs, rs[1:]):
                assert b == c and a <= b
            for lo, hi in rs:
                assert lo % 16 == 0 or lo == hi       # non-empty shards start on a multiple of 16
