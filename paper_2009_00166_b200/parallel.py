"""Multi-GPU exact k-NN over one sharded collection.

The collection is split by series-id range across the ranks of a process group
(one process per GPU); every rank keeps its shard's raw series and SAX array /
index in its own HBM.  A query batch is answered by:

  0. (optional) every rank's approximate answer bounds the k-th NN distance; an
     all-reduce(min) of these per-query bounds (nq floats) lets every shard prune against
     the best seed of any shard (Alg9's shared BSF, across GPUs);
  1. every rank searching its shard with the single-GPU path (libparis kernels),
     ids offset by the shard base;
  2. an exchange of the results: an all-gather of the per-rank rows (nq x k distances + ids,
     a few KB per batch over NVLink/NVSwitch);
  3. an exact merge on the GPU (``paris_merge_topk``): each true top-k member is
     in the top-k of its own shard, so the global k best are among the R*k rows.

Plumbing only (torch.distributed for the collective, NCCL on GPUs); the search and
the merge run in libparis.  ``local`` / ``merge`` may be injected -- the CPU
multi-rank tests (gloo) exercise the exchange and the id bookkeeping with
test-side stand-ins, since the kernels need a GPU.
"""
from __future__ import annotations

import dataclasses

import torch
import torch.distributed as dist

from . import _binding as B


def shard_range(n_total: int, rank: int, world: int, align: int = 16):
    """[lo, hi) of the series ids held by `rank` (contiguous, multiples of `align`
    except the last shard, so each shard keeps the tiled/indexed fast paths)."""
    per = (n_total + world - 1) // world
    per = (per + align - 1) // align * align
    lo = min(n_total, rank * per)
    hi = min(n_total, lo + per)
    return lo, hi


def exchange_tau(tau: torch.Tensor, group=None) -> torch.Tensor:
    """All-reduce(min) of per-query bounds of the k-th NN distance: each shard's approximate
    answer bounds the GLOBAL k-th distance from above (its k seeds are real series), so the
    minimum over shards does too -- Alg9's shared BSF lifted to N GPUs."""
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        tau = tau.clone()
        dist.all_reduce(tau, op=dist.ReduceOp.MIN, group=group)
    return tau


def knn_sharded(queries: torch.Tensor, k: int, shard_base: int, local, group=None, merge=None, approx=None):
    """Exact k-NN of `queries` over the union of all ranks' shards.

    approx(queries, k) -> tau [nq] float32: this shard's bound of the k-th NN distance (its
        approximate answer's k-th distance, paris_knn_index_approx); when given, the bounds are
        all-reduced with min before the search (the tau_seed exchange of SURVEY §8(e) step 1),
        so every shard prunes against the best seed of all shards.
    local(queries, k, tau_in) -> (idx [nq][k] int64 shard-local ids (-1 = none), dist [nq][k] float32);
        tau_in: None, or the exchanged bounds (rows with no local series within them come back -1).
    merge(dist [R][nq][k], idx [R][nq][k]) -> (idx [nq][k], dist [nq][k]); default paris_merge_topk.
    Returns (idx, dist) with global ids, identical on every rank.
    """
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    tau = None
    if approx is not None and world > 1:
        tau = exchange_tau(approx(queries, k).contiguous(), group)
    idx, dst = local(queries, k, tau)
    gidx = torch.where(idx >= 0, idx + int(shard_base), idx)
    if world == 1:
        return gidx, dst  # one shard: its rows are the answer (no exchange, no merge)
    li = [torch.empty_like(gidx) for _ in range(world)]
    ld = [torch.empty_like(dst) for _ in range(world)]
    dist.all_gather(li, gidx.contiguous(), group=group)
    dist.all_gather(ld, dst.contiguous(), group=group)
    all_idx, all_dst = torch.stack(li), torch.stack(ld)
    merge = merge or B.merge_topk
    return merge(all_dst.contiguous(), all_idx.contiguous())


def local_index_search(raw_shard: torch.Tensor, index, config=None, raw16=None, paa16=None):
    """`local` for knn_sharded over a shard indexed with paris_index_build (with the bf16 / PAA
    refinement pre-filters when given, as the single-GPU bench path)."""
    def run(queries, k, tau_in=None):
        cfg = config
        if tau_in is not None:
            cfg = dataclasses.replace(config or B.KnnConfig(), tau_in=tau_in)
        return B.knn_index(raw_shard, index, queries, k=k, config=cfg, raw16=raw16, paa16=paa16)
    return run


def approx_index_search(raw_shard: torch.Tensor, index, config=None):
    """`approx` for knn_sharded: this shard's approximate k-NN (paris_knn_index_approx); the
    k-th distance bounds the k-th NN distance of the whole collection from above."""
    def run(queries, k):
        _, d = B.knn_approx(raw_shard, None, queries, k=k, index=index, config=config)
        return d[:, k - 1].contiguous()
    return run


def local_flat_search(raw_shard: torch.Tensor, sax_shard: torch.Tensor, w: int = 16, card: int = 256,
                      config=None):
    """`local` for knn_sharded over a shard's flat SAX array (paris_knn_exact)."""
    def run(queries, k, tau_in=None):
        cfg = config
        if tau_in is not None:
            cfg = dataclasses.replace(config or B.KnnConfig(), tau_in=tau_in)
        return B.knn_exact(raw_shard, sax_shard, queries, k=k, w=w, card=card, config=cfg)
    return run
