"""Multi-GPU exact k-NN over one sharded collection.

The collection is split by series-id range across the ranks of a process group
(one process per GPU); every rank keeps its shard's raw series and SAX array /
index in its own HBM.  A query batch is answered by:

  1. every rank searching its shard with the single-GPU path (libparis kernels),
     ids offset by the shard base;
  2. ONE exchange: an all-gather of the per-rank rows (nq x k distances + ids,
     a few KB per batch over NVLink/NVSwitch);
  3. an exact merge on the GPU (``paris_merge_topk``): each true top-k member is
     in the top-k of its own shard, so the global k best are among the R*k rows.

Plumbing only (torch.distributed for the collective, NCCL on GPUs); the search and
the merge run in libparis.  ``local`` / ``merge`` may be injected -- the CPU
multi-rank tests (gloo) exercise the exchange and the id bookkeeping with
test-side stand-ins, since the kernels need a GPU.
"""
from __future__ import annotations

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


def knn_sharded(queries: torch.Tensor, k: int, shard_base: int, local, group=None, merge=None):
    """Exact k-NN of `queries` over the union of all ranks' shards.

    local(queries, k) -> (idx [nq][k] int64 shard-local ids (-1 = none), dist [nq][k] float32)
    merge(dist [R][nq][k], idx [R][nq][k]) -> (idx [nq][k], dist [nq][k]); default paris_merge_topk.
    Returns (idx, dist) with global ids, identical on every rank.
    """
    idx, dst = local(queries, k)
    gidx = torch.where(idx >= 0, idx + int(shard_base), idx)
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    if world == 1:
        all_idx, all_dst = gidx.unsqueeze(0), dst.unsqueeze(0)
    else:
        li = [torch.empty_like(gidx) for _ in range(world)]
        ld = [torch.empty_like(dst) for _ in range(world)]
        dist.all_gather(li, gidx.contiguous(), group=group)
        dist.all_gather(ld, dst.contiguous(), group=group)
        all_idx, all_dst = torch.stack(li), torch.stack(ld)
    merge = merge or B.merge_topk
    return merge(all_dst.contiguous(), all_idx.contiguous())


def local_index_search(raw_shard: torch.Tensor, index, config=None):
    """`local` for knn_sharded over a shard indexed with paris_index_build."""
    def run(queries, k):
        return B.knn_index(raw_shard, index, queries, k=k, config=config)
    return run


def local_flat_search(raw_shard: torch.Tensor, sax_shard: torch.Tensor, w: int = 16, card: int = 256,
                      config=None):
    """`local` for knn_sharded over a shard's flat SAX array (paris_knn_exact)."""
    def run(queries, k):
        return B.knn_exact(raw_shard, sax_shard, queries, k=k, w=w, card=card, config=config)
    return run
