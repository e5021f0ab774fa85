"""A12 — shard and gather across GPUs (BASELINE.json north_star).

Clusters are independent units of C-BFS (P:1004 loops them one after the
other; nothing crosses between two clusters' traversals), so the multi-GPU
path has no per-round exchange: the graph is replicated on every rank and
cluster c goes to rank c mod R (round-robin balances the degree-ordered
selection, whose early clusters are the largest).  NCCL (torch.distributed)
is used only at the end, in one of two ways:

  * gather_label_images — the boundary's way: each rank builds
    a cbfs_labels handle of its clusters, exports its flat image, the images
    are all-gathered and imported as one handle per rank;
  * gather_labels — the same with raw tensors: each rank
    builds the labels of its clusters with cbfs_run (planes = d, P:1438-1447,
    R14) and the shards are all-gathered; a gathered store is R shards of the
    cbfs_run layout, and cbfs_query_distance min-merges over them one by one
    (the query is a min over clusters, so the cluster order does
    not matter).
  * query_stream_sharded — the store cannot be resident (config 5, H3): each
    rank streams its clusters through cbfs_query_stream and the partial
    answers are MIN-all-reduced.

Argument marshalling only: every step of the path runs in libcbfs.so; this
module holds the partition rule and the collectives.  The partition rule and
the reductions are plain functions so that the world-size-2 gloo tests in
tests/test_dist_cpu.py can check them on CPU.
"""
from __future__ import annotations

import torch
import torch.distributed as dist

from . import (CBFS_QUERY_UNREACHED, CBFS_UNREACHED_U8, CBFS_UNREACHED_U16, cbfs_labels_build, cbfs_labels_export,
               cbfs_labels_import, cbfs_labels_info, cbfs_labels_query, cbfs_query_distance, cbfs_query_stream,
               cbfs_run)


def cluster_shard(n_clusters: int, world: int, rank: int) -> torch.Tensor:
    """Indices of the clusters rank `rank` owns: c = rank, rank + R, ...."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return torch.arange(rank, max(rank, n_clusters), world, dtype=torch.int64)


def shard_width(n_clusters: int, world: int) -> int:
    """Columns of every rank's label shard (equal shapes for all_gather; ranks
    with fewer clusters pad with unreachable columns that the query skips, R16)."""
    return (n_clusters + world - 1) // world


def _world(group):
    return dist.get_world_size(group), dist.get_rank(group)


def local_clusters(sources: torch.Tensor, sizes: torch.Tensor, group=None):
    """This rank's rows of the (replicated) selection."""
    world, rank = _world(group)
    idx = cluster_shard(int(sizes.shape[0]), world, rank).to(sources.device)
    return sources.index_select(0, idx).contiguous(), sizes.index_select(0, idx).contiguous()


def build_label_shard(graph, sources: torch.Tensor, sizes: torch.Tensor, d: int, dist_bytes: int = 2, group=None,
                      stream=None):
    """Labels (Delta + S_v[0..d-1], R14) of this rank's clusters in the cbfs_run
    layout, padded to shard_width columns.  Returns (dist [n][W], masks
    [d][n][W], sizes [W])."""
    world, _ = _world(group)
    src_r, sz_r = local_clusters(sources, sizes, group)
    W = shard_width(int(sizes.shape[0]), world)
    dev = sources.device
    n = graph.n
    planes = d if d > 0 else 1
    dist_t = torch.empty((n, W), dtype=torch.uint8 if dist_bytes == 1 else torch.int16, device=dev)
    masks = torch.zeros((planes, n, W), dtype=torch.int64, device=dev)
    szp = torch.ones((W,), dtype=torch.uint8, device=dev)
    C = int(sz_r.shape[0])
    if C == W:
        cbfs_run(graph.h, src_r, sz_r, C, d, dist_bytes, dist_t, masks, planes, None, 0, stream)
        szp.copy_(sz_r)
    else:  # ragged last shard: run into a [n][C] buffer, pad to W unreachable columns
        dist_t.fill_(CBFS_UNREACHED_U8 if dist_bytes == 1 else -1)  # 0xFFFF as int16
        if C:
            dc = torch.empty((n, C), dtype=dist_t.dtype, device=dev)
            mc = torch.empty((planes, n, C), dtype=torch.int64, device=dev)
            cbfs_run(graph.h, src_r, sz_r, C, d, dist_bytes, dc, mc, planes, None, 0, stream)
            dist_t[:, :C].copy_(dc)
            masks[:, :, :C].copy_(mc)
            szp[:C].copy_(sz_r)
    return dist_t, masks, szp


def all_gather_shards(tensors, group=None):
    """all_gather each tensor of `tensors` (same shape on every rank); returns
    per tensor a list of R shards, rank order."""
    world, _ = _world(group)
    out = []
    for x in tensors:
        # moved as raw bytes: NCCL has no 16-bit integer type (u16 Delta, R10)
        xb = x.contiguous().view(torch.uint8)
        parts = [torch.empty_like(xb) for _ in range(world)]
        dist.all_gather(parts, xb, group=group)
        out.append([p.view(x.dtype) for p in parts])
    return out


def gather_labels(dist_t: torch.Tensor, masks: torch.Tensor, sizes: torch.Tensor, group=None):
    """All-gather the label shards (NCCL over NVLink on GPUs): returns a list of
    R (dist, masks, sizes) shards, every one a label store in the cbfs_run
    layout."""
    d_parts, m_parts, s_parts = all_gather_shards([dist_t, masks, sizes], group)
    return list(zip(d_parts, m_parts, s_parts))


def query_gathered(stores, d: int, s: torch.Tensor, t: torch.Tensor, dist_bytes: int = 2, stream=None):
    """cbfs_query_distance over every gathered shard, min-merged (R15, R16)."""
    best = torch.full((int(s.shape[0]),), CBFS_QUERY_UNREACHED, dtype=torch.int32, device=s.device)
    for dist_t, masks, sizes in stores:
        n, W = int(dist_t.shape[0]), int(dist_t.shape[1])
        cbfs_query_distance(n, W, d, int(masks.shape[0]), dist_t, dist_bytes, masks, sizes, s, t, best, stream)
    return best


def build_local_labels(graph, sources: torch.Tensor, sizes: torch.Tensor, d: int, dist_bytes: int = 2, group=None,
                       word_bits: int = 64):
    """This rank's label store as a cbfs_labels handle (cbfs_labels_build_w
    over its round-robin clusters, store word size word_bits)."""
    src_r, sz_r = local_clusters(sources, sizes, group)
    return cbfs_labels_build(graph.h, src_r, sz_r, int(sz_r.shape[0]), d, dist_bytes, word_bits=word_bits)


def gather_label_images(graph, labels, group=None):
    """cbfs_labels_export -> NCCL all_gather of the flat
    images (padded to the largest; the header carries each image's size) ->
    cbfs_labels_import.  Returns one handle per rank, rank order."""
    world, _ = _world(group)
    size = cbfs_labels_info(labels)["image_bytes"]
    dev = torch.device(f"cuda:{graph.device}") if torch.cuda.is_available() else torch.device("cpu")
    sizes = [torch.zeros(1, dtype=torch.int64, device=dev) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([size], dtype=torch.int64, device=dev), group=group)
    top = int(max(int(x.item()) for x in sizes))
    img = torch.zeros(top, dtype=torch.uint8, device=dev)
    cbfs_labels_export(labels, img[:size])
    parts = [torch.empty_like(img) for _ in range(world)]
    dist.all_gather(parts, img, group=group)
    return [cbfs_labels_import(graph.h, p[:int(sz.item())]) for p, sz in zip(parts, sizes)]


def query_label_handles(handles, s: torch.Tensor, t: torch.Tensor) -> torch.Tensor:
    """cbfs_labels_query over every gathered store, min-merged (R15, R16)."""
    best = torch.full((int(s.shape[0]),), CBFS_QUERY_UNREACHED, dtype=torch.int32, device=s.device)
    for h in handles:
        cbfs_labels_query(h, s, t, best)
    return best


def query_block(q: int, world: int, rank: int):
    """[lo, hi) of the contiguous block of q queries rank `rank` answers, and
    the common block length (equal shapes for all_gather)."""
    per = (q + world - 1) // world if world else q
    lo = min(rank * per, q)
    return lo, min(lo + per, q), per


def query_index_sharded(answer_fn, s: torch.Tensor, t: torch.Tensor, group=None) -> torch.Tensor:
    """once every rank holds every label store (the
    all-gather above), the queries are sharded by index — rank r answers its
    contiguous block with answer_fn(s_block, t_block) (e.g. a
    query_label_handles closure) — and the int32 blocks are all-gathered, so
    every rank ends with all q answers."""
    world, rank = _world(group)
    q = int(s.shape[0])
    lo, hi, per = query_block(q, world, rank)
    mine = torch.full((per,), CBFS_QUERY_UNREACHED, dtype=torch.int32, device=s.device)
    if hi > lo:
        mine[:hi - lo] = answer_fn(s[lo:hi], t[lo:hi])
    if world == 1:
        return mine[:q]
    parts = [torch.empty_like(mine) for _ in range(world)]
    dist.all_gather(parts, mine, group=group)
    return torch.cat(parts)[:q]


def min_reduce_answers(best: torch.Tensor, group=None) -> torch.Tensor:
    """MIN all-reduce of per-rank partial answers (int32, CBFS_QUERY_UNREACHED =
    no cluster reached both ends), in place."""
    dist.all_reduce(best, op=dist.ReduceOp.MIN, group=group)
    return best


def query_stream_sharded(graph, sources: torch.Tensor, sizes: torch.Tensor, d: int, s: torch.Tensor,
                         t: torch.Tensor, group=None, stream=None, out_stats=None) -> torch.Tensor:
    """Config-5 path (H3): this rank streams its clusters through
    cbfs_query_stream, then the answers are MIN-all-reduced over ranks."""
    src_r, sz_r = local_clusters(sources, sizes, group)
    best = torch.full((int(s.shape[0]),), CBFS_QUERY_UNREACHED, dtype=torch.int32, device=s.device)
    if int(sz_r.shape[0]):
        cbfs_query_stream(graph.h, src_r, sz_r, int(sz_r.shape[0]), d, s, t, best, out_stats, stream)
    return min_reduce_answers(best, group)


__all__ = ["cluster_shard", "shard_width", "local_clusters", "build_label_shard", "all_gather_shards",
           "gather_labels", "query_gathered", "build_local_labels", "gather_label_images", "query_label_handles",
           "min_reduce_answers", "query_stream_sharded", "query_block", "query_index_sharded", "CBFS_UNREACHED_U16"]
