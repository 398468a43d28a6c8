"""Multi-NODE plumbing over torch.distributed (NCCL between nodes, gloo in
CPU tests).  Only data movement lives here; all method arithmetic stays in
libmc.so.

Inside one node, ONE multi-GPU handle (mc_config.n_gpus) drives every GPU:
partitions on the devices, the read all-gather over NVLink peer memory and
the hit exchange fused into the merge kernel (libmc.so).
Across nodes, one process per node holds a handle over its node's
partitions (partition_begin / n_local_partitions) and this module moves the
data: a read batch is all-gathered so every node sees every record (the
paper forwards read windows/sketches along a GPU chain), every
node computes its partitions' top-m hits for all records
(mc_query_partials), and one all-to-all sends the hits of record slice h to
node h (the paper merges top lists GPU to GPU), which merges the
lists and classifies its slice (mc_merge_classify).
"""
from __future__ import annotations

import torch
import torch.distributed as dist

HIT_WORDS = 6  # mc_hit = 6 x uint32


def slice_bounds(n: int, world: int, rank: int) -> tuple[int, int]:
    """Record slice [lo, hi) owned by `rank` (equal split, remainder to the first ranks)."""
    q, r = divmod(n, world)
    lo = rank * q + min(rank, r)
    return lo, lo + q + (1 if rank < r else 0)


def _comm_device(t: torch.Tensor, group=None) -> torch.device:
    """gloo moves host tensors only: with a gloo group (CPU tests, or the
    one-GPU rehearsal of the multi-rank bench) device tensors are staged
    through the host; NCCL works on them in place."""
    return torch.device("cpu") if dist.get_backend(group) == "gloo" else t.device


def allgather_records(local: torch.Tensor, counts: list[int], group=None) -> torch.Tensor:
    """Concatenate each rank's fixed-width record block (rows = records) in
    rank order.  `counts[r]` = rows rank r contributes."""
    world = dist.get_world_size(group)
    dev = _comm_device(local, group)
    mx = max(counts)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=dev)
    pad[:local.shape[0]] = local
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    return torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0).to(local.device)


def allgather_flat(buf: torch.Tensor, offs: torch.Tensor, group=None,
                   sizes: list[tuple[int, int]] | None = None) -> tuple[torch.Tensor, torch.Tensor]:
    """Variable-length records: concatenate every rank's flat byte buffer
    (`buf`, uint8) and record offsets (`offs`, int64 [n + 1], offs[0] = 0) in
    rank order.  Returns (all bytes, all offsets) on buf's device.
    sizes: every rank's (records, bytes) when the caller knows them (fixed-
    length reads, a planned batch); then no size exchange and no host
    synchronisation happen.  Otherwise one all-gather of the sizes and one
    device-to-host read of them."""
    world = dist.get_world_size(group)
    dev = _comm_device(buf, group)
    n = offs.numel() - 1
    if sizes is None:
        meta = torch.tensor([n, buf.numel()], dtype=torch.int64, device=dev)
        metas = torch.empty((world, 2), dtype=torch.int64, device=dev)
        dist.all_gather_into_tensor(metas, meta, group=group) if dev.type != "cpu" else \
            dist.all_gather(list(metas.unbind(0)), meta, group=group)
        sizes = [tuple(x) for x in metas.tolist()]  # (the one host synchronisation)
    ns = [int(x[0]) for x in sizes]
    nb = [int(x[1]) for x in sizes]
    pb = torch.zeros(max(max(nb), 1), dtype=buf.dtype, device=dev)
    pb[:buf.numel()] = buf
    po = torch.zeros(max(ns) + 1, dtype=torch.int64, device=dev)
    po[:n + 1] = offs
    bparts = [torch.empty_like(pb) for _ in range(world)]
    oparts = [torch.empty_like(po) for _ in range(world)]
    dist.all_gather(bparts, pb, group=group)
    dist.all_gather(oparts, po, group=group)
    base, outs = 0, [torch.zeros(1, dtype=torch.int64, device=dev)]
    for r in range(world):
        outs.append(oparts[r][1:ns[r] + 1] + base)
        base += nb[r]
    all_buf = torch.cat([bparts[r][:nb[r]] for r in range(world)])
    return all_buf.to(buf.device), torch.cat(outs).to(buf.device)


def exchange_hits(hits: torch.Tensor, n: int, group=None) -> torch.Tensor:
    """hits: int32 [n, m * 6] -- this rank's partition top-m for ALL n records.
    Returns int32 [n_mine, world, m * 6]: for this rank's record slice, the
    lists of every partition in rank order (mc_merge_classify's layout)."""
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    width = hits.shape[1]
    bounds = [slice_bounds(n, world, r) for r in range(world)]
    in_splits = [hi - lo for lo, hi in bounds]
    lo, hi = bounds[rank]
    dev = _comm_device(hits, group)
    out = torch.empty(((hi - lo) * world, width), dtype=hits.dtype, device=dev)
    dist.all_to_all_single(out, hits.contiguous().to(dev), output_split_sizes=[hi - lo] * world,
                           input_split_sizes=in_splits, group=group)
    return out.view(world, hi - lo, width).transpose(0, 1).contiguous().to(hits.device)
