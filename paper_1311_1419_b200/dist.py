"""Sharding of the encode across ranks.

GOPs are independent (every CS frame references only its own GOP's key),
so the path shards without any data exchange.  Two schemes:

* ``shard_streams`` -- weak scaling: rank r encodes its own streams (bench.py default).
* ``shard_gops`` -- one long sequence split into contiguous GOP ranges, encoded per rank with
  ``Encoder.encode_batch_gops``; rank r's measurements are the slice
  ``out[cs_offset(r) : cs_offset(r) + cs_count(r)]`` of the single-device output.

Host logic only (no device code); ``tests/test_dist_gloo.py`` runs it on 2 gloo ranks.
"""
from __future__ import annotations


def n_gops(T: int, G: int) -> int:
    return (T + G - 1) // G


def cs_frames_in_gops(T: int, G: int, g0: int, g1: int) -> int:
    """CS frames of GOPs [g0, g1) of one T-frame stream (short last GOP counted)."""
    return sum(max(0, min(G, T - g * G) - 1) for g in range(g0, g1))


def shard_gops(T: int, G: int, world: int, rank: int):
    """Contiguous GOP range [g0, g1) of `rank`, balanced by CS-frame count."""
    ng = n_gops(T, G)
    total = cs_frames_in_gops(T, G, 0, ng)
    # boundary b_r = first GOP whose cumulative CS count reaches r/world of the total
    bounds = [0]
    acc, g = 0, 0
    for r in range(1, world):
        target = total * r / world
        # take GOP g while its midpoint lies before the target (nearest boundary)
        while g < ng and acc + max(0, min(G, T - g * G) - 1) / 2.0 <= target:
            acc += max(0, min(G, T - g * G) - 1)
            g += 1
        bounds.append(g)
    bounds.append(ng)
    return bounds[rank], bounds[rank + 1]


def cs_offset(T: int, G: int, world: int, rank: int) -> int:
    """Index of rank's first CS frame in the single-device output order (one stream)."""
    g0, _ = shard_gops(T, G, world, rank)
    return cs_frames_in_gops(T, G, 0, g0)


def shard_streams(n_streams: int, world: int, rank: int):
    """Contiguous stream range [s0, s1) of `rank` (balanced)."""
    base, extra = divmod(n_streams, world)
    s0 = rank * base + min(rank, extra)
    return s0, s0 + base + (1 if rank < extra else 0)


def gather_measurements(local, dst: int = 0, group=None):
    """Optional payload gather to one sink (off the encode path): every rank's
    measurement shard (a tensor whose leading dimension is CS frames, same trailing shape on all
    ranks, possibly empty) is concatenated on rank `dst` in rank order -- with shard_gops /
    shard_streams that is the single-device output order.  Works with NCCL (CUDA tensors, over
    NVLink) and gloo (CPU).  Returns the concatenation on `dst`, None on the other ranks."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    n = torch.tensor([local.shape[0]], dtype=torch.int64, device=local.device)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n, group=group)
    sizes = [int(s.item()) for s in sizes]
    mx = max(sizes)
    pad = torch.zeros((mx,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    if local.shape[0]:
        pad[: local.shape[0]] = local
    bufs = [torch.empty_like(pad) for _ in range(world)] if rank == dst else None
    dist.gather(pad, bufs, dst=dst, group=group)
    if rank != dst:
        return None
    return torch.cat([b[:k] for b, k in zip(bufs, sizes)], dim=0)
