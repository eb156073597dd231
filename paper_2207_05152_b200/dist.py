"""Multi-GPU sharding of independent units (images) — one process per GPU.

Units never exchange payload (P:103 lanes are per row, Q16 tiles/images are
independent), so ranks take disjoint contiguous blocks of the batch and code
them on their own device.  The single collective is an all_gather of the
per-image container sizes (north_star: "NCCL is used only for the final gather
of stream sizes"), from which every rank derives the global byte offsets of its
containers in the batch index.  The plan/offset logic is pure Python so it is
tested with the gloo backend on CPU (tests/test_dist.py); the device work is
the C-ABI batch calls.
"""

from __future__ import annotations

import numpy as np


def shard_range(n_units: int, world: int, rank: int):
    """Contiguous block of units for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def global_offsets(all_sizes):
    """Exclusive prefix sum over ranks' size lists (rank-major, unit order)."""
    flat = np.concatenate([np.asarray(s, dtype=np.int64).reshape(-1) for s in all_sizes])
    off = np.zeros(len(flat) + 1, dtype=np.int64)
    np.cumsum(flat, out=off[1:])
    return off


def gather_sizes(local_sizes, group=None):
    """all_gather of per-unit container sizes (int64); the only collective.
    Works on any torch.distributed backend; with NCCL the tensor must be on
    the rank's device.  Ranks may hold different unit counts."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    t = torch.as_tensor(local_sizes, dtype=torch.int64)
    if dist.get_backend(group) == "nccl":
        t = t.cuda()
    n = torch.tensor([t.numel()], dtype=torch.int64, device=t.device)
    ns = [torch.empty_like(n) for _ in range(world)]
    dist.all_gather(ns, n, group=group)
    m = int(max(int(x) for x in ns))
    pad = torch.zeros(m, dtype=torch.int64, device=t.device)
    pad[: t.numel()] = t
    outs = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(outs, pad, group=group)
    return [o[: int(k)].cpu().numpy() for o, k in zip(outs, ns)]


def encode_batch_distributed(encode_shard, images, group=None):
    """Encode `images` (n, H, W) across the ranks of `group`.

    encode_shard(shard) -> list of container bytes (the caller binds the
    device path, e.g. dlic_encode_batch_device on this rank's GPU).
    Returns (my_containers, my_first_unit, offsets) where offsets[i] is the
    global byte offset of unit i in the concatenated batch and offsets[-1] the
    total; every rank can write its containers at its own offsets without any
    payload exchange."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(len(images), world, rank)
    mine = encode_shard(images[lo:hi]) if hi > lo else []
    sizes = gather_sizes([len(b) for b in mine], group)
    return mine, lo, global_offsets(sizes)


def assemble(parts_by_rank, offsets):
    """Concatenate every rank's containers at their offsets (host index)."""
    out = bytearray(int(offsets[-1]))
    i = 0
    for part in parts_by_rank:
        for b in part:
            out[offsets[i]:offsets[i + 1]] = b
            i += 1
    return bytes(out)
