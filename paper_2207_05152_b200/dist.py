"""Multi-GPU sharding of independent units — one process per GPU.

Units never exchange payload: the rANS coder instances are per pixel row
 and tiles/images are independent units with fill 0 at their borders
(reading Q16), so ranks take disjoint contiguous blocks of units and code them
on their own device.  The single collective is an all_gather of container (or
stream) sizes (north_star: "NCCL is used only for the final gather of stream
sizes"), from which every rank derives the global byte offsets of its output.

Two granularities, both used by bench.py and covered by the world-size-2 gloo
tests (tests/test_dist.py) with the same functions:
  * coded_step      -- weak scaling: every rank codes its own batch of images
                       (device batch API); per step one all_gather of the
                       per-image container sizes, on the device (no host sync);
  * encode_units_distributed / decode_units_distributed -- one image's tiles
                       split across ranks (C4: "tiled into independent streams
                       across 1/2/4/8 B200"): each rank codes a unit range
                       (dlic_encode_units), the per-stream sizes are gathered,
                       and any rank frames the container (dlic_container_build).
The coding itself is passed in as callables, so the same code runs with the
C-ABI on GPUs and with the oracle under gloo on CPU.
"""

from __future__ import annotations

import numpy as np


def shard_range(n_units: int, world: int, rank: int):
    """Contiguous block of units for `rank` (sizes differ by at most one)."""
    base, extra = divmod(n_units, world)
    lo = rank * base + min(rank, extra)
    return lo, lo + base + (1 if rank < extra else 0)


def global_offsets(all_sizes):
    """Exclusive prefix sum over ranks' size lists (rank-major, unit order);
    the last entry is the total."""
    flat = np.concatenate([np.asarray(s, dtype=np.int64).reshape(-1) for s in all_sizes])
    off = np.zeros(len(flat) + 1, dtype=np.int64)
    np.cumsum(flat, out=off[1:])
    return off


def gather_sizes(local_sizes, group=None):
    """all_gather of per-unit sizes (int64) when ranks hold DIFFERENT counts
    (host lists in, host arrays out).  Works on any backend; with NCCL the
    tensors live on the rank's device."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    dev = torch.device("cuda", torch.cuda.current_device()) if dist.get_backend(group) == "nccl" else None
    t = torch.as_tensor(np.asarray(local_sizes, dtype=np.int64), dtype=torch.int64, device=dev)
    n = torch.tensor([t.numel()], dtype=torch.int64, device=dev)
    ns = torch.empty(world, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(ns, n, group=group)
    counts = [int(x) for x in ns.cpu()]
    m = max(counts)
    pad = torch.zeros(m, dtype=torch.int64, device=dev)
    pad[: t.numel()] = t
    out = torch.empty(world * m, dtype=torch.int64, device=dev)
    dist.all_gather_into_tensor(out, pad, group=group)
    out = out.cpu().numpy().reshape(world, m)
    return [out[r, :counts[r]] for r in range(world)]


def exchange_sizes_device(d_sizes, group=None):
    """The weak-scaling step's only collective: all_gather of this rank's
    per-image container sizes (equal counts on every rank), tensor in, tensor
    out (world, n), stream-ordered -- no host synchronisation."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    src = d_sizes.contiguous().reshape(-1)
    out = torch.empty(world * src.numel(), dtype=src.dtype, device=src.device)
    dist.all_gather_into_tensor(out, src, group=group)
    return out.view((world,) + tuple(d_sizes.shape))


def offsets_device(all_sizes):
    """Exclusive scan of the gathered (world, n) sizes in rank-major order
    (each rank's byte offset of its containers in the job's output)."""
    flat = all_sizes.reshape(-1)
    return flat.cumsum(0) - flat


def coded_step(encode_local, decode_local, group=None):
    """One weak-scaling step on this rank: encode_local() codes the rank's
    batch and returns its per-image sizes (a tensor); the sizes are
    all-gathered and scanned into global offsets (the only exchange); then
    decode_local() decodes the rank's containers.  Returns (all_sizes,
    offsets) as tensors."""
    sizes = encode_local()
    all_sizes = exchange_sizes_device(sizes, group)
    offs = offsets_device(all_sizes)
    decode_local()
    return all_sizes, offs


def encode_units_distributed(encode_units, n_units: int, group=None):
    """One image's units split across the ranks of `group`.

    encode_units(lo, hi) -> (payload bytes, per-stream sizes) codes units
    [lo, hi) (dlic_encode_units on this rank's GPU).  The per-stream sizes
    are all-gathered (the only exchange).  Returns (my_payload, (lo, hi),
    stream_offsets, all_stream_sizes): stream_offsets[k] is the payload byte
    offset of stream k (the last entry the payload total), so every rank knows
    where its payload goes; any rank frames the header from all_stream_sizes
    (dlic_container_build) without seeing another rank's payload."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    lo, hi = shard_range(n_units, world, rank)
    payload, ssz = encode_units(lo, hi) if hi > lo else (b"", [])
    all_ssz = gather_sizes(ssz, group)
    return payload, (lo, hi), global_offsets(all_ssz), np.concatenate([np.asarray(s, np.int64) for s in all_ssz])


def assemble(parts_by_rank, offsets):
    """Concatenate every rank's containers at their offsets (host index)."""
    out = bytearray(int(offsets[-1]))
    i = 0
    for part in parts_by_rank:
        for b in part:
            out[offsets[i]:offsets[i + 1]] = b
            i += 1
    return bytes(out)


def decode_units_distributed(decode_units, n_units: int, group=None):
    """Each rank decodes its unit range of one container (no exchange);
    decode_units(lo, hi) writes those units' pixels.  Returns the range."""
    import torch.distributed as dist

    lo, hi = shard_range(n_units, dist.get_world_size(group), dist.get_rank(group))
    if hi > lo:
        decode_units(lo, hi)
    return lo, hi
