"""Multi-GPU decomposition of the trace transform.

One process per GPU (torchrun); the data path is the fused kernel on each
rank plus ONE collective: the all-gather that assembles the sinogram.

Orientation sharding keeps the kernel's mirror pairing: rank r of G owns the
angle block [a0, a0+cnt) of the first half AND its mirror block
[A/2+a0, A/2+a0+cnt), launched as one tt_trace_device call with
pair_stride = A/2 (rows [cnt] + [cnt]).  The mirrored line of a pair reuses
the same taps, so a shard costs half the sampling of two unpaired blocks, and
every shard is bit-identical to the corresponding rows of a single launch.

Image sharding (feature extraction, config C4) gives each rank whole images;
only per-image features are gathered.
"""
from __future__ import annotations


def orientation_shard(angles: int, world: int, rank: int):
    """(a0, cnt, pair_stride) of rank's shard: angles a0..a0+cnt-1 and their
    mirrors a0+A/2..; requires an even angle count."""
    if angles % 2:
        raise ValueError("orientation sharding pairs theta with theta+pi: the angle count must be even")
    h = angles // 2
    a0 = rank * h // world
    cnt = (rank + 1) * h // world - a0
    return a0, cnt, h


def shard_rows(angles: int, world: int, rank: int):
    """Angle index of each output row of rank's shard."""
    a0, cnt, h = orientation_shard(angles, world, rank)
    return list(range(a0, a0 + cnt)) + list(range(h + a0, h + a0 + cnt))


def assemble(gathered, angles: int, world: int):
    """Reorder an all-gathered [world * 2cnt, ...] tensor (equal shards) into
    angle order [angles, ...] (returns a new tensor)."""
    h = angles // 2
    if h % world:
        raise ValueError("equal shards need (angles/2) % world == 0")
    cnt = h // world
    rest = tuple(gathered.shape[1:])
    return gathered.reshape(world, 2, cnt, *rest).transpose(0, 1).reshape(angles, *rest)


def gather_sinograms(local, angles: int, dist, group=None, out=None, raw=None):
    """The single collective of the orientation-sharded transform: all-gather
    every rank's [2cnt, F, n] block (NCCL over NVLink on GPUs, gloo on CPU)
    and assemble [angles, F, n]."""
    import torch

    world = dist.get_world_size(group)
    if raw is None:
        raw = torch.empty((world * local.shape[0],) + tuple(local.shape[1:]), dtype=local.dtype,
                          device=local.device)
    dist.all_gather_into_tensor(raw, local.contiguous(), group=group)
    full = assemble(raw, angles, world)
    if out is not None:
        out.copy_(full)
        return out
    return full


def image_shard(images: int, world: int, rank: int):
    """Contiguous block of image indices for rank (batched feature extraction)."""
    lo = rank * images // world
    return lo, (rank + 1) * images // world - lo


def direct_shard_rows(angles: int, world: int, rank: int, F: int, n: int):
    """Launch geometry of rank's orientation shard written straight into the
    full [angles][F][n] sinogram (and [angles][2][n] medians): returns
    (a0, a_count, pair_stride, row0, partner_row) for tt_trace_device with
    out = base + row0 rows and partner_row = angles / 2."""
    a0, cnt, h = orientation_shard(angles, world, rank)
    return a0, 2 * cnt, h, a0, h


def share_device_buffers(ptrs, dist, device: int, src: int = 0, group=None):
    """Rank `src` exports its device pointers (CUDA IPC handles), every rank
    maps them (peer access over NVLink / NVSwitch).  Returns (pointers,
    close) where close() unmaps the imported ones.  The fused kernel then
    writes each shard's rows directly into rank src's buffers: the sinogram
    assembly needs no gather collective, only a completion signal."""
    from . import trace as _tr

    rank = dist.get_rank(group)
    handles = [[_tr.ipc_export(p) for p in ptrs] if rank == src else None]
    dist.broadcast_object_list(handles, src=src, group=group)
    if rank == src:
        return list(ptrs), (lambda: None)
    mapped = [_tr.ipc_import(h, device) for h in handles[0]]

    def close():
        for p in mapped:
            _tr.ipc_close(p)
    return mapped, close
