"""Multi-GPU sharding of the render path: one process per GPU, the field replicated,
rays partitioned with NO data-path collective -- frames shard by view (weak scaling) or by
contiguous row band (strong scaling) -- and one final gather of the finished buffers over
NVLink (torch.distributed, NCCL on GPUs; the same code runs on gloo/CPU tensors in the tests).

The reference has no distributed code at all (its only parallelism is a thread pool over row
bands, surface.py:326-333); row bands are the unit it already proves result-invariant.
"""

from __future__ import annotations

import numpy as np


def shard_views(n_views: int, rank: int, world: int) -> list[int]:
    """Round-robin views -> ranks (view v goes to rank v % world)."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    return list(range(rank, n_views, world))


def shard_rows(height: int, rank: int, world: int) -> tuple[int, int]:
    """Contiguous, balanced row band [row0, row1) of rank `rank`; bands tile [0, height) in rank order.
    Ranks beyond the row count get an empty band."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    base, extra = divmod(height, world)
    row0 = rank * base + min(rank, extra)
    return row0, row0 + base + (1 if rank < extra else 0)


def gather_row_bands(local, height: int, group=None):
    """All-gather row bands (first dim = rows of this rank's band) into the full (height, ...) tensor.

    Bands are padded to the largest band so one all_gather_into_tensor moves everything; every
    rank returns the assembled frame.  Works for CUDA tensors over NCCL and CPU tensors over gloo.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    bands = [shard_rows(height, r, world) for r in range(world)]
    if local.shape[0] != bands[rank][1] - bands[rank][0]:
        raise ValueError("local band has the wrong number of rows")
    tallest = max(b[1] - b[0] for b in bands)
    padded = torch.zeros((tallest,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    out = torch.empty((world * tallest,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, padded.contiguous(), group=group)
    pieces = [out[r * tallest : r * tallest + (b[1] - b[0])] for r, b in enumerate(bands)]
    return torch.cat(pieces, dim=0)


def shard_rows_interleaved(height: int, rank: int, world: int, band: int = 32) -> list[tuple[int, int]]:
    """Row bands of `band` rows dealt round-robin: band b = rows [b * band, min((b + 1) * band, height)) goes to rank
    b % world.  Silhouette rows cost several times more than background rows, so contiguous bands leave the
    ranks that own the image centre with most of the work; interleaving evens it out to within one band."""
    if not (0 <= rank < world):
        raise ValueError("rank out of range")
    if band < 1:
        raise ValueError("band must be >= 1")
    n_bands = (height + band - 1) // band
    return [(b * band, min((b + 1) * band, height)) for b in range(rank, n_bands, world)]


def gather_interleaved_bands(local, height: int, band: int = 32, group=None):
    """All-gather buffers whose rows are the concatenation of this rank's shard_rows_interleaved bands into the full
    (height, ...) tensor (rows back in image order), on every rank: one all_gather_into_tensor + one index_select."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    per_rank = [shard_rows_interleaved(height, r, world, band) for r in range(world)]
    rows_of = [sum(b[1] - b[0] for b in bands) for bands in per_rank]
    if local.shape[0] != rows_of[rank]:
        raise ValueError("local buffer has the wrong number of rows")
    tallest = max(rows_of)
    padded = torch.zeros((tallest,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    padded[: local.shape[0]] = local
    out = torch.empty((world * tallest,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out, padded.contiguous(), group=group)
    src = np.empty(height, dtype=np.int64)  # image row -> row of `out`
    for r, bands in enumerate(per_rank):
        at = r * tallest
        for r0, r1 in bands:
            src[r0:r1] = np.arange(at, at + (r1 - r0))
            at += r1 - r0
    return out.index_select(0, torch.as_tensor(src, device=local.device))


def gather_views(local, group=None):
    """All-gather one finished per-rank buffer (e.g. a colour frame) -> (world, ...) on every rank."""
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group)
    out = torch.empty((world,) + tuple(local.shape), dtype=local.dtype, device=local.device)
    dist.all_gather_into_tensor(out.view(world * local.shape[0], *local.shape[1:]) if local.dim() > 0 else out,
                                local.contiguous(), group=group)
    return out


def render_frame_sharded(surface, pose, settings=None, background=(1.0, 1.0, 1.0), supersample: int = 1, group=None,
                         render_rows=None, interleave: int = 0):
    """One frame split into row bands across the ranks of `group`, assembled on every rank.

    Returns (color (H,W,3) f32, depth (H,W) f32, normal (H,W,3) f32, hit (H,W) u8) torch tensors on
    the rank's device.  `render_rows` is injectable so the host logic can be tested without a GPU.
    interleave = 0: one contiguous band per rank (shard_rows); interleave = b > 0: bands of b rows dealt round-robin
    (shard_rows_interleaved) -- better balanced when the object covers only part of the image.
    """
    import torch
    import torch.distributed as dist

    from . import surface as S

    settings = settings or S.RenderSettings()
    render_rows = render_rows or (lambda r0, r1: S.render_rows(surface, pose, settings, background, supersample, r0, r1,
                                                                device_out=True))
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    H = int(pose.height)
    if interleave > 0:
        mine = shard_rows_interleaved(H, rank, world, interleave)
        parts = [render_rows(r0, r1) for r0, r1 in mine]
        if parts:
            local = tuple(torch.cat([p[i] for p in parts], dim=0) for i in range(len(parts[0])))
        else:
            local = tuple(b[:0] for b in render_rows(0, 1))
        return tuple(gather_interleaved_bands(b, H, interleave, group) for b in local)
    r0, r1 = shard_rows(H, rank, world)
    if r1 > r0:
        bands = render_rows(r0, r1)
    else:
        bands = render_rows(0, 1)
        bands = tuple(b[:0] for b in bands)
    return tuple(gather_row_bands(b, H, group) for b in bands)


def render_pathtraced_sharded(scene, pose, spp: int, seed: int, max_bounces: int = 8, sample_offset: int = 0, group=None,
                              interleave: int = 64, pathtrace_rows=None):
    """BASELINE config 5: one path-traced frame split into interleaved row bands across the ranks of `group` (the per-pixel
    counter RNG makes every pixel independent of the banding, pathtrace.py:439-442), hdr radiance assembled on every rank
    with one all_gather.  Returns the (H, W, 3) float64 hdr tensor on the rank's device; `pathtrace_rows(r0, r1)` is
    injectable so the host logic can be tested without a GPU."""
    import torch
    import torch.distributed as dist

    from . import pathtrace as P

    pathtrace_rows = pathtrace_rows or (lambda r0, r1: P.pathtrace_rows(scene, pose, spp, seed, max_bounces, sample_offset, r0, r1,
                                                                        device_out=True))
    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    H = int(pose.height)
    mine = shard_rows_interleaved(H, rank, world, interleave)
    parts = [pathtrace_rows(r0, r1) for r0, r1 in mine]
    local = torch.cat(parts, dim=0) if parts else pathtrace_rows(0, 1)[:0]
    return gather_interleaved_bands(local, H, interleave, group)
