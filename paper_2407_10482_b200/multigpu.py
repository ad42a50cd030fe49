"""Multi-GPU plumbing for the render path.

Rays are independent and the scene is read-only, so the
path shards with no data-path collective: every rank holds a scene replica
and renders its own cameras (camera-batch sharding) or its own interleaved
pixel tiles of one frame (tile sharding). The only exchange is the gather of
finished frames/tiles to rank 0 over NCCL (torch.distributed; gloo on CPU for
the tests). Gathered images are byte-identical to a 1-GPU render because each
pixel is computed by exactly one rank with the same kernels.
"""
from __future__ import annotations

import torch
import torch.distributed as dist


def camera_of(rank: int, world: int, step: int, n_cams: int) -> int:
    """Camera-batch sharding: rank r renders camera (r + N*step) mod n_cams."""
    return (rank + world * step) % n_cams


def cameras_for_rank(rank: int, world: int, n_cams: int) -> list[int]:
    """All cameras of an n_cams batch owned by `rank` (round robin)."""
    return list(range(rank, n_cams, world))


def tile_windows(width: int, height: int, tile: int, rank: int, world: int):
    """Interleaved tile sharding of one frame: tiles (tile x tile pixels, row-major)
    assigned round robin; returns this rank's windows (x0, y0, w, h)."""
    out = []
    nx = (width + tile - 1) // tile
    ny = (height + tile - 1) // tile
    for t in range(rank, nx * ny, world):
        tx, ty = t % nx, t // nx
        x0, y0 = tx * tile, ty * tile
        out.append((x0, y0, min(tile, width - x0), min(tile, height - y0)))
    return out


def gather_frames(frame: torch.Tensor, world: int, dst: int = 0, bufs=None,
                  async_op: bool = False):
    """Gather one equally-shaped frame per rank to `dst` (NCCL gather). Returns the
    list of frames on dst, None elsewhere; with async_op, (list, work) where
    work.wait() orders the caller's current stream after the transfer (NCCL) so a
    render enqueued before the wait overlaps the gather of an earlier frame."""
    if world == 1:
        return ([frame], None) if async_op else [frame]
    rank = dist.get_rank()
    if rank == dst and bufs is None:
        bufs = [torch.empty_like(frame) for _ in range(world)]
    work = dist.gather(frame, gather_list=bufs if rank == dst else None, dst=dst,
                       async_op=async_op)
    out = bufs if rank == dst else None
    return (out, work) if async_op else out


def assemble_tiles(tiles_by_rank, width: int, height: int, tile: int, world: int,
                   channels: int = 3, device=None):
    """Rebuild a full frame from per-rank tile lists (as produced by tile_windows)."""
    img = torch.zeros((height, width, channels), dtype=torch.float32, device=device)
    for r in range(world):
        wins = tile_windows(width, height, tile, r, world)
        for (x0, y0, w, h), t in zip(wins, tiles_by_rank[r]):
            img[y0:y0 + h, x0:x0 + w] = t.reshape(h, w, channels)
    return img


def gather_tiles(tiles: list[torch.Tensor], width: int, height: int, tile: int, world: int,
                 dst: int = 0):
    """Gather interleaved tiles to dst as one flat buffer per rank (padded to the
    largest rank payload) and assemble the frame there."""
    rank = dist.get_rank() if world > 1 else 0
    flat = torch.cat([t.reshape(-1) for t in tiles]) if tiles else torch.zeros(0)
    if world == 1:
        return assemble_tiles([tiles], width, height, tile, 1, device=flat.device)
    sizes = [sum(w * h * 3 for (_, _, w, h) in tile_windows(width, height, tile, r, world))
             for r in range(world)]
    cap = max(sizes)
    buf = torch.zeros(cap, dtype=torch.float32, device=flat.device)
    buf[: flat.numel()] = flat
    got = [torch.empty_like(buf) for _ in range(world)] if rank == dst else None
    dist.gather(buf, gather_list=got, dst=dst)
    if rank != dst:
        return None
    per_rank = []
    for r in range(world):
        wins = tile_windows(width, height, tile, r, world)
        off, lst = 0, []
        for (_, _, w, h) in wins:
            lst.append(got[r][off: off + w * h * 3])
            off += w * h * 3
        per_rank.append(lst)
    return assemble_tiles(per_rank, width, height, tile, world, device=flat.device)
