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


# ---------------------------------------------------------------------------
# Single-launch interleaved-tile sharding (ngprt_render_opts.shard_*)
# ---------------------------------------------------------------------------
def render_tile_shard(scene, cams, opts, rank: int, world: int, tile: int = 32, out=None,
                      stats: bool = False, stream=None):
    """This rank's interleaved tiles of every camera in ONE ngprt_render call (one
    K0/K1/K2 launch): a compact (n_cams, P, 3) buffer, P = shard_pixels(w, h,
    world, tile); local tile j is global tile rank + j * world."""
    from dataclasses import replace
    from . import renderer
    o = replace(opts or renderer.Opts(), shard_world=world, shard_rank=rank, shard_tile=tile)
    return renderer.render(scene, cams, o, out=out, stats=stats, stream=stream)


def gather_tile_shards(shard: torch.Tensor, world: int, width: int, height: int, tile: int = 32,
                       dst: int = 0, bufs=None, async_op: bool = False):
    """Gather every rank's compact shard (n_cams, P, C) to `dst` into one contiguous
    (world, n_cams, P, C) buffer (NCCL gather; equal sizes, no padding step) and
    de-interleave it there with the ngprt_shard_assemble kernel. Returns the
    (n_cams, h, w, C) frames on dst, None elsewhere. With async_op the assembly is
    left to the caller: returns (bufs, work)."""
    from . import renderer
    n_cams, _, ch = shard.shape
    rank = dist.get_rank() if world > 1 else 0
    if rank == dst and bufs is None:
        bufs = torch.empty((world, *shard.shape), dtype=shard.dtype, device=shard.device)
    if world == 1:
        bufs[0].copy_(shard)
        work = None
    else:
        work = dist.gather(shard, gather_list=list(bufs.unbind(0)) if rank == dst else None, dst=dst,
                           async_op=async_op)
    if async_op:
        return bufs, work
    if rank != dst:
        return None
    if not bufs.is_cuda:  # gloo (CPU tests) gathers host tensors; assembly is a device kernel
        bufs = bufs.cuda()
    return renderer.shard_assemble(bufs, world, n_cams, width, height, tile, ch)


# ---------------------------------------------------------------------------
# One process driving several devices (ngprt_multi_*: NCCL communicators from
# ncclCommInitAll, gather to devices[0] inside the library)
# ---------------------------------------------------------------------------
class MultiScene:
    """A scene replica on each of `devices` (ngprt_multi_create). render_tiles()
    splits every frame into interleaved tiles over the devices (one launch per
    device); render_cameras() gives each device whole cameras. Both return frames
    on devices[0]."""

    def __init__(self, desc, devices):
        import ctypes as C
        from . import _abi
        self._keep = desc
        desc_ptr = desc.desc_ptr if hasattr(desc, "desc_ptr") else C.pointer(desc)
        self.devices = list(devices)
        arr = (C.c_int * len(self.devices))(*self.devices)
        h = C.c_void_p()
        _abi.check(_abi.lib().ngprt_multi_create(desc_ptr, arr, len(self.devices), C.byref(h)),
                   "ngprt_multi_create")
        self._h = h

    @property
    def uses_nccl(self) -> bool:
        from . import _abi
        return bool(_abi.lib().ngprt_multi_uses_nccl(self._h))

    def _call(self, fn, cams, opts, extra, stats, stream):
        import ctypes as C
        from . import _abi, renderer
        cams = renderer.camera_array(cams)
        opts = opts or renderer.Opts()
        h, w = renderer._frame_hw(cams, opts)
        dev = torch.device("cuda", self.devices[0])
        out = torch.empty((len(cams), h, w, 3), dtype=torch.float32, device=dev)
        st = torch.empty((len(cams), h, w, 4), dtype=torch.int32, device=dev) if stats else None
        s = stream if stream is not None else torch.cuda.current_stream(dev)
        o = opts.to_c()
        _abi.check(fn(self._h, cams, len(cams), C.byref(o), *extra, out.data_ptr(),
                      st.data_ptr() if st is not None else None, s.cuda_stream), fn.__name__)
        return (out, st) if stats else out

    def render_tiles(self, cams, opts=None, tile: int = 32, stats: bool = False, stream=None):
        from . import _abi
        return self._call(_abi.lib().ngprt_multi_render_tiles, cams, opts, (tile,), stats, stream)

    def render_cameras(self, cams, opts=None, stats: bool = False, stream=None):
        from . import _abi
        return self._call(_abi.lib().ngprt_multi_render_cameras, cams, opts, (), stats, stream)

    def close(self):
        from . import _abi
        if getattr(self, "_h", None):
            _abi.lib().ngprt_multi_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()
