"""CPU (gloo, world_size 2): the multi-GPU host logic — camera sharding, tile
sharding and the gather to rank 0 — reproduces the single-process result
byte for byte. The pixel values are a deterministic function
of (camera, x, y) standing in for the renderer, which needs a GPU."""
from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2407_10482_b200 import multigpu as mg

W, H, TILE, N_CAMS = 37, 23, 8, 6


def fake_render(cam: int, window=None):
    x0, y0, w, h = window or (0, 0, W, H)
    ys = torch.arange(y0, y0 + h, dtype=torch.float32).view(h, 1, 1)
    xs = torch.arange(x0, x0 + w, dtype=torch.float32).view(1, w, 1)
    ch = torch.arange(3, dtype=torch.float32).view(1, 1, 3)
    return torch.sin(cam * 0.37 + xs * 0.11 + ys * 0.07 + ch)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # camera-batch sharding: each step every rank renders one camera; gather to 0
        frames = []
        for step in range(3):
            cam = mg.camera_of(rank, world, step, N_CAMS)
            got = mg.gather_frames(fake_render(cam), world)
            if rank == 0:
                # numpy (pickled by value): torch tensors would travel as shared-memory
                # handles that vanish when this process exits before the parent reads them
                frames.append((step, [g.numpy().copy() for g in got]))
        # interleaved tile sharding of one frame
        wins = mg.tile_windows(W, H, TILE, rank, world)
        tiles = [fake_render(4, w) for w in wins]
        img = mg.gather_tiles(tiles, W, H, TILE, world)
        if rank == 0:
            q.put(("ok", frames, img.numpy().copy()))
    except Exception as e:  # pragma: no cover - surfaced by the assert below
        q.put(("err", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [2])
def test_sharded_render_gathers_identically(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    status, frames, img = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert status == "ok", frames
    for step, got in frames:
        for r in range(world):
            want = fake_render(mg.camera_of(r, world, step, N_CAMS))
            assert torch.equal(torch.from_numpy(got[r]), want)
    assert torch.equal(torch.from_numpy(img), fake_render(4))


def test_sharding_covers_every_camera_and_tile_once():
    for world in [1, 2, 3, 4, 8]:
        cams = sorted(c for r in range(world) for c in mg.cameras_for_rank(r, world, 64))
        assert cams == list(range(64))
        seen = torch.zeros(H, W, dtype=torch.int32)
        for r in range(world):
            for (x0, y0, w, h) in mg.tile_windows(W, H, TILE, r, world):
                seen[y0:y0 + h, x0:x0 + w] += 1
        assert bool((seen == 1).all())
        # weak scaling: over N steps each rank renders N distinct cameras
        for r in range(world):
            assert len({mg.camera_of(r, world, s, 64) for s in range(64 // world)}) == 64 // world


@pytest.mark.gpu
def test_bench_two_rank_flow_on_one_gpu():
    """bench.py's multi-rank path (camera sharding, gather to rank 0, max-over-ranks
    timing, one JSON line from rank 0) end to end with 2 ranks on one GPU over gloo.
    Functional only: the driver's NCCL runs use one GPU per rank."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, NGPRT_BENCH_BACKEND="gloo", NGPRT_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    # `bench.py --gpus 2` launches its own 2 ranks (the driver's direct invocation)
    r = subprocess.run([sys.executable, str(root / "bench.py"),
                        "--gpus", "2", "--config", "c1_256", "--steps", "3", "--warmup", "3"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["steps"] == 3 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["value"] > 0


@pytest.mark.gpu
def test_bench_refuses_more_gpus_than_visible():
    """`bench.py --gpus N` with fewer than N visible GPUs exits non-zero with a
    message instead of silently timing one GPU."""
    import subprocess
    import sys
    from pathlib import Path
    import torch
    root = Path(__file__).resolve().parents[1]
    n = torch.cuda.device_count() + 1
    env = dict(os.environ)
    for k in ("NGPRT_BENCH_SHARE_GPU", "WORLD_SIZE", "RANK", "LOCAL_RANK"):
        env.pop(k, None)
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", str(n), "--steps", "3",
                        "--warmup", "3"], cwd=root, env=env, capture_output=True, text=True,
                       timeout=300)
    assert r.returncode != 0
    assert f"needs {n} visible GPUs" in r.stderr


def _gpu_tile_worker(rank, world, port, q):
    """Interleaved 32x32 tiles of one frame rendered by the real kernels on this
    rank (all ranks share the one GPU of the box), gathered to rank 0 (gloo)."""
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import numpy as np
        import paper_2407_10482_b200 as ng
        from cases import CASE_BY_NAME, make_case
        scene, cam, _ = make_case(ng, CASE_BY_NAME["bench_l2"])
        Wf, Hf = 72, 56   # not a multiple of the 32-pixel tile
        cam = ng.cameras(4, Wf, Hf)[1]
        dev = ng.Scene(scene)
        # (a) one ngprt_render call per tile window (the host-side tile path)
        tiles = []
        for (x0, y0, w, h) in mg.tile_windows(Wf, Hf, 32, rank, world):
            rgb = ng.render(dev, [cam], ng.Opts(mlp="exact", window=(x0, y0, w, h)))
            tiles.append(rgb[0].cpu())
        img = mg.gather_tiles(tiles, Wf, Hf, 32, world)
        # (b) this rank's tiles in ONE launch (compact shard), gathered, de-interleaved
        shard = mg.render_tile_shard(dev, [cam], ng.Opts(mlp="exact"), rank, world, 32)
        img2 = mg.gather_tile_shards(shard.cpu(), world, Wf, Hf, 32)  # gloo: host tensors
        if rank == 0:
            full = ng.render(dev, [cam], ng.Opts(mlp="exact"))[0].cpu()
            same = np.array_equal(img.numpy().view(np.uint32), full.numpy().view(np.uint32))
            same2 = np.array_equal(img2[0].cpu().numpy().view(np.uint32),
                                   full.numpy().view(np.uint32))
            q.put(("ok", bool(same and same2), None))
    except Exception as e:  # pragma: no cover
        q.put(("err", repr(e), None))
        raise
    finally:
        dist.destroy_process_group()


@pytest.mark.gpu
def test_tile_sharded_frame_is_byte_identical_on_gpu():
    """SPEC.md:329-330 / SURVEY §8(e): a frame rendered as interleaved tiles by 2
    ranks and gathered equals the single-render frame bit for bit."""
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gpu_tile_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    status, same, _ = q.get(timeout=300)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert status == "ok", same
    assert same


@pytest.mark.gpu
def test_bench_tile_sharding_mode_two_ranks_on_one_gpu():
    """`bench.py --shard tiles --gpus 2`: one frame per step split into interleaved
    tiles over 2 ranks (one launch each), gathered and de-interleaved on rank 0.
    Functional only (gloo, both ranks on one GPU)."""
    import json
    import subprocess
    import sys
    from pathlib import Path
    root = Path(__file__).resolve().parents[1]
    env = dict(os.environ, NGPRT_BENCH_BACKEND="gloo", NGPRT_BENCH_SHARE_GPU="1")
    env.pop("WORLD_SIZE", None)
    r = subprocess.run([sys.executable, str(root / "bench.py"), "--gpus", "2", "--shard", "tiles",
                        "--config", "c1_256", "--steps", "3", "--warmup", "3"],
                       cwd=root, env=env, capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1, r.stdout[-2000:]
    d = lines[0]
    assert d["n_gpus"] == 2 and d["scaling"] == "strong" and d["value"] > 0
    assert d["gpu_launches"] == 3 * 3 + 3  # rank 0: K0/K1/K2 + assemble per step


def _compact_index_model(W, H, world, tile):
    """Python model of the compact shard layout (include/ngprt_cuda.h,
    ngprt_render_opts.shard_*): rank -> list of (slot, x, y) for real pixels."""
    tx = (W + tile - 1) // tile
    n = tx * ((H + tile - 1) // tile)
    local = (n + world - 1) // world
    out = {r: [] for r in range(world)}
    for r in range(world):
        for j in range(local):
            T = r + j * world
            if T >= n:
                continue
            for ly in range(tile):
                for lx in range(tile):
                    x, y = (T % tx) * tile + lx, (T // tx) * tile + ly
                    if x < W and y < H:
                        out[r].append((j * tile * tile + ly * tile + lx, x, y))
    return out, local * tile * tile


@pytest.mark.parametrize("W,H,world,tile", [(37, 23, 2, 8), (70, 44, 3, 16), (64, 64, 4, 32),
                                            (250, 130, 8, 32), (40, 8, 7, 8)])
def test_compact_shard_layout_covers_every_pixel_once(ng, W, H, world, tile):
    """The compact layout: every pixel of the window lands in exactly one slot of
    one rank, the per-rank size equals ngprt_shard_pixels (C ABI, no GPU needed),
    and the rank's tiles are tile_windows' tiles in the same order."""
    model, per_rank = _compact_index_model(W, H, world, tile)
    assert per_rank == int(ng.lib().ngprt_shard_pixels(W, H, world, tile))
    seen = torch.zeros(H, W, dtype=torch.int32)
    for r in range(world):
        slots = [s for s, _, _ in model[r]]
        assert len(set(slots)) == len(slots) and max(slots, default=0) < per_rank
        for _, x, y in model[r]:
            seen[y, x] += 1
        wins = mg.tile_windows(W, H, tile, r, world)
        firsts = [(x, y) for s, x, y in model[r] if s % (tile * tile) == 0]
        assert firsts == [(x0, y0) for (x0, y0, _, _) in wins]
    assert bool((seen == 1).all())
