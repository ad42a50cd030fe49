"""GPU: interleaved-tile sharding in ONE launch per rank (ngprt_render_opts.shard_*),
the de-interleave kernel (ngprt_shard_assemble), the single-process multi-device
API (ngprt_multi_*: NCCL communicators from ncclCommInitAll; peer copies when
replicas share a device), and concurrent use of the C ABI from several host
threads. Every assembled frame must equal the unsharded single render bit for
bit (the output does not depend on the ray schedule)."""
from __future__ import annotations

import threading

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


@pytest.fixture(scope="module")
def small(ng):
    scene = ng.SynthScene(occupancy="bench", occ_base_res=128, L=2, L_C=128, fine_table_len=1 << 14)
    return scene, ng.Scene(scene)


def bits(t):
    return t.cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("world,tile", [(1, 32), (2, 32), (3, 16), (4, 8), (7, 32)])
def test_sharded_ranks_assemble_to_the_single_render(ng, torch, small, world, tile):
    """Each rank's tiles of two cameras in one call; the rank buffers stacked
    rank-major and de-interleaved equal the unsharded render (RGB and counters),
    for a frame and a window that are not multiples of the tile."""
    synth, dev = small
    cams = ng.cameras(5, 200, 136)
    two = [cams[1], cams[3]]
    for window in [None, (9, 5, 150, 101)]:
        base = ng.Opts(mlp="exact", window=window)
        want_rgb, want_st = ng.render(dev, two, base, stats=True)
        h, w = (window[3], window[2]) if window else (136, 200)
        P = ng.shard_pixels(w, h, world, tile)
        rgb_sh = torch.empty((world, 2, P, 3), dtype=torch.float32, device="cuda")
        st_sh = torch.empty((world, 2, P, 4), dtype=torch.int32, device="cuda")
        from paper_2407_10482_b200 import multigpu as mg
        for r in range(world):
            rgb_r, st_r = mg.render_tile_shard(dev, two, base, r, world, tile, stats=True)
            rgb_sh[r].copy_(rgb_r)
            st_sh[r].copy_(st_r)
        got_rgb = ng.shard_assemble(rgb_sh, world, 2, w, h, tile, 3)
        got_st = ng.shard_assemble(st_sh.view(torch.float32), world, 2, w, h, tile, 4)
        torch.cuda.synchronize()
        assert np.array_equal(bits(got_rgb), bits(want_rgb))
        assert np.array_equal(bits(got_st), bits(want_st))


def test_sharded_tensor_mode_and_padding_black(ng, torch, small):
    """Tensor-MLP mode sharded == unsharded (same kernels, same rays); padding
    slots past the frame edge come out black with zero counters."""
    synth, dev = small
    cam = ng.cameras(2, 70, 44)[1]
    want = ng.render(dev, [cam], ng.Opts())
    world, tile = 2, 32
    P = ng.shard_pixels(70, 44, world, tile)
    sh = torch.stack([ng.render(dev, [cam], ng.Opts(shard_world=world, shard_rank=r, shard_tile=tile))
                      for r in range(world)])
    got = ng.shard_assemble(sh, world, 1, 70, 44, tile, 3)
    torch.cuda.synchronize()
    assert np.array_equal(bits(got), bits(want))
    # rank 0 holds global tiles 0, 2, 4 (3 x 2 tiles); tile 4 = (x 32..63, y 32..43): rows >= 12 pad
    rgb0, st0 = ng.render(dev, [cam], ng.Opts(shard_world=world, shard_rank=0, shard_tile=tile),
                          stats=True)
    t4 = rgb0[0, 2 * tile * tile:3 * tile * tile].reshape(tile, tile, 3)
    assert float(t4[12:].abs().max()) == 0.0
    assert int(st0[0, 2 * tile * tile:3 * tile * tile].reshape(tile, tile, 4)[12:].abs().max()) == 0
    assert P == 3 * tile * tile


def test_shard_rejects_bad_parameters(ng, torch, small):
    _, dev = small
    cam = ng.cameras(1, 64, 64)[0]
    with pytest.raises(ng.NgprtError, match="multiple of 8"):
        ng.render(dev, [cam], ng.Opts(shard_world=2, shard_rank=0, shard_tile=12))
    with pytest.raises(ng.NgprtError, match="shard_rank"):
        ng.render(dev, [cam], ng.Opts(shard_world=2, shard_rank=2))
    with pytest.raises(ValueError, match="contiguous"):
        ng.render(dev, [cam], ng.Opts(), out=torch.empty((1, 10, 10, 3), device="cuda"))


def test_sharded_1080p_config3_two_ranks(ng, torch):
    """Config 3 at full size, 2 ranks of 32x32 tiles, one launch each: the
    assembled frame and counters equal the single render bit for bit."""
    synth = ng.SynthScene(**dict(ng.CONFIGS["c3_1080p"]))
    dev = ng.Scene(synth)
    cam = ng.cameras(64, 1920, 1080)[9]
    want_rgb, want_st = ng.render(dev, [cam], ng.Opts(), stats=True)
    from paper_2407_10482_b200 import multigpu as mg
    parts = [mg.render_tile_shard(dev, [cam], ng.Opts(), r, 2, 32, stats=True) for r in range(2)]
    rgb = ng.shard_assemble(torch.stack([p[0] for p in parts]), 2, 1, 1920, 1080, 32, 3)
    st = ng.shard_assemble(torch.stack([p[1] for p in parts]).view(torch.float32), 2, 1, 1920, 1080, 32, 4)
    torch.cuda.synchronize()
    assert np.array_equal(bits(rgb), bits(want_rgb))
    assert np.array_equal(bits(st), bits(want_st))


def test_multi_api_one_device_uses_nccl(ng, torch, small):
    """ngprt_multi_* over devices [0]: an NCCL communicator (ncclCommInitAll) is
    created; tile and camera rendering equal the plain render."""
    from paper_2407_10482_b200 import multigpu as mg
    synth, dev = small
    m = mg.MultiScene(synth, [0])
    assert m.uses_nccl
    cams = ng.cameras(3, 96, 72)
    want_rgb, want_st = ng.render(dev, cams, ng.Opts(mlp="exact"), stats=True)
    rgb, st = m.render_tiles(cams, ng.Opts(mlp="exact"), tile=16, stats=True)
    torch.cuda.synchronize()
    assert np.array_equal(bits(rgb), bits(want_rgb)) and np.array_equal(bits(st), bits(want_st))
    rgb = m.render_cameras(cams, ng.Opts(mlp="exact"))
    torch.cuda.synchronize()
    assert np.array_equal(bits(rgb), bits(want_rgb))
    m.close()


@pytest.mark.parametrize("n_rep", [2, 3])
def test_multi_api_replicas_on_one_device(ng, torch, small, n_rep):
    """n replicas on device 0 (peer-copy gather, NCCL needs distinct devices):
    n-way tile sharding and camera sharding equal the single render."""
    from paper_2407_10482_b200 import multigpu as mg
    synth, dev = small
    m = mg.MultiScene(synth, [0] * n_rep)
    assert not m.uses_nccl
    cams = ng.cameras(5, 120, 90)
    want_rgb, want_st = ng.render(dev, cams, ng.Opts(mlp="exact"), stats=True)
    for _ in range(2):  # buffer reuse across calls
        rgb, st = m.render_tiles(cams, ng.Opts(mlp="exact"), tile=32, stats=True)
        torch.cuda.synchronize()
        assert np.array_equal(bits(rgb), bits(want_rgb)) and np.array_equal(bits(st), bits(want_st))
        rgb, st = m.render_cameras(cams, ng.Opts(mlp="exact"), stats=True)
        torch.cuda.synchronize()
        assert np.array_equal(bits(rgb), bits(want_rgb)) and np.array_equal(bits(st), bits(want_st))
    m.close()


def test_concurrent_renders_from_host_threads(ng, torch, small):
    """SPEC.md:329-330 and the header's concurrency promise: four host threads
    render the same scene at once on their own streams, and a second scene in
    the same process, each result equal to the serial render."""
    synth, dev = small
    other_synth = ng.SynthScene(occupancy="toy", occ_base_res=64, L=3, L_C=64, fine_table_len=1 << 12)
    other = ng.Scene(other_synth)
    cams = ng.cameras(8, 80, 60)
    want = [ng.render(dev, [c], ng.Opts(mlp="exact")).cpu() for c in cams]
    want_o = [ng.render(other, [c], ng.Opts()).cpu() for c in cams]
    got, errs = {}, []

    def work(k):
        try:
            s = torch.cuda.Stream()
            with torch.cuda.stream(s):
                for rep in range(3):
                    for i, c in enumerate(cams):
                        if (i + k) % 2:
                            r = ng.render(dev, [c], ng.Opts(mlp="exact"), stream=s)
                            key = ("a", k, rep, i)
                        else:
                            r = ng.render(other, [c], ng.Opts(), stream=s)
                            key = ("b", k, rep, i)
                        s.synchronize()
                        got[key] = r.cpu()
        except Exception as e:  # pragma: no cover
            errs.append(e)

    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errs, errs
    for (which, k, rep, i), r in got.items():
        ref = want[i] if which == "a" else want_o[i]
        assert np.array_equal(r.numpy().view(np.uint32), ref.numpy().view(np.uint32)), (which, k, i)


def test_duplicate_coarse_keys_keep_the_first_row(ng, torch):
    """A descriptor that repeats coarse keys: the first row of each key wins, as
    the reference's SparseCoarseGrid::add_row (index.emplace) keeps it; the
    render equals the compiled reference on the same descriptor bit for bit."""
    import ctypes as C
    from checkers import CpuScene
    synth = ng.SynthScene(occupancy="bench", occ_base_res=64, L=2, L_C=64, fine_table_len=1 << 12)
    keys, rows = synth.coarse_keys(), synth.coarse_rows()
    rng = np.random.RandomState(1)
    pick = rng.choice(len(keys), 500, replace=False)
    k2 = np.ascontiguousarray(np.concatenate([keys, keys[pick]]))
    r2 = np.ascontiguousarray(np.concatenate([rows, rows[pick] * 3.0 + 1.0]).astype(np.float32))
    d = ng._abi.SceneDesc.from_buffer_copy(synth.desc)
    d.n_coarse = len(k2)
    d.coarse_keys = k2.ctypes.data_as(C.POINTER(C.c_uint64))
    d.coarse_rows = r2.ctypes.data_as(C.POINTER(C.c_float))
    cam = ng.cameras(3, 64, 48)[2]
    dup = ng.Scene(d)
    rgb, st = ng.render(dup, [cam], ng.Opts(mlp="exact"), stats=True)
    want_rgb, want_st = CpuScene(C.pointer(d), "ref").render(cam, ng.Opts(mlp="exact").to_c())
    base = ng.render(ng.Scene(synth), [cam], ng.Opts(mlp="exact"))
    torch.cuda.synchronize()
    assert np.array_equal(bits(rgb[0]), want_rgb.view(np.uint32))
    assert np.array_equal(st[0].cpu().numpy().view(np.uint32), want_st)
    assert np.array_equal(bits(rgb), bits(base))


def test_sharded_host_buffer_calls_match_device_calls(ng, torch, small):
    """ngprt_render_host and ngprt_render_host_async accept sharded options and
    return the same compact buffer as the device-buffer call."""
    _, dev = small
    cams = ng.cameras(3, 72, 40)
    o = ng.Opts(mlp="exact", shard_world=3, shard_rank=1, shard_tile=16)
    want = ng.render(dev, cams, o).cpu().numpy()
    got = ng.render_host(dev, cams, o)
    assert got.shape == want.shape
    assert np.array_equal(got.view(np.uint32), want.view(np.uint32))
    out = np.zeros_like(want)
    ng.render_host_async(dev, cams, out, o)
    ng.render_host_wait(dev)
    assert np.array_equal(out.view(np.uint32), want.view(np.uint32))
