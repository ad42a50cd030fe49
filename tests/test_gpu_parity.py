"""GPU parity: the CUDA path through the C ABI against the reference's own
outputs (golden fixtures from oracle/_ref) and the C restatement oracle.

Bar (north_star): bit-exact hash indices, occupancy pyramid, distance grid and
per-ray march counters; RGB bit-exact in the exact-MLP mode, and max-abs
<= 1e-3 with PSNR >= 60 dB in the tensor-core MLP mode."""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from cases import CASES, make_case, random_grid_words, scene_crc
from checkers import REF_SO, CpuScene, host_expf_range

pytestmark = pytest.mark.gpu

GOLD = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLD / "golden.json").read_text())
RGB_TOL = 1e-3     # north_star: per-pixel RGB max-abs error <= 1e-3
PSNR_MIN = 60.0    # north_star: PSNR >= 60 dB


@pytest.fixture(scope="module")
def torch():
    import torch
    assert torch.cuda.is_available(), "GPU tests need a CUDA device"
    return torch


def crc(ng, a):
    a = np.ascontiguousarray(a)
    return int(ng.lib().ngprt_crc32(a.ctypes.data, a.nbytes, 0))


def psnr(a, b):
    mse = float(np.mean((a.astype(np.float64) - b.astype(np.float64)) ** 2))
    return 99.0 if mse <= 0 else min(99.0, 10 * np.log10(1.0 / mse))  # image.hpp:90-101


def gpu_render(ng, torch, scene_dev, cam, opts):
    rgb, st = ng.render(scene_dev, [cam], opts, stats=True)
    torch.cuda.synchronize()
    return rgb[0].cpu().numpy(), st[0].cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_render_exact_matches_reference(ng, torch, case):
    scene, cam, opts = make_case(ng, case)
    assert scene_crc(ng, scene) == G["cases"][case["name"]]["scene_crc"]
    dev = ng.Scene(scene)
    opts.mlp = "exact"
    rgb, stats = gpu_render(ng, torch, dev, cam, opts)
    ref = np.load(GOLD / f"render_{case['name']}.npz")
    assert np.array_equal(stats, ref["stats"]), \
        f"counters differ at {np.argwhere((stats != ref['stats']).any(-1))[:5]}"
    diff = np.abs(rgb - ref["rgb"])
    assert np.array_equal(rgb.view(np.uint32), ref["rgb"].view(np.uint32)), \
        f"rgb not bit-exact: max abs {diff.max()} at {np.unravel_index(diff.argmax(), diff.shape)}"


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_render_tensor_within_tolerance(ng, torch, case):
    scene, cam, opts = make_case(ng, case)
    dev = ng.Scene(scene)
    opts.mlp = "tensor"
    rgb, stats = gpu_render(ng, torch, dev, cam, opts)
    ref = np.load(GOLD / f"render_{case['name']}.npz")
    assert np.array_equal(stats, ref["stats"])
    # the black/shade branch (final_t < 1) is decided before the MLP: exact
    assert np.array_equal(rgb.sum(-1) == 0, ref["rgb"].sum(-1) == 0)
    assert np.abs(rgb - ref["rgb"]).max() <= RGB_TOL
    assert psnr(rgb, ref["rgb"]) >= PSNR_MIN


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_device_pyramid_and_distance_grid(ng, torch, case):
    """The pyramid (K3) and distance grid (K4) the scene built on the device are
    bit-identical to the reference's build_pyramid / build_distance_grid."""
    scene, _, _ = make_case(ng, case)
    gold = G["cases"][case["name"]]
    dev = ng.Scene(scene)
    info = dev.info()
    torch.cuda.synchronize()
    r0 = int(scene.desc.occ_base_res)
    lv = [_dev_copy(info.dev_pyramid[k], (((r0 >> k) ** 3 + 63) // 64) * 8).view(np.uint64)
          for k in range(1, 5)]
    assert crc(ng, np.concatenate(lv)) == gold["pyramid_crc"]
    if "dist_crc" in gold:
        dr = int(scene.desc.dist_res)
        assert crc(ng, _dev_copy(info.dev_dist, dr ** 3)) == gold["dist_crc"]


def _dev_copy(ptr, nbytes):
    """Copy nbytes from a raw device pointer into a host uint8 array (cudaMemcpy D2H)."""
    out = np.empty(nbytes, np.uint8)
    rc = _cudart().cudaMemcpy(out.ctypes.data, ptr, nbytes, 2)
    assert rc == 0, f"cudaMemcpy failed {rc}"
    return out


_CUDART = None


def _cudart():
    global _CUDART
    if _CUDART is None:
        import glob
        import os
        import torch
        cands = glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia",
                                       "cuda_runtime", "lib", "libcudart.so*"))
        cands += ["libcudart.so.12", "libcudart.so"]
        for c in cands:
            try:
                _CUDART = C.CDLL(c)
                break
            except OSError:
                continue
        _CUDART.cudaMemcpy.argtypes = [C.c_void_p, C.c_void_p, C.c_size_t, C.c_int]
    return _CUDART


def test_distance_grid_random_grids(ng, torch):
    for res, dens, seed, wcrc, dcrc in G["dt_random"]:
        words = random_grid_words(ng, res, dens, seed)
        w = torch.from_numpy(words.view(np.int64)).cuda()
        out = ng.build_distance_grid(w, res)
        assert crc(ng, out.cpu().numpy()) == dcrc, (res, dens)


def test_distance_grid_single_voxel(ng, torch):
    words = np.zeros(256 ** 3 // 64, np.uint64)
    i = 128 + 256 * (128 + 256 * 128)
    words[i >> 6] |= np.uint64(1) << np.uint64(i & 63)
    out = ng.build_distance_grid(torch.from_numpy(words.view(np.int64)).cuda(), 256).cpu().numpy()
    assert out[133 + 256 * (128 + 256 * 128)] == 4
    assert crc(ng, out) == G["dt_single_voxel"]["crc"]


DT_U8_GRIDS = [(256, 0.0, 21), (256, 2e-7, 22), (256, 1e-4, 23), (256, 0.3, 24),
               (200, 1e-6, 25), (96, 0.002, 26), (33, 0.05, 27), (4, 0.3, 28), ("corner", 0, 0),
               ("diagonal", 0, 0)]
_DT_WANT = {}


def _dt_case(ng, R, res, dens, seed):
    key = (res, dens, seed)
    if res == "corner":  # one voxel at (0,0,0): D = 255 at the far corner (G = 254)
        words = np.zeros(256 ** 3 // 64, np.uint64)
        words[0] = np.uint64(1)
        res = 256
    elif res == "diagonal":  # the plane x = 2y at z < 128: slope-2 ramps, long deques
        bits = np.zeros((256, 256, 256), np.uint8)  # z, y, x
        y = np.arange(128)
        bits[:128, y, 2 * y] = 1
        words = np.zeros(256 ** 3 // 64, np.uint64)
        words.view(np.uint8)[:] = np.packbits(bits.ravel(), bitorder="little")
        res = 256
    else:
        words = random_grid_words(ng, res, dens, seed)
    if key not in _DT_WANT:
        want = np.zeros(res ** 3, np.uint8)
        R.ref_build_distance_grid(words.ctypes.data, res, want.ctypes.data)
        _DT_WANT[key] = want
    return words, res, _DT_WANT[key]


@pytest.mark.parametrize("depth", [None, "16", "1", "2"])
def test_distance_grid_u8_passes_match_reference(ng, torch, monkeypatch, depth):
    """K4's u8 passes (r <= 256: distances saturated at 255, the all-empty grid
    flagged by pass X) equal the compiled reference's build_distance_grid
    (occupancy.hpp:136-194) byte for byte on empty, near-empty (distances up to
    255), dense, diagonal-plane, non-multiple-of-32 and tiny grids. Default: the
    range-minimum kernel where r is a multiple of 32, the deque kernel
    elsewhere. NGPRT_DT_RING forces the deque kernel everywhere, with the
    default ring (16 entries; the diagonal plane overflows it) and with rings
    of 1 and 2 entries (every or most columns redone with the global deque)."""
    from checkers import ref
    R = ref()
    assert R is not None, "compiled reference (oracle/_ref) required"
    if depth:
        monkeypatch.setenv("NGPRT_DT_RING", depth)
    for res, dens, seed in DT_U8_GRIDS:
        words, r, want = _dt_case(ng, R, res, dens, seed)
        got = ng.build_distance_grid(torch.from_numpy(words.view(np.int64)).cuda(), r).cpu().numpy()
        assert np.array_equal(got, want), (res, dens, depth, int((got != want).sum()))
        if res == "corner":
            assert want[-1] == 254


@pytest.mark.parametrize("res,dens,seed", [(288, 1e-5, 41), (300, 0.01, 42), (512, 2e-6, 43)])
def test_distance_grid_above_256_matches_reference(ng, torch, res, dens, seed):
    """r > 256 takes the u16 passes (pass X per row, envelope sweeps with u16
    stack indices up to r = 1024): byte-identical to the reference."""
    from checkers import ref
    R = ref()
    assert R is not None, "compiled reference (oracle/_ref) required"
    words = random_grid_words(ng, res, dens, seed)
    want = np.zeros(res ** 3, np.uint8)
    R.ref_build_distance_grid(words.ctypes.data, res, want.ctypes.data)
    got = ng.build_distance_grid(torch.from_numpy(words.view(np.int64)).cuda(), res).cpu().numpy()
    assert np.array_equal(got, want), int((got != want).sum())


def test_pyramid_matches_oracle_on_random_grids(ng, torch):
    from checkers import oracle
    O = oracle()
    for res, dens, seed in [(64, 0.01, 11), (128, 0.001, 12), (256, 0.02, 13), (32, 1.0, 14)]:
        words = random_grid_words(ng, res, dens, seed)
        n = sum(((res >> k) ** 3 + 63) // 64 for k in range(1, 5))
        want = np.zeros(n, np.uint64)
        O.orc_build_pyramid(words.ctypes.data, res, want.ctypes.data)
        got = ng.build_pyramid(torch.from_numpy(words.view(np.int64)).cuda(), res)
        got = np.concatenate([g.cpu().numpy().view(np.uint64) for g in got])
        assert np.array_equal(got, want), res


def test_hash_index_on_device(ng, torch):
    rows = G["hash_index"]
    for res, maxlen in sorted({(r[0], r[1]) for r in rows}):
        sel = [r for r in rows if r[0] == res and r[1] == maxlen]
        corners = np.array([[r[2], r[3], r[4]] for r in sel], np.int32)
        want = np.array([r[5] for r in sel], np.uint64)
        ncorn = (res + 1) ** 3
        hashed = 0 if ncorn <= maxlen else 1
        tlen = ncorn if ncorn <= maxlen else maxlen
        c = torch.from_numpy(corners).cuda()
        out = torch.empty(len(sel), dtype=torch.int64, device="cuda")
        ng._abi.check(ng.lib().ngprt_test_hash_index(c.data_ptr(), len(sel), res, tlen, hashed,
                                                     out.data_ptr(), None), "hash")
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (res, maxlen)


def test_expf_kat_on_device(ng, torch):
    xs = np.uint32([r[0] for r in G["expf"]]).view(np.float32)
    want = np.uint32([r[1] for r in G["expf"]])
    x = torch.from_numpy(xs).cuda()
    y = torch.empty_like(x)
    ng._abi.check(ng.lib().ngprt_test_expf(x.data_ptr(), y.data_ptr(), len(xs), None), "expf")
    torch.cuda.synchronize()
    got = y.cpu().numpy().view(np.uint32)
    assert np.array_equal(got, want)


def test_expf_exhaustive_vs_host_glibc(ng, torch):
    """All 2^32 inputs: the device port of glibc expf == this host's glibc expf."""
    chunk = 1 << 28
    y = torch.empty(chunk, dtype=torch.int32, device="cuda")
    bad = 0
    for first in range(0, 1 << 32, chunk):
        ng._abi.check(ng.lib().ngprt_test_expf_range(first, chunk, y.data_ptr(), None), "expf")
        torch.cuda.synchronize()
        got = y.cpu().numpy().view(np.uint32)
        want = host_expf_range(first, chunk)
        neq = got != want
        if neq.any():  # NaN payloads: both must be NaN
            gf, wf = got[neq].view(np.float32), want[neq].view(np.float32)
            bad += int((~(np.isnan(gf) & np.isnan(wf))).sum())
    assert bad == 0


def ref_scene(desc_ptr):
    """The compiled reference (oracle/_ref) holding this scene; required on the GPU box."""
    assert REF_SO.exists(), "oracle/_ref/libngprt_ref.so missing (built by __graft_entry__.build())"
    return CpuScene(desc_ptr, "ref")


@pytest.mark.parametrize("config,cam_i", [("c3_1080p", 7), ("c3_1080p_f32", 11), ("c3_mip360", 0)])
def test_full_1080p_frame_matches_reference(ng, torch, config, cam_i):
    """Config 3 at full size (the calibrated bench scene and the round-1 mip360
    preset): every ray of a 1920x1080 frame, bit-exact vs the compiled reference
    (counters and RGB)."""
    cfg = dict(ng.CONFIGS[config])
    scene = ng.SynthScene(**cfg)
    cam = ng.cameras(64, 1920, 1080)[cam_i]
    opts = ng.Opts(mlp="exact")
    dev = ng.Scene(scene)
    assert dev.info().storage == (1 if config.endswith("_f32") else 2)  # f32 / fp16 rows
    rgb, stats = gpu_render(ng, torch, dev, cam, opts)
    o = ref_scene(scene.desc_ptr)
    want_rgb, want_stats = o.render(cam, opts.to_c())
    assert np.array_equal(stats, want_stats)
    assert np.array_equal(rgb.view(np.uint32), want_rgb.view(np.uint32))
    # the bench mode (tensor MLP, FMA colour accumulation in K1): counters still
    # bit-exact on every ray, RGB within the north_star tolerance
    t_rgb, t_stats = gpu_render(ng, torch, dev, cam, ng.Opts(mlp="tensor"))
    assert np.array_equal(t_stats, want_stats)
    assert np.array_equal(t_rgb.sum(-1) == 0, want_rgb.sum(-1) == 0)
    assert np.abs(t_rgb - want_rgb).max() <= RGB_TOL
    assert psnr(t_rgb, want_rgb) >= PSNR_MIN


@pytest.mark.parametrize("config,width,height,cam_i", [
    ("c1_256", 256, 256, 0), ("c2_blob800", 800, 800, 5), ("c5_2160p", 3840, 2160, 0)])
def test_full_frame_matches_reference(ng, torch, config, width, height, cam_i):
    """Configs 1, 2 and 5 at full size (C1 256^2 L=4; C2 800^2 L=2 2^22; C5 3840x2160
    L=2 2^22, 8.3 M rays): counters and exact-mode RGB bit-exact vs the compiled
    reference on every ray, the tensor-core mode within the north_star tolerance,
    and a ragged window at the frame's far corner equal to the crop of the frame."""
    scene = ng.SynthScene(**dict(ng.CONFIGS[config]))
    cam = ng.cameras(max(cam_i + 1, 1), width, height)[cam_i]
    dev = ng.Scene(scene)
    rgb, stats = gpu_render(ng, torch, dev, cam, ng.Opts(mlp="exact"))
    o = ref_scene(scene.desc_ptr)
    want_rgb, want_stats = o.render(cam, ng.Opts(mlp="exact").to_c())
    assert np.array_equal(stats, want_stats)
    assert np.array_equal(rgb.view(np.uint32), want_rgb.view(np.uint32))
    assert (want_stats[..., 0] > 0).any() and (want_rgb.sum(-1) > 0).any()  # not a blank frame
    t_rgb, t_stats = gpu_render(ng, torch, dev, cam, ng.Opts(mlp="tensor"))
    assert np.array_equal(t_stats, want_stats)
    assert np.abs(t_rgb - want_rgb).max() <= RGB_TOL
    assert psnr(t_rgb, want_rgb) >= PSNR_MIN
    win = ng.render(dev, [cam], ng.Opts(mlp="exact", window=(width - 37, height - 19, 37, 19)))
    assert np.array_equal(win.cpu().numpy()[0].view(np.uint32), rgb[height - 19:, width - 37:].view(np.uint32))


def test_c4_64_camera_batch_matches_single_renders_and_reference(ng, torch):
    """Config 4 at full size: one launch of 64 1080p cameras. Every camera's
    counters and RGB equal its own single-camera render, and the last camera
    (largest camera offset in the batch index math) is bit-exact vs the compiled
    reference."""
    scene = ng.SynthScene(**dict(ng.CONFIGS["c4_1080p_x64"]))
    cams = ng.cameras(64, 1920, 1080)
    dev = ng.Scene(scene)
    opts = ng.Opts(mlp="exact")
    rgb, st = ng.render(dev, cams, opts, stats=True)
    torch.cuda.synchronize()
    for i in [0, 17, 42, 63]:
        one_rgb, one_st = gpu_render(ng, torch, dev, cams[i], opts)
        assert np.array_equal(st[i].cpu().numpy().view(np.uint32), one_st), i
        assert np.array_equal(rgb[i].cpu().numpy().view(np.uint32), one_rgb.view(np.uint32)), i
    want_rgb, want_stats = ref_scene(scene.desc_ptr).render(cams[63], opts.to_c())
    assert np.array_equal(st[63].cpu().numpy().view(np.uint32), want_stats)
    assert np.array_equal(rgb[63].cpu().numpy().view(np.uint32), want_rgb.view(np.uint32))


def test_multi_camera_batch_and_window_consistency(ng, torch):
    """A 70-camera batch (two launches of <= 64) equals per-camera renders, and a
    window render equals the crop of the full frame."""
    scene = ng.SynthScene(occupancy="bench", occ_base_res=128, L=2, L_C=128,
                          fine_table_len=1 << 14)
    dev = ng.Scene(scene)
    cams = ng.cameras(70, 40, 32)
    batch = ng.render(dev, cams, ng.Opts(mlp="exact")).cpu().numpy()
    for i in [0, 33, 63, 64, 69]:
        one = ng.render(dev, [cams[i]], ng.Opts(mlp="exact")).cpu().numpy()[0]
        assert np.array_equal(one.view(np.uint32), batch[i].view(np.uint32))
    full = batch[5]
    win = ng.render(dev, [cams[5]], ng.Opts(mlp="exact", window=(7, 3, 20, 17))).cpu().numpy()[0]
    assert np.array_equal(win.view(np.uint32), full[3:20, 7:27].view(np.uint32))
    again = ng.render(dev, cams, ng.Opts(mlp="exact")).cpu().numpy()
    assert np.array_equal(again.view(np.uint32), batch.view(np.uint32))  # determinism


def test_render_host_matches_device_render(ng, torch):
    scene = ng.SynthScene(occupancy="toy", occ_base_res=64, L=2, L_C=64, fine_table_len=1 << 12)
    dev = ng.Scene(scene)
    cams = ng.cameras(3, 32, 24)
    a = ng.render(dev, cams, ng.Opts(mlp="exact")).cpu().numpy()
    b = ng.render_host(dev, cams, ng.Opts(mlp="exact"))
    assert np.array_equal(a.view(np.uint32), b.view(np.uint32))


def test_render_host_async_pipeline_matches_sync(ng, torch):
    """ngprt_render_host_async: five frames through two slots (the third and
    later enqueues wait for a slot), pinned and pageable outputs, stats too;
    every frame equals the synchronous ngprt_render_host result."""
    scene = ng.SynthScene(occupancy="toy", occ_base_res=64, L=2, L_C=64, fine_table_len=1 << 12)
    dev = ng.Scene(scene)
    cams = ng.cameras(5, 40, 24)
    opts = ng.Opts(mlp="tensor")
    want = [ng.render_host(dev, [c], opts) for c in cams]
    outs = [torch.empty((1, 24, 40, 3), dtype=torch.float32).pin_memory().numpy() if i % 2 == 0
            else np.empty((1, 24, 40, 3), np.float32) for i in range(5)]
    stats = [np.empty((1, 24, 40, 4), np.uint32) for _ in range(5)]
    for c, o, st in zip(cams, outs, stats):
        ng.render_host_async(dev, [c], o, opts, stats=st)
    ng.render_host_wait(dev)
    for i in range(5):
        assert np.array_equal(outs[i].view(np.uint32), want[i].view(np.uint32)), i
        want_st = np.empty((1, 24, 40, 4), np.uint32)
        ng.render_host(dev, [cams[i]], opts, stats=want_st)
        assert np.array_equal(stats[i], want_st), i


def test_errors_are_reported(ng, torch):
    scene = ng.SynthScene(occupancy="slab", occ_base_res=64, L=2, L_C=32, fine_table_len=1 << 10)
    dev = ng.Scene(scene)
    cam = ng.cameras(1, 16, 16)[0]
    with pytest.raises(ng.NgprtError, match="keep_level"):
        ng.render(dev, [cam], ng.Opts(keep_level=3))
    with pytest.raises(ng.NgprtError, match="out of bounds"):
        ng.render(dev, [cam], ng.Opts(window=(10, 10, 8, 8)))
    scene.desc.fusion_tag = 5  # MLP fusion without its {8L,64,8} weights
    with pytest.raises(ng.NgprtError, match="fusion MLP"):
        ng.Scene(scene)


@pytest.mark.parametrize("mlp", ["exact", "tensor"])
def test_axis_aligned_rays_match_reference(ng, torch, mlp):
    """Axis-aligned cameras with odd image sizes: the centre row / column rays
    have direction components that are exactly zero, which voxel_exit_step skips
    (occupancy.hpp:244) and the GPU's approximate-argmin path must hand to its
    exact fallback. Counters bit-exact in both modes, RGB bit-exact in exact mode."""
    scene = ng.SynthScene(occupancy="toy", occ_base_res=128, L=2, L_C=64, fine_table_len=1 << 14)
    dev = ng.Scene(scene)
    o = ref_scene(scene.desc_ptr)
    for (o3, rot) in [((0.13, 0.21, -2.6), np.eye(3)),                      # looks down +z
                      ((-2.7, 0.05, 0.11), np.array([[0, 0, 1], [0, 1, 0], [-1, 0, 0]]))]:
        cam = ng._abi.Camera()
        m = np.eye(4)
        m[:3, :3] = rot
        m[:3, 3] = o3
        for i, v in enumerate(m.reshape(-1)):
            cam.c2w[i] = float(v)
        cam.width, cam.height = 33, 25
        cam.fx = cam.fy = 1.1 * 33
        cam.cx, cam.cy = 16.5, 12.5
        opts = ng.Opts(mlp=mlp)
        rgb, st = gpu_render(ng, torch, dev, cam, opts)
        want_rgb, want_st = o.render(cam, opts.to_c())
        assert np.array_equal(st, want_st)
        if mlp == "exact":
            assert np.array_equal(rgb.view(np.uint32), want_rgb.view(np.uint32))
        else:
            assert np.abs(rgb - want_rgb).max() <= RGB_TOL
        assert (want_st[..., 0] > 0).any()  # the rays do march


EDGE_SCENES = [
    # empty scene (SPEC.md:315 render_ray KAT: black; occupancy_probe KAT :382: one
    # access per marching point, the level-4 bit)
    dict(name="empty", scene=dict(occupancy="boxes", n_boxes=0, occ_base_res=64, L=2, L_C=64,
                                  fine_table_len=1 << 12), cam=dict(w=37, h=23, n=4, i=0)),
    # dense: 2240 boxes at 64^3 (most of the ROI occupied), ragged 37x23 frame
    dict(name="dense", scene=dict(occupancy="boxes", n_boxes=2240, occ_base_res=64, L=2, L_C=64,
                                  fine_table_len=1 << 12), cam=dict(w=37, h=23, n=4, i=1)),
    # a single-pixel frame and a 1-row frame
    dict(name="one_pixel", scene=dict(occupancy="bench", occ_base_res=64, L=3, L_C=64,
                                      fine_table_len=1 << 12), cam=dict(w=1, h=1, n=4, i=2)),
    dict(name="one_row", scene=dict(occupancy="toy", occ_base_res=64, L=1, L_C=64,
                                    fine_table_len=1 << 12), cam=dict(w=97, h=1, n=4, i=3)),
]


@pytest.mark.parametrize("case", EDGE_SCENES, ids=[c["name"] for c in EDGE_SCENES])
def test_edge_scenes_match_compiled_reference(ng, torch, case):
    """Empty / dense scenes and ragged frames (sizes not multiples of the 4x8 ray
    tile): counters and exact-mode RGB bit-identical to the compiled reference,
    tensor mode within the north_star tolerance."""
    scene = ng.SynthScene(**case["scene"])
    cm = case["cam"]
    cam = ng.cameras(cm["n"], cm["w"], cm["h"])[cm["i"]]
    want_rgb, want_stats = CpuScene(scene.desc_ptr, "ref").render(cam, ng.Opts().to_c())
    dev = ng.Scene(scene)
    rgb, stats = gpu_render(ng, torch, dev, cam, ng.Opts(mlp="exact"))
    assert np.array_equal(stats, want_stats)
    assert np.array_equal(rgb.view(np.uint32), want_rgb.view(np.uint32))
    rgb_t, stats_t = gpu_render(ng, torch, dev, cam, ng.Opts(mlp="tensor"))
    assert np.array_equal(stats_t, want_stats)
    assert float(np.abs(rgb_t - want_rgb).max(initial=0.0)) <= RGB_TOL
    if case["name"] == "empty":
        assert not rgb.any() and not stats[..., 1].any()          # black, no occupied point
        assert np.array_equal(stats[..., 2], stats[..., 0])       # one bit read per point


@pytest.mark.parametrize("mlp", ["exact", "tensor"])
def test_render_without_counters_is_identical(ng, torch, mlp):
    """Renders that request no per-ray counters run kernel variants with the
    counter updates compiled out; their RGB must equal the counted render's."""
    for case in CASES[:3] + [c for c in CASES if c["name"] == "mip360_window"]:
        scene, cam, opts = make_case(ng, case)
        dev = ng.Scene(scene)
        opts.mlp = mlp
        rgb_s, _ = gpu_render(ng, torch, dev, cam, opts)
        rgb = ng.render(dev, [cam], opts)
        torch.cuda.synchronize()
        rgb = rgb[0].cpu().numpy()
        assert np.array_equal(rgb.view(np.uint32), rgb_s.view(np.uint32)), case["name"]


def test_forced_fp16_storage_is_within_tolerance(ng, torch):
    """The opt-in lossy mode: an f32 scene (values not fp16-representable) stored
    as fp16 anyway (storage = NGPRT_STORAGE_F16) renders within the north_star
    RGB tolerance of the compiled reference (max-abs <= 1e-3, PSNR >= 60 dB) on a
    full 1080p frame of config 3; the counters may differ where early stop moves."""
    scene = ng.SynthScene(**dict(ng.CONFIGS["c3_1080p_f32"]))
    dev = ng.Scene(scene, storage=ng._abi.STORAGE_F16)
    assert dev.info().storage == 2
    cam = ng.cameras(64, 1920, 1080)[6]
    rgb = ng.render(dev, [cam], ng.Opts())
    torch.cuda.synchronize()
    want_rgb, want_st = ref_scene(scene.desc_ptr).render(cam, ng.Opts(mlp="exact").to_c())
    got = rgb[0].cpu().numpy()
    assert np.abs(got - want_rgb).max() <= RGB_TOL
    assert psnr(got, want_rgb) >= PSNR_MIN


@pytest.mark.parametrize("L", [2, 3, 4])
@pytest.mark.parametrize("fusion", ["sum", "shared_att_inv", "separate_att_inv", "shared_att_v",
                                    "separate_att_v"])
@pytest.mark.parametrize("fp16_exact", [1, 0])
def test_fusion_storage_matrix_matches_reference(ng, torch, L, fusion, fp16_exact):
    """Every fusion mode x L = 2..4 x fp16 / f32 storage through the fast decode
    (K1's fp16 and f32 variants): counters and exact-mode RGB bit-exact against
    the compiled reference, tensor mode within the north_star tolerance."""
    scene = ng.SynthScene(occupancy="toy", occ_base_res=64, L=L, L_C=48, fine_table_len=1 << 12,
                          fusion_tag=fusion, fp16_exact=fp16_exact, psi_bias_scale=0.1)
    dev = ng.Scene(scene)
    assert dev.info().storage == (2 if fp16_exact else 1)
    cam = ng.cameras(5, 40, 32)[L]
    rgb, st = gpu_render(ng, torch, dev, cam, ng.Opts(mlp="exact"))
    want_rgb, want_st = ref_scene(scene.desc_ptr).render(cam, ng.Opts(mlp="exact").to_c())
    assert np.array_equal(st, want_st)
    assert np.array_equal(rgb.view(np.uint32), want_rgb.view(np.uint32))
    t_rgb, t_st = gpu_render(ng, torch, dev, cam, ng.Opts(mlp="tensor"))
    assert np.array_equal(t_st, want_st)
    assert np.abs(t_rgb - want_rgb).max() <= RGB_TOL
