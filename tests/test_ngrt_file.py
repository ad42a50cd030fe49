"""The reference's baked-scene file (.ngrt, baking.hpp:229-485) as input.

CPU: a scene saved by the reference's own save_baked is read back by
ngprt_baked_load bit for bit (every section), and corrupt/truncated files fail
with the reference's error texts. GPU: the loaded file renders bit-exactly like
the reference renders the same BakedScene."""
from __future__ import annotations

import numpy as np
import pytest

from checkers import CpuScene, ref

SCENE = dict(occupancy="toy", occ_base_res=512, L=2, L_C=64, fine_table_len=1 << 12,
             fusion_tag="separate_att_inv")


@pytest.fixture(scope="module")
def saved(tmp_path_factory, ng):
    R = ref()
    if R is None:
        pytest.skip("compiled reference (oracle/_ref) not available")
    synth = ng.SynthScene(**SCENE)
    rs = CpuScene(synth.desc_ptr, "ref")
    path = tmp_path_factory.mktemp("ngrt") / "scene.ngrt"
    assert R.ref_save_baked(rs.h, str(path).encode()) == 0
    return synth, rs, path


def _arr(ptr, n, dt):
    import ctypes as C
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dt))), shape=(n,))


def test_load_matches_saved_scene(ng, saved):
    synth, _, path = saved
    b = ng.BakedFile(path)
    d, s = b.desc, synth.desc
    assert (d.L, d.L_C, d.fusion_tag) == (s.L, s.L_C, s.fusion_tag)
    assert list(d.fine_res)[: d.L] == list(s.fine_res)[: s.L]
    assert list(d.fine_table_len)[: d.L] == list(s.fine_table_len)[: s.L]
    # coarse map: the file is sorted by key (baking.hpp:288-291); compare as sets of rows
    w = 8 + 2 * d.L
    ks, rs = synth.coarse_keys(), synth.coarse_rows()
    kf = _arr(d.coarse_keys, d.n_coarse, np.uint64)
    rf = _arr(d.coarse_rows, d.n_coarse * w, np.float32).reshape(-1, w)
    order = np.argsort(ks)
    assert np.array_equal(kf, ks[order])
    assert np.array_equal(rf.view(np.uint32), rs[order].view(np.uint32))
    for l in range(d.L):
        n = int(d.fine_table_len[l]) * 8
        assert np.array_equal(_arr(d.fine_tables[l], n, np.float32), synth.fine_table(l).ravel())
    ws, bs = synth.psi()
    for k, (wk, bk) in enumerate(zip(ws, bs)):
        assert np.array_equal(_arr(d.psi_w[k], wk.size, np.float32), wk.ravel())
        assert np.array_equal(_arr(d.psi_b[k], bk.size, np.float32), bk)
    assert np.array_equal(_arr(d.att_globals, 2 * d.L, np.float32),
                          _arr(s.att_globals, 2 * s.L, np.float32))
    # pyramid level 0 is the scene's occupancy; levels 1..4 / distance grid are the reference's
    assert np.array_equal(_arr(d.pyramid_words[0], 512 ** 3 // 64, np.uint64), synth.base_words())
    assert d.occ_base_res == 512 and d.dist_res == 256


def test_corrupt_files_fail_like_the_reference(ng, saved, tmp_path):
    _, _, path = saved
    data = bytearray(path.read_bytes())
    bad_magic = tmp_path / "magic.ngrt"
    bad_magic.write_bytes(b"XXXX" + bytes(data[4:]))
    with pytest.raises(ng.NgprtError, match="bad magic at offset 0"):
        ng.BakedFile(bad_magic)
    flipped = bytearray(data)
    flipped[len(flipped) // 2] ^= 0xFF
    p = tmp_path / "flip.ngrt"
    p.write_bytes(bytes(flipped))
    with pytest.raises(ng.NgprtError, match="checksum failure in section"):
        ng.BakedFile(p)
    p2 = tmp_path / "trunc.ngrt"
    p2.write_bytes(bytes(data[: len(data) - 100]))
    with pytest.raises(ng.NgprtError, match="truncated section"):
        ng.BakedFile(p2)
    with pytest.raises(ng.NgprtError, match="cannot open"):
        ng.BakedFile(tmp_path / "missing.ngrt")


def test_crafted_lengths_are_rejected(ng, saved, tmp_path):
    """Header / section lengths the reference never bounds (baking.hpp:396-405):
    a section length near 2^64 (the end-of-section test would wrap), a fine
    table length that would make the section-2 arithmetic wrap, and a section 2
    whose size does not match the table lengths all fail with a message."""
    import struct
    _, _, path = saved
    data = bytearray(path.read_bytes())
    # header: "NGRT", u32 version, u32 L_C, u32 L, u32 fine_res[2], u64 lens[6 + 2], u8 tag, pad
    first_section = 8 + ((4 + 4 + 8 + 64 + 1 + 7) // 8) * 8
    assert struct.unpack_from("<I", data, first_section)[0] == 1
    wrap = bytearray(data)
    struct.pack_into("<Q", wrap, first_section + 4, (1 << 64) - 8)
    p = tmp_path / "wrap.ngrt"
    p.write_bytes(bytes(wrap))
    with pytest.raises(ng.NgprtError, match="truncated section 1"):
        ng.BakedFile(p)
    huge = bytearray(data)
    struct.pack_into("<Q", huge, 8 + 16 + 6 * 8, 1 << 61)  # fine level 0 table length
    p = tmp_path / "huge.ngrt"
    p.write_bytes(bytes(huge))
    with pytest.raises(ng.NgprtError, match="fine table length out of range"):
        ng.BakedFile(p)
    small = bytearray(data)
    struct.pack_into("<Q", small, 8 + 16 + 6 * 8, 1 << 11)  # half the stored rows
    p = tmp_path / "small.ngrt"
    p.write_bytes(bytes(small))
    with pytest.raises(ng.NgprtError, match="fine table section size mismatch"):
        ng.BakedFile(p)


@pytest.mark.gpu
def test_loaded_file_renders_like_the_reference(ng, saved):
    import torch
    _, rs, path = saved
    dev = ng.Scene(ng.BakedFile(path))
    cam = ng.cameras(4, 48, 40)[1]
    opts = ng.Opts(mlp="exact")
    rgb, st = ng.render(dev, [cam], opts, stats=True)
    torch.cuda.synchronize()
    want_rgb, want_st = rs.render(cam, opts.to_c(), nthreads=8)
    assert np.array_equal(st[0].cpu().numpy().view(np.uint32), want_st)
    assert np.array_equal(rgb[0].cpu().numpy().view(np.uint32), want_rgb.view(np.uint32))


@pytest.mark.gpu
def test_full_scale_bench_scene_through_the_reference_file(ng, tmp_path):
    """The bench scene itself (config 3: 512^3 pyramid, 256^3 distance grid, L_C =
    512, 2^21-row tables, ~19 M coarse rows) written by the reference's save_baked,
    loaded by ngprt_scene_load and rendered at 1080p: counters and exact-mode RGB
    bit-exact against the reference rendering the same BakedScene."""
    import torch
    R = ref()
    assert R is not None, "compiled reference (oracle/_ref) required"
    synth = ng.SynthScene(**dict(ng.CONFIGS["c3_1080p"]))
    rs = CpuScene(synth.desc_ptr, "ref")
    path = tmp_path / "c3.ngrt"
    assert R.ref_save_baked(rs.h, str(path).encode()) == 0
    dev = ng.Scene(ng.BakedFile(path))
    assert dev.info().storage == 2  # the file's f32 values are fp16-exact: lossless fp16 rows
    cam = ng.cameras(64, 1920, 1080)[13]
    rgb, st = ng.render(dev, [cam], ng.Opts(mlp="exact"), stats=True)
    torch.cuda.synchronize()
    want_rgb, want_st = rs.render(cam, ng.Opts(mlp="exact").to_c())
    assert np.array_equal(st[0].cpu().numpy().view(np.uint32), want_st)
    assert np.array_equal(rgb[0].cpu().numpy().view(np.uint32), want_rgb.view(np.uint32))
    assert (want_st[..., 1] > 0).mean() > 0.5  # most rays reach occupied points
