"""CPU: pin the C restatement (oracle/ngprt_oracle.c) and the synthetic-scene
generator against fixtures produced by the reference itself
(tests/golden/gen_golden.py over oracle/_ref). Bit-exact throughout."""
from __future__ import annotations

import ctypes as C
import json
from pathlib import Path

import numpy as np
import pytest

from cases import CASES, make_case, random_grid_words, scene_crc
from checkers import CpuScene, fptr, oracle

GOLD = Path(__file__).resolve().parent / "golden"
G = json.loads((GOLD / "golden.json").read_text())


def f32(bits):
    return np.uint32(bits).view(np.float32)


def crc(ng, a):
    a = np.ascontiguousarray(a)
    return int(ng.lib().ngprt_crc32(a.ctypes.data, a.nbytes, 0))


def test_hash_index_kat():
    O = oracle()
    for res, maxlen, x, y, z, want in G["hash_index"]:
        corners = (res + 1) ** 3
        hashed = 0 if corners <= maxlen else 1
        tlen = corners if corners <= maxlen else maxlen
        assert O.orc_hash_index(res, tlen, hashed, x, y, z) == want, (res, maxlen, x, y, z)


def test_spec_hash_examples():
    # SPEC.md:137-139 and SURVEY.md §4: (1,2,3) at 2^19/2^21/2^22 and (1024,1024,1024)
    O = oracle()
    assert O.orc_hash_index(16, 17 ** 3, 0, 0, 0, 0) == 0
    assert O.orc_hash_index(16, 17 ** 3, 0, 1, 0, 0) == 1
    for tl, want in [(1 << 19, 128476), (1 << 21, 652764), (1 << 22, 2749916)]:
        assert O.orc_hash_index(1024, tl, 1, 1, 2, 3) == want
    for tl, want in [(1 << 19, 37888), (1 << 21, 1610752), (1 << 22, 3707904)]:
        assert O.orc_hash_index(1024, tl, 1, 1024, 1024, 1024) == want


@pytest.mark.parametrize("kind", ["density", "sigmoid"])
def test_activation_kat(kind):
    O = oracle()
    fn = O.orc_activate_density if kind == "density" else O.orc_activate_sigmoid
    for xb, yb in G[kind]:
        y = np.float32(fn(float(f32(xb))))
        assert y.view(np.uint32) == yb, (kind, f32(xb))


def test_alpha_and_expf_kat():
    O = oracle()
    for sb, db, ab in G["alpha"]:
        assert np.float32(O.orc_alpha(float(f32(sb)), float(f32(db)))).view(np.uint32) == ab
    for xb, yb in G["expf"]:
        y = np.float32(O.orc_expf(float(f32(xb))))
        assert y.view(np.uint32) == yb or (np.isnan(y) and np.isnan(f32(yb)))
    # sigma = 3, delta = 0.1 -> 0.2591818
    assert abs(O.orc_alpha(3.0, 0.1) - 0.2591818) < 1e-7


def test_sh_encode_kat():
    O = oracle()
    for d, want in G["sh_encode"]:
        d = np.uint32(d).view(np.float32)
        o = np.zeros(16, np.float32)
        O.orc_sh_encode(fptr(np.ascontiguousarray(d)), fptr(o))
        assert list(o.view(np.uint32)) == want


def test_mlp_kat():
    O = oracle()
    w = np.uint32(G["mlp"]["w"]).view(np.float32)
    b = np.uint32(G["mlp"]["b"]).view(np.float32)
    offs_w = [0, 23 * 64, 23 * 64 + 64 * 64]
    offs_b = [0, 64, 128]
    W = (C.POINTER(C.c_float) * 3)(*[fptr(w[o:]) if False else w[o:].ctypes.data_as(C.POINTER(C.c_float)) for o in offs_w])
    B = (C.POINTER(C.c_float) * 3)(*[b[o:].ctypes.data_as(C.POINTER(C.c_float)) for o in offs_b])
    widths = (C.c_int * 4)(23, 64, 64, 3)
    O.orc_mlp_forward.argtypes = [C.c_int, C.POINTER(C.c_int), C.POINTER(C.POINTER(C.c_float)),
                                  C.POINTER(C.POINTER(C.c_float)), C.POINTER(C.c_float),
                                  C.POINTER(C.c_float)]
    for c in G["mlp"]["cases"]:
        x = np.uint32(c["in"]).view(np.float32)
        o = np.zeros(3, np.float32)
        O.orc_mlp_forward(3, widths, W, B, fptr(np.ascontiguousarray(x)), fptr(o))
        assert list(o.view(np.uint32)) == c["out"]


def test_dt_random_grids(ng):
    O = oracle()
    for res, dens, seed, wcrc, dcrc in G["dt_random"]:
        words = random_grid_words(ng, res, dens, seed)
        assert crc(ng, words) == wcrc
        out = np.zeros(res ** 3, np.uint8)
        O.orc_build_distance_grid(words.ctypes.data, res, out.ctypes.data)
        assert crc(ng, out) == dcrc, (res, dens)


def test_dt_single_voxel(ng):
    # single occupied voxel (128,128,128), query (133,128,128) -> 4
    O = oracle()
    words = np.zeros(256 ** 3 // 64, np.uint64)
    i = 128 + 256 * (128 + 256 * 128)
    words[i >> 6] |= np.uint64(1) << np.uint64(i & 63)
    out = np.zeros(256 ** 3, np.uint8)
    O.orc_build_distance_grid(words.ctypes.data, 256, out.ctypes.data)
    assert out[133 + 256 * (128 + 256 * 128)] == 4 == G["dt_single_voxel"]["value"]
    assert out[i] == 0 and out[i + 1] == 0  # occupied -> 0; face-adjacent -> 0
    assert crc(ng, out) == G["dt_single_voxel"]["crc"]


def test_synth_pins(ng):
    """The generator restates make_scene/scene_occupancy, sphere_views, TinyMlp::init, Rng."""
    for name, seed, res, want in G["pins"]["scene_occupancy"]:
        s = ng.SynthScene(occupancy=name, scene_seed=seed, occ_base_res=res, L_C=8,
                          fine_table_len=64)
        assert crc(ng, s.base_words()) == want, (name, res)
    cams = ng.cameras(100, 8, 8)
    views = np.array([list(c.c2w) for c in cams], np.float64)
    assert crc(ng, views) == G["pins"]["sphere_views_100_2.9"]
    s = ng.SynthScene(occupancy="slab", occ_base_res=16, L_C=4, fine_table_len=64, fp16_exact=0)
    ws, bs = s.psi()
    w = np.concatenate([a.ravel() for a in ws])
    b = np.concatenate([a.ravel() for a in bs])
    assert [crc(ng, w), crc(ng, b)] == G["pins"]["tiny_mlp_init_psi_11"]
    u = np.zeros(1000, np.float64)
    ng.lib().ngprt_rng_uniform(7, -1.0, 1.0, 1000, u.ctypes.data_as(C.POINTER(C.c_double)))
    assert crc(ng, u) == G["pins"]["rng_uniform_7"]
    assert abs(ng.K_BASE_STEP - np.float32(G["pins"]["base_step"])) == 0


@pytest.mark.parametrize("case", CASES, ids=[c["name"] for c in CASES])
def test_oracle_render_matches_reference(ng, case):
    scene, cam, opts = make_case(ng, case)
    gold = G["cases"][case["name"]]
    assert scene_crc(ng, scene) == gold["scene_crc"]
    o = CpuScene(scene.desc_ptr, "oracle")
    rgb, stats = o.render(cam, opts.to_c(), nthreads=8)
    ref = np.load(GOLD / f"render_{case['name']}.npz")
    assert np.array_equal(stats, ref["stats"]), "MarchCounters differ"
    assert np.array_equal(rgb.view(np.uint32), ref["rgb"].view(np.uint32)), \
        f"rgb max abs {np.abs(rgb - ref['rgb']).max()}"
    # pyramid and distance grid the oracle built
    O = oracle()
    r0 = int(scene.desc.occ_base_res)
    lv = []
    for k in range(1, 5):
        n = ((r0 >> k) ** 3 + 63) // 64
        p = O.orc_scene_pyramid_level(o.h, k)
        lv.append(np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint64)), shape=(n,)).copy())
    assert crc(ng, np.concatenate(lv)) == gold["pyramid_crc"]
    if "dist_crc" in gold:
        dr = int(scene.desc.dist_res)
        p = O.orc_scene_dist(o.h)
        d = np.ctypeslib.as_array(C.cast(p, C.POINTER(C.c_uint8)), shape=(dr ** 3,))
        assert crc(ng, d) == gold["dist_crc"]
