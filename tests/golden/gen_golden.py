"""Generate the golden fixtures in tests/golden/ FROM THE REFERENCE ITSELF.

Runs only where /root/reference exists (this container): it builds
oracle/_ref/libngprt_ref.so (the unmodified reference headers compiled in
place by oracle/Makefile) and records what the reference's own functions
return for:
  * every parity case of tests/cases.py: RGB (f32) and per-ray MarchCounters of
    the canonical render_ray composition, plus CRC-32s of the
    synthetic scene arrays, of build_pyramid levels and of build_distance_grid;
  * known-answer tests of the path's functions (hash_index, sh_encode,
    activate_density/sigmoid, alpha, composite, TinyMlp::forward, expf);
  * pins for the synthetic-scene generator (make_scene/scene_occupancy,
    sphere_views, TinyMlp::init, Rng).
Usage: python tests/golden/gen_golden.py
"""
from __future__ import annotations

import ctypes as C
import json
import sys
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
sys.path.insert(0, str(HERE.parents[1]))
sys.path.insert(0, str(HERE.parent))

import paper_2407_10482_b200 as ng  # noqa: E402
from cases import CASES, make_case, random_grid_words, scene_crc  # noqa: E402
from checkers import CpuScene, fptr, ref  # noqa: E402

F = C.POINTER(C.c_float)


def fbits(x):
    return int(np.float32(x).view(np.uint32))


def crc(a):
    a = np.ascontiguousarray(a)
    return int(ng.lib().ngprt_crc32(a.ctypes.data, a.nbytes, 0))


def main():
    R = ref()
    assert R is not None, "needs /root/reference (compiled reference)"
    kat = {}

    # ---- hash_index (hash_grid.hpp:83-94); SPEC.md:137-139 examples included ----
    rs = np.random.RandomState(5)
    hashes = []
    for res, maxlen in [(16, 1 << 19), (1024, 1 << 19), (1024, 1 << 21), (2048, 1 << 22),
                        (4096, 1 << 22), (8192, 1 << 19), (1024, 3001), (1024, 1 << 32)]:
        pts = [(0, 0, 0), (1, 0, 0), (1, 2, 3), (res, res, res)] + \
              [tuple(int(v) for v in rs.randint(0, res + 1, 3)) for _ in range(24)]
        for (x, y, z) in pts:
            hashes.append([res, maxlen, x, y, z, int(R.ref_hash_index(res, maxlen, x, y, z))])
    kat["hash_index"] = hashes

    # ---- scalar activations (nn.hpp:80-94, volume.hpp:30-33) ----
    xs = np.concatenate([np.float32([0, np.log(2), 40, 1, 50, -50, 15, -15, 16, -16, 88.7, -104,
                                     1e-30, -1e-30, 3e-8, -3e-8]),
                         rs.uniform(-20, 20, 200).astype(np.float32)])
    kat["density"] = [[fbits(x), fbits(R.ref_activate_density(float(x)))] for x in xs]
    kat["sigmoid"] = [[fbits(x), fbits(R.ref_activate_sigmoid(float(x)))] for x in xs]
    sig = np.abs(rs.standard_normal(100).astype(np.float32)) * 50
    kat["alpha"] = [[fbits(s), fbits(d), fbits(R.ref_alpha(float(s), float(d)))]
                    for s, d in zip(np.concatenate([[3.0], sig]).astype(np.float32),
                                    np.concatenate([[0.1], np.full(100, ng.K_BASE_STEP)]).astype(np.float32))]
    ex = np.concatenate([rs.uniform(-110, 90, 4000), rs.uniform(-1, 1, 4000),
                         rs.standard_normal(2000) * 1e-6]).astype(np.float32)
    ex = np.concatenate([ex, np.float32([np.inf, -np.inf, 88.72283, 88.72284, -103.97208,
                                          -103.97209, 0.0, -0.0])])
    kat["expf"] = [[fbits(x), fbits(R.ref_expf(float(x)))] for x in ex]

    # ---- sh_encode (nn.hpp:107-132) ----
    dirs = [np.float32([0, 0, 1])]
    for _ in range(40):
        v = rs.standard_normal(3)
        dirs.append((v / np.linalg.norm(v)).astype(np.float32))
    shs = []
    for d in dirs:
        d = np.ascontiguousarray(d, np.float32)
        o = np.zeros(16, np.float32)
        R.ref_sh_encode(fptr(d), fptr(o))
        shs.append([[fbits(v) for v in d], [fbits(v) for v in o]])
    kat["sh_encode"] = shs

    # ---- composite (volume.hpp:51-75), incl. SPEC.md:297-299 ----
    comps = []
    for n, early in [(0, 1), (2, 0), (8, 1), (40, 1), (40, 0)]:
        t = np.cumsum(np.full(n, 0.01, np.float32)).astype(np.float32)
        dl = np.full(n, ng.K_BASE_STEP, np.float32)
        feat = rs.uniform(-1, 6, (n, 8)).astype(np.float32)
        out = np.zeros(9, np.float32)
        R.ref_composite(n, fptr(t), fptr(dl), fptr(np.ascontiguousarray(feat)), early, fptr(out))
        comps.append({"n": n, "early": early, "t": [fbits(v) for v in t],
                      "delta": [fbits(v) for v in dl], "feat": [fbits(v) for v in feat.ravel()],
                      "out": [fbits(v) for v in out]})
    kat["composite"] = comps

    # ---- TinyMlp::forward (nn.hpp:175-196) on the psi shape ----
    widths = (C.c_int * 4)(23, 64, 64, 3)
    w = rs.uniform(-0.3, 0.3, 23 * 64 + 64 * 64 + 64 * 3).astype(np.float32)
    b = rs.uniform(-0.1, 0.1, 64 + 64 + 3).astype(np.float32)
    mlp = []
    for _ in range(8):
        x = rs.uniform(-2, 2, 23).astype(np.float32)
        o = np.zeros(3, np.float32)
        R.ref_tiny_mlp_forward(widths, 4, fptr(w), fptr(b), fptr(x), fptr(o))
        mlp.append({"in": [fbits(v) for v in x], "out": [fbits(v) for v in o]})
    kat["mlp"] = {"w": [fbits(v) for v in w], "b": [fbits(v) for v in b], "cases": mlp}

    # ---- synthetic-generator pins (scene.hpp, nn.hpp, common.hpp) ----
    pins = {"scene_occupancy": []}
    for name in ["bench", "toy", "slab"]:
        for res in [32, 64, 128, 256, 512]:
            words = np.zeros((res ** 3 + 63) // 64, np.uint64)
            R.ref_scene_occupancy(name.encode(), 41, res, words.ctypes.data)
            pins["scene_occupancy"].append([name, 41, res, crc(words)])
    views = np.zeros(16 * 100, np.float64)
    R.ref_sphere_views(100, 2.9, views.ctypes.data_as(C.POINTER(C.c_double)))
    pins["sphere_views_100_2.9"] = crc(views)
    wi = np.zeros(23 * 64 + 64 * 64 + 64 * 3, np.float32)
    bi = np.zeros(64 + 64 + 3, np.float32)
    R.ref_tiny_mlp_init(widths, 4, 11, fptr(wi), fptr(bi))
    pins["tiny_mlp_init_psi_11"] = [crc(wi), crc(bi)]
    u = np.zeros(1000, np.float64)
    R.ref_rng_uniform(7, -1.0, 1.0, 1000, u.ctypes.data_as(C.POINTER(C.c_double)))
    pins["rng_uniform_7"] = crc(u)
    pins["base_step"] = float(R.ref_base_step())
    kat["pins"] = pins

    # ---- distance transform on random grids (occupancy.hpp:136-194) ----
    dts = []
    for res, dens, seed in [(32, 0.0, 1), (32, 1.0, 2), (64, 1e-4, 3), (64, 0.003, 4),
                            (64, 0.05, 5), (48, 0.2, 6), (128, 1e-5, 7), (128, 0.001, 8)]:
        words = random_grid_words(ng, res, dens, seed)
        out = np.zeros(res ** 3, np.uint8)
        R.ref_build_distance_grid(words.ctypes.data, res, out.ctypes.data)
        dts.append([res, dens, seed, crc(words), crc(out)])
    # single voxel at (128,128,128)
    words = np.zeros(256 ** 3 // 64, np.uint64)
    i = 128 + 256 * (128 + 256 * 128)
    words[i >> 6] |= np.uint64(1) << np.uint64(i & 63)
    out = np.zeros(256 ** 3, np.uint8)
    R.ref_build_distance_grid(words.ctypes.data, 256, out.ctypes.data)
    kat["dt_single_voxel"] = {"q": [133, 128, 128], "value": int(out[133 + 256 * (128 + 256 * 128)]),
                              "crc": crc(out)}
    kat["dt_random"] = dts

    # ---- full-path parity cases ----
    cases = {}
    for case in CASES:
        scene, cam, opts = make_case(ng, case)
        rs_ = CpuScene(scene.desc_ptr, "ref")
        rgb, stats = rs_.render(cam, opts.to_c(), nthreads=8)
        r0 = int(scene.desc.occ_base_res)
        levels = np.zeros(sum(((r0 >> k) ** 3 + 63) // 64 for k in range(1, 5)), np.uint64)
        R.ref_build_pyramid(scene.base_words().ctypes.data, r0, levels.ctypes.data)
        entry = {"scene_crc": scene_crc(ng, scene), "pyramid_crc": crc(levels)}
        if scene.desc.dist_res:
            dr = int(scene.desc.dist_res)
            k = [r0 >> j for j in range(5)].index(dr)
            off = sum(((r0 >> j) ** 3 + 63) // 64 for j in range(1, k))
            src = scene.base_words() if k == 0 else levels[off: off + ((dr ** 3 + 63) // 64)]
            dist = np.zeros(dr ** 3, np.uint8)
            R.ref_build_distance_grid(np.ascontiguousarray(src).ctypes.data, dr, dist.ctypes.data)
            entry["dist_crc"] = crc(dist)
        np.savez_compressed(HERE / f"render_{case['name']}.npz", rgb=rgb, stats=stats)
        s = stats.reshape(-1, 4).astype(np.float64).mean(0)
        entry["mean_stats"] = [round(float(v), 4) for v in s]
        cases[case["name"]] = entry
        print(case["name"], entry["mean_stats"], "shaded", float((rgb.sum(-1) > 0).mean()))
        rs_.close()
        scene.close()
    kat["cases"] = cases
    (HERE / "golden.json").write_text(json.dumps(kat, indent=0))
    print("wrote", HERE / "golden.json")


if __name__ == "__main__":
    main()
