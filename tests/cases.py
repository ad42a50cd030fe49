"""Parity cases shared by the golden-fixture generator, the CPU oracle tests and
the GPU parity tests. Each case is a seeded synthetic scene (ngprt_synth), one
camera of sphere_views(n, 2.9) and render options. Together they cover every
fusion mode of the render path (fusion.hpp:44-51 minus the MLP ablation),
L = 2..4, fp16 and f32 storage, power-of-two and generic table lengths,
with/without the distance grid, early stop on/off, max_step_rule, keep_level,
non-default step, and a pixel window of a 1080p camera."""
from __future__ import annotations

import numpy as np

K_BASE_STEP = float(np.float32(2.0 * np.sqrt(3.0) / 512.0))

CASES = [
    dict(name="bench_l2", scene=dict(occupancy="bench", occ_base_res=128, L=2, L_C=128,
                                     fine_table_len=1 << 14),
         cam=dict(w=64, h=64, n=4, i=0), opts=dict()),
    dict(name="c1_l4_256", scene=dict(occupancy="bench", occ_base_res=256, L=4, L_C=256,
                                      fine_table_len=1 << 19),
         cam=dict(w=64, h=64, n=1, i=0), opts=dict()),
    dict(name="toy_sum_l3", scene=dict(occupancy="toy", occ_base_res=128, L=3, L_C=64,
                                       fine_table_len=1 << 15, fusion_tag="sum"),
         cam=dict(w=56, h=48, n=4, i=1), opts=dict()),
    dict(name="slab_shared_inv", scene=dict(occupancy="slab", occ_base_res=64, L=2, L_C=64,
                                            fine_table_len=1 << 12, fusion_tag="shared_att_inv"),
         cam=dict(w=48, h=48, n=4, i=2), opts=dict()),
    dict(name="blob_sep_inv_maxstep", scene=dict(occupancy="blob", occ_base_res=128, L=2, L_C=128,
                                                 fine_table_len=1 << 16,
                                                 fusion_tag="separate_att_inv"),
         cam=dict(w=64, h=48, n=4, i=3), opts=dict(max_step_rule=True)),
    dict(name="bench_nogrid_noearly", scene=dict(occupancy="bench", occ_base_res=128, L=2,
                                                 L_C=128, fine_table_len=1 << 14),
         cam=dict(w=48, h=48, n=4, i=1), opts=dict(use_dist_grid=False, early_stop=False)),
    dict(name="bench_keep2_shared_v", scene=dict(occupancy="bench", occ_base_res=128, L=3,
                                                 L_C=128, fine_table_len=1 << 14,
                                                 fusion_tag="shared_att_v"),
         cam=dict(w=48, h=48, n=4, i=2), opts=dict(keep_level=2)),
    dict(name="f32_storage_bias", scene=dict(occupancy="bench", occ_base_res=128, L=2, L_C=96,
                                             fine_table_len=1 << 13, fp16_exact=0,
                                             psi_bias_scale=0.2, sigma_lo=-1.0, sigma_hi=3.0),
         cam=dict(w=48, h=40, n=4, i=0), opts=dict()),
    dict(name="nonpow2_table_step2", scene=dict(occupancy="toy", occ_base_res=64, L=2, L_C=64,
                                                fine_table_len=3001),
         cam=dict(w=48, h=48, n=4, i=3), opts=dict(step=2 * K_BASE_STEP)),
    dict(name="mlp_fusion_l2", scene=dict(occupancy="bench", occ_base_res=128, L=2, L_C=128,
                                          fine_table_len=1 << 14, fusion_tag="mlp",
                                          psi_bias_scale=0.1),
         cam=dict(w=48, h=48, n=4, i=0), opts=dict()),
    dict(name="mlp_fusion_l4_keep3", scene=dict(occupancy="toy", occ_base_res=64, L=4, L_C=64,
                                                fine_table_len=1 << 12, fusion_tag="mlp"),
         cam=dict(w=40, h=40, n=4, i=2), opts=dict(keep_level=3)),
    dict(name="mip360_window", scene=dict(occupancy="mip360", occ_base_res=512, L=2, L_C=512,
                                          fine_table_len=1 << 21, sigma_lo=1.0, sigma_hi=4.0),
         cam=dict(w=1920, h=1080, n=1, i=0), opts=dict(window=(928, 508, 64, 64))),
]

CASE_BY_NAME = {c["name"]: c for c in CASES}


def make_case(ng, case):
    """-> (SynthScene, Camera, Opts) for a case."""
    scene = ng.SynthScene(**case["scene"])
    cm = case["cam"]
    cam = ng.cameras(cm["n"], cm["w"], cm["h"])[cm["i"]]
    opts = ng.Opts(**case["opts"])
    return scene, cam, opts


def scene_crc(ng, scene) -> dict:
    """CRC-32 of every array of a synthetic scene (pins the generator)."""
    crc = lambda a: int(ng.lib().ngprt_crc32(a.ctypes.data, a.nbytes, 0))
    ws, bs = scene.psi()
    out = {"keys": crc(np.ascontiguousarray(scene.coarse_keys())),
           "rows": crc(np.ascontiguousarray(scene.coarse_rows())),
           "base": crc(np.ascontiguousarray(scene.base_words())),
           "psi": [crc(np.ascontiguousarray(w)) for w in ws] + [crc(np.ascontiguousarray(b)) for b in bs]}
    out["fine"] = [crc(np.ascontiguousarray(scene.fine_table(l))) for l in range(scene.L)]
    return out


def random_grid_words(ng, res: int, density: float, seed: int) -> np.ndarray:
    """A reproducible random occupancy grid from the splitmix64 stream (common.hpp:46-60)."""
    import ctypes as C
    n = res ** 3
    u = np.empty(n, np.float64)
    ng.lib().ngprt_rng_uniform(seed, 0.0, 1.0, n, u.ctypes.data_as(C.POINTER(C.c_double)))
    bits = (u < density).astype(np.uint8)
    packed = np.packbits(bits, bitorder="little")
    words = np.zeros((n + 63) // 64, np.uint64)
    words.view(np.uint8)[: packed.size] = packed
    return words


# Bake cases (baking.hpp:107-202): a seeded synthetic NgpRtModel (SynthModel)
# and its training occupancy. `scene` keys go to ngprt_synth_model_create
# (occ_base_res = training resolution); sigma_lo = sigma_hi sets the aux
# decoder's density bias so the cull keeps roughly half the voxels. Together
# they cover every fusion mode including the MLP ablation, L = 2..4, L_C above,
# equal to and below the training resolution, dilation 0..2, non-default
# cull step and threshold.
BAKE_CASES = [
    dict(name="toy_sepv_up2", scene=dict(occupancy="toy", occ_base_res=64, L=2, L_C=128,
                                         fine_table_len=1 << 16, sigma_lo=-0.5, sigma_hi=-0.5),
         opts=dict()),
    dict(name="bench_sharedinv_eq", scene=dict(occupancy="bench", occ_base_res=64, L=3, L_C=64,
                                               fine_table_len=1 << 15, fusion_tag="shared_att_inv",
                                               sigma_lo=-0.5, sigma_hi=-0.5),
         opts=dict()),
    dict(name="toy_sum_down2_dil2", scene=dict(occupancy="toy", occ_base_res=128, L=2, L_C=64,
                                               fine_table_len=1 << 14, fusion_tag="sum",
                                               sigma_lo=0.0, sigma_hi=0.0),
         opts=dict(dilate_voxels=2)),
    dict(name="toy_mlp_l4_down2_nodil", scene=dict(occupancy="toy", occ_base_res=64, L=4, L_C=32,
                                                   fine_table_len=1 << 12, fusion_tag="mlp",
                                                   sigma_lo=-0.5, sigma_hi=-0.5),
         opts=dict(dilate_voxels=0)),
    dict(name="blob_sepinv_up4_step", scene=dict(occupancy="blob", occ_base_res=32, L=2, L_C=128,
                                                 fine_table_len=1 << 13,
                                                 fusion_tag="separate_att_inv",
                                                 sigma_lo=-1.0, sigma_hi=-1.0),
         opts=dict(cull_step=0.01, cull_alpha_thresh=0.01)),
    dict(name="bench_sharedv_l2", scene=dict(occupancy="bench", occ_base_res=64, L=2, L_C=128,
                                             fine_table_len=1 << 16, fusion_tag="shared_att_v",
                                             sigma_lo=-0.5, sigma_hi=-0.5),
         opts=dict()),
]


def bake_opts(o: dict):
    from paper_2407_10482_b200 import _abi
    return _abi.BakeOpts(o.get("cull_step", 0.0), o.get("cull_alpha_thresh", 0.005),
                         o.get("dilate_voxels", 1), 0)
