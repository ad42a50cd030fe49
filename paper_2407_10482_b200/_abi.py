"""ctypes mirror of include/ngprt_cuda.h (the C ABI). Field order and types
match the header exactly; tests/test_abi.py checks the struct sizes against the
C compiler's."""
from __future__ import annotations

import ctypes as C
from pathlib import Path

import os  # noqa: E402

LIB_PATH = Path(os.environ.get("NGPRT_LIB") or
                Path(__file__).resolve().parent / "_lib" / "libngprt_cuda.so")

MAX_FINE_LEVELS = 4
PYRAMID_LEVELS = 5

OK, EINVAL, ECUDA, ENOMEM, EUNSUPPORTED, ENODEV, ENCCL = range(7)
STATUS_NAMES = {0: "OK", 1: "EINVAL", 2: "ECUDA", 3: "ENOMEM", 4: "EUNSUPPORTED", 5: "ENODEV",
                6: "ENCCL"}

FUSION = {"sum": 0, "shared_att_inv": 1, "separate_att_inv": 2, "shared_att_v": 3,
          "separate_att_v": 4, "mlp": 5}  # fusion_tag_name, fusion.hpp:53-63
STORAGE_AUTO, STORAGE_F32, STORAGE_F16 = 0, 1, 2
MLP_TENSOR, MLP_EXACT = 0, 1


class SceneDesc(C.Structure):
    _fields_ = [
        ("L", C.c_uint32),
        ("L_C", C.c_uint32),
        ("fine_res", C.c_uint32 * MAX_FINE_LEVELS),
        ("fine_table_len", C.c_uint64 * MAX_FINE_LEVELS),
        ("fine_hashed", C.c_uint8 * MAX_FINE_LEVELS),
        ("fusion_tag", C.c_uint8),
        ("storage", C.c_uint8),
        ("reserved", C.c_uint8 * 2),
        ("n_coarse", C.c_uint64),
        ("coarse_keys", C.POINTER(C.c_uint64)),
        ("coarse_rows", C.POINTER(C.c_float)),
        ("fine_tables", C.POINTER(C.c_float) * MAX_FINE_LEVELS),
        ("psi_w", C.POINTER(C.c_float) * 3),
        ("psi_b", C.POINTER(C.c_float) * 3),
        ("att_globals", C.POINTER(C.c_float)),
        ("occ_base_res", C.c_uint32),
        ("dist_res", C.c_uint32),
        ("pyramid_words", C.POINTER(C.c_uint64) * PYRAMID_LEVELS),
        ("dist_values", C.POINTER(C.c_uint8)),
        ("fusion_mlp_w", C.POINTER(C.c_float) * 2),
        ("fusion_mlp_b", C.POINTER(C.c_float) * 2),
    ]


class Camera(C.Structure):
    _fields_ = [
        ("c2w", C.c_double * 16),
        ("fx", C.c_double),
        ("fy", C.c_double),
        ("cx", C.c_double),
        ("cy", C.c_double),
        ("width", C.c_uint32),
        ("height", C.c_uint32),
    ]


class RenderOpts(C.Structure):
    _fields_ = [
        ("step", C.c_float),
        ("use_dist_grid", C.c_uint8),
        ("max_step_rule", C.c_uint8),
        ("early_stop", C.c_uint8),
        ("keep_level", C.c_int8),
        ("mlp_mode", C.c_uint8),
        ("profile", C.c_uint8),
        ("reserved", C.c_uint8 * 2),
        ("x0", C.c_uint32),
        ("y0", C.c_uint32),
        ("w", C.c_uint32),
        ("h", C.c_uint32),
        ("shard_world", C.c_uint32),
        ("shard_rank", C.c_uint32),
        ("shard_tile", C.c_uint32),
        ("reserved2", C.c_uint32),
    ]


class RayStats(C.Structure):
    _fields_ = [("marching", C.c_uint32), ("occupied", C.c_uint32), ("occ_acc", C.c_uint32),
                ("dist_acc", C.c_uint32)]


class SceneInfo(C.Structure):
    _fields_ = [
        ("device", C.c_int),
        ("storage", C.c_uint8),
        ("reserved", C.c_uint8 * 3),
        ("coarse_row_stride", C.c_uint32),
        ("device_bytes", C.c_uint64),
        ("coarse_bytes", C.c_uint64),
        ("fine_bytes", C.c_uint64),
        ("pyramid_bytes", C.c_uint64),
        ("dist_bytes", C.c_uint64),
        ("dev_pyramid", C.c_void_p * PYRAMID_LEVELS),
        ("dev_dist", C.c_void_p),
    ]


class SynthParams(C.Structure):
    _fields_ = [
        ("occupancy", C.c_char * 32),
        ("scene_seed", C.c_uint64),
        ("n_boxes", C.c_uint32),
        ("occ_base_res", C.c_uint32),
        ("dist_level", C.c_uint32),
        ("L", C.c_uint32),
        ("L_C", C.c_uint32),
        ("fusion_tag", C.c_uint32),
        ("fine_table_len", C.c_uint64),
        ("table_seed", C.c_uint64),
        ("coarse_seed", C.c_uint64),
        ("psi_seed", C.c_uint64),
        ("sigma_lo", C.c_double),
        ("sigma_hi", C.c_double),
        ("feat_scale", C.c_double),
        ("att_scale", C.c_double),
        ("psi_bias_scale", C.c_double),
        ("fp16_exact", C.c_uint8),
        ("reserved", C.c_uint8 * 7),
    ]


class ModelDesc(C.Structure):
    """ngprt_model_desc: a trained NgpRtModel (model.hpp:27-107), the bake input."""
    _fields_ = [
        ("L", C.c_uint32),
        ("L_C", C.c_uint32),
        ("coarse_res", C.c_uint32 * 6),
        ("coarse_table_len", C.c_uint64),
        ("coarse_tables", C.POINTER(C.c_float) * 6),
        ("aux_w", C.POINTER(C.c_float) * 2),
        ("aux_b", C.POINTER(C.c_float) * 2),
        ("fine_res", C.c_uint32 * MAX_FINE_LEVELS),
        ("fine_table_len", C.c_uint64 * MAX_FINE_LEVELS),
        ("fine_hashed", C.c_uint8 * MAX_FINE_LEVELS),
        ("fine_tables", C.POINTER(C.c_float) * MAX_FINE_LEVELS),
        ("psi_w", C.POINTER(C.c_float) * 3),
        ("psi_b", C.POINTER(C.c_float) * 3),
        ("fusion_tag", C.c_uint8),
        ("reserved", C.c_uint8 * 7),
        ("att_globals", C.POINTER(C.c_float)),
        ("fusion_mlp_w", C.POINTER(C.c_float) * 2),
        ("fusion_mlp_b", C.POINTER(C.c_float) * 2),
    ]


class BakeOpts(C.Structure):
    """ngprt_bake_opts: BakeOptions (baking.hpp:93-97)."""
    _fields_ = [
        ("cull_step", C.c_double),
        ("cull_alpha_thresh", C.c_double),
        ("dilate_voxels", C.c_uint32),
        ("reserved", C.c_uint32),
    ]


# name -> (restype, argtypes): every function declared in include/ngprt_cuda.h
SIGNATURES = {
    "ngprt_abi_version": (C.c_int, []),
    "ngprt_last_error": (C.c_char_p, []),
    "ngprt_scene_create": (C.c_int, [C.POINTER(SceneDesc), C.c_int, C.POINTER(C.c_void_p)]),
    "ngprt_scene_destroy": (None, [C.c_void_p]),
    "ngprt_scene_info_get": (C.c_int, [C.c_void_p, C.POINTER(SceneInfo)]),
    "ngprt_render": (C.c_int, [C.c_void_p, C.POINTER(Camera), C.c_int, C.POINTER(RenderOpts),
                               C.c_void_p, C.c_void_p, C.c_void_p]),
    "ngprt_render_host": (C.c_int, [C.c_void_p, C.POINTER(Camera), C.c_int, C.POINTER(RenderOpts),
                                    C.c_void_p, C.c_void_p]),
    "ngprt_render_host_async": (C.c_int, [C.c_void_p, C.POINTER(Camera), C.c_int,
                                          C.POINTER(RenderOpts), C.c_void_p, C.c_void_p]),
    "ngprt_render_host_wait": (C.c_int, [C.c_void_p]),
    "ngprt_render_timing": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                      C.POINTER(C.c_int)]),
    "ngprt_render_timing3": (C.c_int, [C.c_void_p, C.POINTER(C.c_float), C.POINTER(C.c_float),
                                       C.POINTER(C.c_float), C.POINTER(C.c_int)]),
    "ngprt_shard_pixels": (C.c_uint64, [C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32]),
    "ngprt_shard_assemble": (C.c_int, [C.c_void_p, C.c_uint32, C.c_uint32, C.c_uint32, C.c_uint32,
                                       C.c_uint32, C.c_uint32, C.c_void_p, C.c_void_p]),
    "ngprt_multi_create": (C.c_int, [C.POINTER(SceneDesc), C.POINTER(C.c_int), C.c_int,
                                     C.POINTER(C.c_void_p)]),
    "ngprt_multi_destroy": (None, [C.c_void_p]),
    "ngprt_multi_uses_nccl": (C.c_int, [C.c_void_p]),
    "ngprt_multi_scene": (C.c_void_p, [C.c_void_p, C.c_int]),
    "ngprt_multi_render_tiles": (C.c_int, [C.c_void_p, C.POINTER(Camera), C.c_int,
                                           C.POINTER(RenderOpts), C.c_uint32, C.c_void_p,
                                           C.c_void_p, C.c_void_p]),
    "ngprt_multi_render_cameras": (C.c_int, [C.c_void_p, C.POINTER(Camera), C.c_int,
                                             C.POINTER(RenderOpts), C.c_void_p, C.c_void_p,
                                             C.c_void_p]),
    "ngprt_build_pyramid": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p * (PYRAMID_LEVELS - 1),
                                      C.c_void_p]),
    "ngprt_build_distance_grid": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p]),
    "ngprt_test_expf": (C.c_int, [C.c_void_p, C.c_void_p, C.c_uint64, C.c_void_p]),
    "ngprt_test_expf_range": (C.c_int, [C.c_uint32, C.c_uint64, C.c_void_p, C.c_void_p]),
    "ngprt_test_march_segments": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.c_float, C.c_int,
                                            C.c_int, C.c_int, C.c_void_p, C.c_void_p, C.c_void_p,
                                            C.c_void_p, C.c_void_p, C.c_void_p]),
    "ngprt_test_hash_index": (C.c_int, [C.c_void_p, C.c_uint64, C.c_uint32, C.c_uint64, C.c_uint8,
                                        C.c_void_p, C.c_void_p]),
    "ngprt_baked_load": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p)]),
    "ngprt_baked_desc": (C.POINTER(SceneDesc), [C.c_void_p]),
    "ngprt_baked_free": (None, [C.c_void_p]),
    "ngprt_scene_load": (C.c_int, [C.c_char_p, C.c_int, C.POINTER(C.c_void_p)]),
    "ngprt_baked_save": (C.c_int, [C.c_void_p, C.c_char_p]),
    "ngprt_bake": (C.c_int, [C.POINTER(ModelDesc), C.c_void_p, C.c_uint32, C.POINTER(BakeOpts),
                             C.c_int, C.POINTER(C.c_void_p)]),
    "ngprt_synth_default_params": (None, [C.POINTER(SynthParams)]),
    "ngprt_synth_create": (C.c_int, [C.POINTER(SynthParams), C.POINTER(C.c_void_p)]),
    "ngprt_synth_last_error": (C.c_char_p, []),
    "ngprt_synth_desc": (C.POINTER(SceneDesc), [C.c_void_p]),
    "ngprt_synth_destroy": (None, [C.c_void_p]),
    "ngprt_synth_model_create": (C.c_int, [C.POINTER(SynthParams), C.POINTER(C.c_void_p)]),
    "ngprt_synth_model_desc": (C.POINTER(ModelDesc), [C.c_void_p]),
    "ngprt_synth_model_train_words": (C.POINTER(C.c_uint64), [C.c_void_p, C.POINTER(C.c_uint32)]),
    "ngprt_synth_model_destroy": (None, [C.c_void_p]),
    "ngprt_synth_cameras": (C.c_int, [C.c_int, C.c_double, C.c_uint32, C.c_uint32,
                                      C.POINTER(Camera)]),
    "ngprt_crc32": (C.c_uint32, [C.c_void_p, C.c_uint64, C.c_uint32]),
    "ngprt_rng_uniform": (None, [C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                 C.POINTER(C.c_double)]),
}

_lib = None


def lib() -> C.CDLL:
    """Load the native library. Fails loudly: there is no CPU fallback."""
    global _lib
    if _lib is None:
        if not LIB_PATH.exists():
            raise RuntimeError(
                f"native library {LIB_PATH} is missing: run __graft_entry__.build() "
                "(nvcc, sm_100a). The renderer has no CPU fallback.")
        L = C.CDLL(str(LIB_PATH))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        _lib = L
    return _lib


def bind_synth(L: C.CDLL) -> None:
    """Set the ngprt_synth_* signatures on a library that exports the synthetic-scene
    generator (the product library, or oracle/_ref's reference checker, which links
    the same host-only csrc/synth.cpp)."""
    if getattr(L, "_ngprt_synth_bound", False):
        return
    for name, (res, args) in SIGNATURES.items():
        if name.startswith("ngprt_synth_") and hasattr(L, name):
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
    L._ngprt_synth_bound = True


class NgprtError(RuntimeError):
    def __init__(self, status: int, where: str):
        msg = lib().ngprt_last_error().decode(errors="replace")
        super().__init__(f"{where}: {STATUS_NAMES.get(status, status)}: {msg}")
        self.status = status


def check(status: int, where: str) -> None:
    if status != OK:
        raise NgprtError(status, where)
