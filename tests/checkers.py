"""ctypes access to the CPU checkers (TEST INFRASTRUCTURE):

  oracle()  -> oracle/_build/libngprt_oracle.so, the C restatement of the
               reference render path (oracle/ngprt_oracle.c). Always buildable.
  ref()     -> oracle/_ref/libngprt_ref.so, the unmodified reference headers
               compiled in place (oracle/ref_driver.cpp). Only buildable where
               /root/reference exists; None elsewhere.
"""
from __future__ import annotations

import ctypes as C
import subprocess
from pathlib import Path

import numpy as np

from paper_2407_10482_b200._abi import Camera, RenderOpts, SceneDesc

ROOT = Path(__file__).resolve().parents[1]
ORACLE_SO = ROOT / "oracle" / "_build" / "libngprt_oracle.so"
REF_SO = ROOT / "oracle" / "_ref" / "libngprt_ref.so"

_oracle = None
_ref = None

P = C.c_void_p
F = C.POINTER(C.c_float)
U32 = C.POINTER(C.c_uint32)


def oracle() -> C.CDLL:
    global _oracle
    if _oracle is None:
        if not ORACLE_SO.exists():
            subprocess.run(["make", "-C", str(ROOT / "oracle"), "oracle"], check=True,
                           capture_output=True)
        L = C.CDLL(str(ORACLE_SO))
        L.orc_scene_create.restype = P
        L.orc_scene_create.argtypes = [C.POINTER(SceneDesc)]
        L.orc_scene_destroy.argtypes = [P]
        L.orc_render.restype = C.c_int
        L.orc_render.argtypes = [P, C.POINTER(Camera), C.POINTER(RenderOpts), F, U32, C.c_int]
        L.orc_build_pyramid.argtypes = [P, C.c_int, P]
        L.orc_build_distance_grid.argtypes = [P, C.c_int, P]
        L.orc_hash_index.restype = C.c_uint64
        L.orc_hash_index.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int32, C.c_int32, C.c_int32]
        L.orc_expf.restype = C.c_float
        L.orc_expf.argtypes = [C.c_float]
        L.orc_sh_encode.argtypes = [F, F]
        L.orc_activate_density.restype = C.c_float
        L.orc_activate_density.argtypes = [C.c_float]
        L.orc_activate_sigmoid.restype = C.c_float
        L.orc_activate_sigmoid.argtypes = [C.c_float]
        L.orc_alpha.restype = C.c_float
        L.orc_alpha.argtypes = [C.c_float, C.c_float]
        L.orc_decode_point.argtypes = [P, F, C.c_int, F]
        L.orc_generate_ray.restype = C.c_int
        L.orc_generate_ray.argtypes = [C.POINTER(Camera), C.c_double, C.c_double, F]
        L.orc_scene_pyramid_level.restype = P
        L.orc_scene_pyramid_level.argtypes = [P, C.c_int]
        L.orc_scene_dist.restype = P
        L.orc_scene_dist.argtypes = [P]
        _oracle = L
    return _oracle


def ref():
    """The compiled reference, or None when it is not available (GPU box without it)."""
    global _ref
    if _ref is None:
        if not REF_SO.exists():
            if not Path("/root/reference/proj/include").exists():
                return None
            subprocess.run(["make", "-C", str(ROOT / "oracle"), "ref"], check=True,
                           capture_output=True)
        L = C.CDLL(str(REF_SO))
        L.ref_last_error.restype = C.c_char_p
        L.ref_scene_create.restype = P
        L.ref_scene_create.argtypes = [C.POINTER(SceneDesc)]
        L.ref_scene_destroy.argtypes = [P]
        L.ref_render.restype = C.c_int
        L.ref_render.argtypes = [P, C.POINTER(Camera), C.POINTER(RenderOpts), F, U32, C.c_int]
        L.ref_build_pyramid.argtypes = [P, C.c_int, P]
        L.ref_build_distance_grid.argtypes = [P, C.c_int, P]
        L.ref_hash_index.restype = C.c_uint64
        L.ref_hash_index.argtypes = [C.c_int, C.c_uint64, C.c_int, C.c_int, C.c_int]
        L.ref_sh_encode.argtypes = [F, F]
        for n in ("ref_activate_density", "ref_activate_sigmoid", "ref_expf"):
            getattr(L, n).restype = C.c_float
            getattr(L, n).argtypes = [C.c_float]
        L.ref_alpha.restype = C.c_float
        L.ref_alpha.argtypes = [C.c_float, C.c_float]
        L.ref_composite.argtypes = [C.c_int, F, F, F, C.c_int, F]
        L.ref_decode_point.restype = C.c_int
        L.ref_decode_point.argtypes = [P, F, C.c_int, F]
        L.ref_shade.restype = C.c_int
        L.ref_shade.argtypes = [P, F, F, F]
        L.ref_generate_ray.restype = C.c_int
        L.ref_generate_ray.argtypes = [C.POINTER(Camera), C.c_double, C.c_double, F]
        L.ref_march_segments.restype = C.c_int
        L.ref_march_segments.argtypes = [P, F, C.c_float, C.c_int, C.c_int, U32, F, C.c_int, F,
                                         C.c_int, C.POINTER(C.c_int), C.POINTER(C.c_int)]
        L.ref_dda_hits.restype = C.c_int
        L.ref_dda_hits.argtypes = [P, F, C.c_float, C.c_float, C.c_double]
        L.ref_scene_occupancy.restype = C.c_int
        L.ref_scene_occupancy.argtypes = [C.c_char_p, C.c_uint64, C.c_int, P]
        L.ref_scene_boxes.restype = C.c_int
        L.ref_scene_boxes.argtypes = [C.c_char_p, C.c_uint64, C.POINTER(C.c_double), C.c_int]
        L.ref_sphere_views.argtypes = [C.c_int, C.c_double, C.POINTER(C.c_double)]
        L.ref_tiny_mlp_init.argtypes = [C.POINTER(C.c_int), C.c_int, C.c_uint64, F, F]
        L.ref_tiny_mlp_forward.argtypes = [C.POINTER(C.c_int), C.c_int, F, F, F, F]
        L.ref_rng_uniform.argtypes = [C.c_uint64, C.c_double, C.c_double, C.c_uint64,
                                      C.POINTER(C.c_double)]
        L.ref_crc32.restype = C.c_uint32
        L.ref_crc32.argtypes = [P, C.c_uint64]
        L.ref_base_step.restype = C.c_double
        L.ref_save_baked.restype = C.c_int
        L.ref_save_baked.argtypes = [P, C.c_char_p]
        L.ref_bake.restype = C.c_int
        L.ref_bake.argtypes = [C.c_void_p, C.c_void_p, C.c_int, C.c_void_p, C.c_char_p]
        _ref = L
    return _ref


def oracle_synth() -> C.CDLL:
    """The C restatement's library; it links the synthetic-scene generator too."""
    return oracle()


def fptr(a: np.ndarray):
    assert a.dtype == np.float32 and a.flags.c_contiguous
    return a.ctypes.data_as(F)


def u32ptr(a: np.ndarray):
    assert a.dtype == np.uint32 and a.flags.c_contiguous
    return a.ctypes.data_as(U32)


def out_hw(cam: Camera, opts: RenderOpts):
    if opts.w and opts.h:
        return int(opts.h), int(opts.w)
    return int(cam.height), int(cam.width)


class CpuScene:
    """A scene loaded into one of the CPU checkers ('oracle' or 'ref')."""

    def __init__(self, desc_ptr, which: str = "oracle"):
        self.which = which
        self.L = oracle() if which == "oracle" else ref()
        if self.L is None:
            raise RuntimeError("reference checker unavailable")
        create = self.L.orc_scene_create if which == "oracle" else self.L.ref_scene_create
        self.h = create(desc_ptr)
        if not self.h:
            msg = self.L.ref_last_error().decode() if which == "ref" else "orc_scene_create"
            raise RuntimeError(msg)

    def render(self, cam: Camera, opts: RenderOpts, nthreads: int = 0):
        h, w = out_hw(cam, opts)
        rgb = np.zeros((h, w, 3), np.float32)
        stats = np.zeros((h, w, 4), np.uint32)
        fn = self.L.orc_render if self.which == "oracle" else self.L.ref_render
        rc = fn(self.h, C.byref(cam), C.byref(opts), fptr(rgb), u32ptr(stats), nthreads)
        if rc != 0:
            raise RuntimeError(f"{self.which} render failed")
        return rgb, stats

    def close(self):
        if self.h:
            (self.L.orc_scene_destroy if self.which == "oracle" else self.L.ref_scene_destroy)(self.h)
            self.h = None

    def __del__(self):
        self.close()


def host_expf_range(first: int, n: int, nthreads: int = 0) -> np.ndarray:
    """bits(glibc expf(x)) for the n consecutive float bit patterns from `first`."""
    L = oracle()
    L.orc_expf_range.argtypes = [C.c_uint32, C.c_uint64, U32, C.c_int]
    out = np.empty(n, np.uint32)
    L.orc_expf_range(first, n, u32ptr(out), nthreads)
    return out
