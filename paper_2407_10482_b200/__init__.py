"""B200-native NGP-RT per-ray renderer (arXiv 2407.10482 render path).

The product is the C-ABI library _lib/libngprt_cuda.so (include/ngprt_cuda.h)
built from csrc/ for sm_100a; this package is the thin host mirror over it.
"""
from ._abi import NgprtError, lib  # noqa: F401
from .renderer import (CONFIGS, K_BASE_STEP, BakedFile, Opts, Scene, SynthModel, SynthScene, bake,
                       build_distance_grid,  # noqa: F401
                       build_pyramid, camera_array, cameras, render, render_host, render_host_async,
                       render_host_wait, render_timing, render_timing3, shard_assemble,
                       shard_pixels)

__all__ = ["CONFIGS", "K_BASE_STEP", "BakedFile", "Opts", "Scene", "SynthModel", "SynthScene", "bake", "NgprtError", "lib",
           "build_distance_grid", "build_pyramid", "camera_array", "cameras", "render",
           "render_host", "render_host_async", "render_host_wait", "render_timing", "render_timing3",
           "shard_assemble", "shard_pixels"]
