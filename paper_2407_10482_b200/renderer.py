"""Host-side API of the B200 NGP-RT renderer, mirroring the reference's render
path interface (names and argument meaning follow /root/reference/proj/include/ngprt):

    BakedScene            baking.hpp:55-64        -> Scene (device-resident, immutable)
    PosedDataset / Frame  scene.hpp:191-201       -> Camera (ngprt_camera)
    sphere_views          scene.hpp:254-265       -> cameras()
    render_ray over a frame     -> render() / render_host()
    MarchCounters         occupancy.hpp:197-210   -> the `stats` output (marching, occupied,
                                                     occ_acc, dist_acc per ray)
    build_pyramid         occupancy.hpp:114-119   -> build_pyramid()
    build_distance_grid   occupancy.hpp:136-194   -> build_distance_grid()

Everything below calls the C ABI (include/ngprt_cuda.h) in
_lib/libngprt_cuda.so; errors surface as NgprtError carrying the library's
message (the reference throws std::invalid_argument / domain_error etc.).
There is no CPU path: without the native library and a B200 these raise.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass

import numpy as np

from . import _abi
from ._abi import Camera, RenderOpts, SceneDesc, SceneInfo, SynthParams, check, lib

K_BASE_STEP = float(np.float32(2.0 * np.sqrt(3.0) / 512.0))  # kBaseStep, config.hpp:11


# ---------------------------------------------------------------------------
# Synthetic scenes (host)
# ---------------------------------------------------------------------------
# Named BASELINE.json configs -> synthetic scene parameters.
CONFIGS = {
    # 1. random-init NGP-RT scene, "16 levels" -> L = 4 (reference max), 2^19, 128^3 DT, 256x256
    "c1_256": dict(occupancy="bench", occ_base_res=256, L=4, L_C=256, fine_table_len=1 << 19,
                   width=256, height=256, n_cams=1),
    # 2. 800x800 Blender-style bounded blob, 100-camera orbit (EncodingConfig{} defaults)
    "c2_blob800": dict(occupancy="blob", occ_base_res=512, L=2, L_C=512, fine_table_len=1 << 22,
                       width=800, height=800, n_cams=100),
    # 3. 1920x1080 Mip-NeRF-360-shaped scene, 2^21 entries/level (the 108 fps headline),
    #    calibrated to PAPER Table 4 (46.7 marching / 17.3 occupied points per ray)
    "c3_1080p": dict(occupancy="mip360c", n_boxes=16, occ_base_res=512, L=2, L_C=512,
                     fine_table_len=1 << 21, sigma_lo=1.85, sigma_hi=4.85,
                     width=1920, height=1080, n_cams=1),
    # 3 with values that are not fp16-representable: f32 storage (the real-scene case:
    # any bake or reference .ngrt), bit-exact, twice the gathered bytes
    "c3_1080p_f32": dict(occupancy="mip360c", n_boxes=16, occ_base_res=512, L=2, L_C=512,
                         fine_table_len=1 << 21, sigma_lo=1.85, sigma_hi=4.85, fp16_exact=0,
                         width=1920, height=1080, n_cams=1),
    # 3'. the round-1 Mip-NeRF-360-shaped preset (60 marching / 13.5 occupied per ray)
    "c3_mip360": dict(occupancy="mip360", occ_base_res=512, L=2, L_C=512,
                      fine_table_len=1 << 21, sigma_lo=1.0, sigma_hi=4.0,
                      width=1920, height=1080, n_cams=1),
    # 4. 1080p 64-camera batch (sharded across GPUs), config 3's scene
    "c4_1080p_x64": dict(occupancy="mip360c", n_boxes=16, occ_base_res=512, L=2, L_C=512,
                         fine_table_len=1 << 21, sigma_lo=1.85, sigma_hi=4.85,
                         width=1920, height=1080, n_cams=64),
    # 5. 3840x2160, 2^22 entries/level, occupancy sweep (n_boxes)
    "c5_2160p": dict(occupancy="boxes", n_boxes=140, occ_base_res=512, L=2, L_C=512,
                     fine_table_len=1 << 22, width=3840, height=2160, n_cams=1),
}
SCENE_KEYS = {f for f, _ in SynthParams._fields_}


class SynthScene:
    """Seeded synthetic BakedScene in host memory (ngprt_synth_*): the input both
    the GPU renderer and the CPU oracle consume."""

    def __init__(self, _lib=None, **overrides):
        # _lib: a library exporting the ngprt_synth_* generator (default: the product
        # library; bench.py's reference arm passes the CPU reference checker, which
        # links the same generator, so that arm loads no product code)
        self._lib = L = _lib if _lib is not None else lib()
        _abi.bind_synth(L)
        p = SynthParams()
        L.ngprt_synth_default_params(C.byref(p))
        for k, v in overrides.items():
            if k not in SCENE_KEYS:
                continue
            if k == "occupancy":
                v = v.encode()
            if k == "fusion_tag" and isinstance(v, str):
                v = _abi.FUSION[v]
            setattr(p, k, v)
        self.params = p
        h = C.c_void_p()
        st = L.ngprt_synth_create(C.byref(p), C.byref(h))
        if st != _abi.OK:
            raise ValueError("ngprt_synth_create failed: " +
                             L.ngprt_synth_last_error().decode(errors="replace"))
        self._h = h
        self.desc_ptr = L.ngprt_synth_desc(h)
        self.desc: SceneDesc = self.desc_ptr.contents

    # numpy views over the synth-owned arrays (valid while self is alive)
    def _view(self, ptr, n, dtype):
        if n == 0:
            return np.zeros(0, dtype)
        return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))),
                                     shape=(n,))

    @property
    def L(self):
        return int(self.desc.L)

    def coarse_keys(self):
        return self._view(self.desc.coarse_keys, self.desc.n_coarse, np.uint64)

    def coarse_rows(self):
        w = 8 + 2 * self.L
        return self._view(self.desc.coarse_rows, self.desc.n_coarse * w, np.float32).reshape(-1, w)

    def fine_table(self, l):
        n = int(self.desc.fine_table_len[l]) * 8
        return self._view(self.desc.fine_tables[l], n, np.float32).reshape(-1, 8)

    def base_words(self):
        r = int(self.desc.occ_base_res)
        return self._view(self.desc.pyramid_words[0], (r ** 3 + 63) // 64, np.uint64)

    def psi(self):
        shapes = [(64, 23), (64, 64), (3, 64)]
        ws = [self._view(self.desc.psi_w[k], a * b, np.float32).reshape(a, b)
              for k, (a, b) in enumerate(shapes)]
        bs = [self._view(self.desc.psi_b[k], a, np.float32) for k, (a, _) in enumerate(shapes)]
        return ws, bs

    def occupancy_fraction(self):
        r = int(self.desc.occ_base_res)
        bits = np.unpackbits(self.base_words().view(np.uint8)).sum()
        return float(bits) / r ** 3

    def close(self):
        if getattr(self, "_h", None):
            self._lib.ngprt_synth_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def _view(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype)
    return np.ctypeslib.as_array(C.cast(ptr, C.POINTER(np.ctypeslib.as_ctypes_type(dtype))),
                                 shape=(int(n),))


class BakedFile:
    """A host BakedScene (baking.hpp:55-64): read from the reference's `.ngrt`
    file (load_baked, baking.hpp:351-485; CRC-checked sections, the file's own
    512..32 pyramid and 256^3 distance grid) or produced by bake(). Pass it to
    Scene() to upload; save() writes the `.ngrt` file (save_baked, :266-349)."""

    def __init__(self, path=None, *, _handle=None):
        if _handle is None:
            h = C.c_void_p()
            check(lib().ngprt_baked_load(str(path).encode(), C.byref(h)), "ngprt_baked_load")
            _handle = h
        self._h = _handle
        self.desc_ptr = lib().ngprt_baked_desc(self._h)
        self.desc: SceneDesc = self.desc_ptr.contents

    @property
    def L(self):
        return int(self.desc.L)

    def save(self, path) -> None:
        check(lib().ngprt_baked_save(self._h, str(path).encode()), "ngprt_baked_save")

    # numpy views over the owned arrays (valid while self is alive)
    def coarse_keys(self):
        return _view(self.desc.coarse_keys, self.desc.n_coarse, np.uint64)

    def coarse_rows(self):
        w = 8 + 2 * self.L
        return _view(self.desc.coarse_rows, self.desc.n_coarse * w, np.float32).reshape(-1, w)

    def pyramid_words(self, k):
        r = int(self.desc.occ_base_res) >> k
        return _view(self.desc.pyramid_words[k], (r ** 3 + 63) // 64, np.uint64)

    def dist_values(self):
        r = int(self.desc.dist_res)
        return _view(self.desc.dist_values, r ** 3, np.uint8)

    def close(self):
        if getattr(self, "_h", None):
            lib().ngprt_baked_free(self._h)
            self._h = None

    def __del__(self):
        self.close()


class SynthModel:
    """Seeded synthetic trained NgpRtModel (model.hpp:27-107) plus its training
    occupancy grid (ngprt_synth_model_*): the bake input. Same overrides as
    SynthScene (occupancy, occ_base_res = training resolution, L, L_C, ...)."""

    def __init__(self, **overrides):
        p = SynthParams()
        lib().ngprt_synth_default_params(C.byref(p))
        for k, v in overrides.items():
            if k not in SCENE_KEYS:
                continue
            if k == "occupancy":
                v = v.encode()
            if k == "fusion_tag" and isinstance(v, str):
                v = _abi.FUSION[v]
            setattr(p, k, v)
        self.params = p
        h = C.c_void_p()
        if lib().ngprt_synth_model_create(C.byref(p), C.byref(h)) != _abi.OK:
            raise ValueError("ngprt_synth_model_create: " +
                             lib().ngprt_synth_last_error().decode(errors="replace"))
        self._h = h
        self.desc_ptr = lib().ngprt_synth_model_desc(h)
        self.desc = self.desc_ptr.contents
        res = C.c_uint32()
        self.train_ptr = lib().ngprt_synth_model_train_words(h, C.byref(res))
        self.train_res = int(res.value)

    def train_words(self):
        return _view(self.train_ptr, (self.train_res ** 3 + 63) // 64, np.uint64)

    def close(self):
        if getattr(self, "_h", None):
            lib().ngprt_synth_model_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def bake(model, train_words=None, train_res: int | None = None, *, cull_step: float = 0.0,
         cull_alpha_thresh: float = 0.005, dilate_voxels: int = 1, device: int = 0) -> BakedFile:
    """bake(model, train_grid, BakeOptions) (baking.hpp:107-202) on the GPU.
    `model` is a SynthModel (or anything with desc_ptr / train_words()); the
    result is a host BakedFile, bit-identical to the reference's bake."""
    if train_words is None:
        train_words, train_res = model.train_words(), model.train_res
    words = np.ascontiguousarray(train_words, dtype=np.uint64)
    o = _abi.BakeOpts(cull_step, cull_alpha_thresh, dilate_voxels, 0)
    h = C.c_void_p()
    check(lib().ngprt_bake(model.desc_ptr, words.ctypes.data, int(train_res), C.byref(o), device,
                           C.byref(h)), "ngprt_bake")
    return BakedFile(_handle=h)


def cameras(n: int, width: int, height: int, radius: float = 2.9, _lib=None):
    """sphere_views(n, radius) with synth_dataset intrinsics (scene.hpp:254-265, 388-395)."""
    L = _lib if _lib is not None else lib()
    _abi.bind_synth(L)
    cams = (Camera * n)()
    if L.ngprt_synth_cameras(n, radius, width, height, cams) != _abi.OK:
        raise ValueError("ngprt_synth_cameras failed")
    return cams


def camera_array(cams):
    """ctypes Camera array from a list/sequence of Camera."""
    if isinstance(cams, C.Array):
        return cams
    arr = (Camera * len(cams))()
    for i, c in enumerate(cams):
        arr[i] = c
    return arr


@dataclass
class Opts:
    """Render options (march() arguments, occupancy.hpp:302-305; CLI flags SPEC.md:676)."""
    step: float = 0.0            # <= 0 -> kBaseStep
    use_dist_grid: bool = True
    max_step_rule: bool = False
    early_stop: bool = True
    keep_level: int = 0
    mlp: str = "tensor"          # "tensor" (tcgen05, <= 1e-3) | "exact" (bit-exact CUDA cores)
    window: tuple | None = None  # (x0, y0, w, h)
    profile: bool = False        # per-kernel CUDA-event timing (render_timing())
    # interleaved-tile sharding (ngprt_render_opts.shard_*): world 0 = off; the
    # output is then the compact (n, shard_pixels, 3) buffer of this rank's tiles
    shard_world: int = 0
    shard_rank: int = 0
    shard_tile: int = 32

    def to_c(self) -> RenderOpts:
        o = RenderOpts()
        o.profile = int(self.profile)
        o.step = self.step
        o.use_dist_grid = int(self.use_dist_grid)
        o.max_step_rule = int(self.max_step_rule)
        o.early_stop = int(self.early_stop)
        o.keep_level = int(self.keep_level)
        o.mlp_mode = _abi.MLP_EXACT if self.mlp == "exact" else _abi.MLP_TENSOR
        if self.window:
            o.x0, o.y0, o.w, o.h = self.window
        o.shard_world, o.shard_rank, o.shard_tile = self.shard_world, self.shard_rank, self.shard_tile
        return o


# ---------------------------------------------------------------------------
# Device scene and render
# ---------------------------------------------------------------------------
class Scene:
    """A BakedScene resident on one B200 (ngprt_scene). Immutable after creation."""

    def __init__(self, desc, device: int = 0, storage: int = _abi.STORAGE_AUTO):
        if hasattr(desc, "desc_ptr"):  # SynthScene / BakedFile: keep host arrays alive
            self._synth = desc
            desc_ptr = desc.desc_ptr
        else:
            desc_ptr = C.pointer(desc)
        desc_ptr.contents.storage = storage
        h = C.c_void_p()
        check(lib().ngprt_scene_create(desc_ptr, device, C.byref(h)), "ngprt_scene_create")
        self._h = h
        self.device = device
        self.L = int(desc_ptr.contents.L)

    @property
    def handle(self):
        return self._h

    def info(self) -> SceneInfo:
        i = SceneInfo()
        check(lib().ngprt_scene_info_get(self._h, C.byref(i)), "ngprt_scene_info_get")
        return i

    def close(self):
        if getattr(self, "_h", None):
            lib().ngprt_scene_destroy(self._h)
            self._h = None

    def __del__(self):
        self.close()


def _frame_hw(cams, opts: Opts):
    if opts.window:
        return opts.window[3], opts.window[2]
    return int(cams[0].height), int(cams[0].width)


def shard_pixels(width: int, height: int, world: int, tile: int = 32) -> int:
    """Pixels per camera in each rank's compact sharded output (ngprt_shard_pixels)."""
    return int(lib().ngprt_shard_pixels(width, height, world, tile))


def _out_shape(cams, opts: Opts):
    """Per-camera output shape: (h, w) for a frame / window, (P,) when sharded."""
    h, w = _frame_hw(cams, opts)
    if opts.shard_world:
        return (shard_pixels(w, h, opts.shard_world, opts.shard_tile),)
    return (h, w)


def _check_out(t, shape, dtype, dev, what):
    """The C ABI writes through raw pointers: reject anything it would overrun."""
    import torch
    numel = 1
    for d in shape:
        numel *= d
    if not isinstance(t, torch.Tensor) or t.dtype != dtype or t.device != dev or \
            not t.is_contiguous() or t.numel() < numel:
        raise ValueError(f"{what} must be a contiguous {dtype} tensor on {dev} with at least "
                         f"{numel} elements {tuple(shape)}")


def render(scene: Scene, cams, opts: Opts | None = None, out=None, stats: bool = False,
           stream=None):
    """Render len(cams) frames on the scene's GPU. Returns a torch float32 tensor
    (n, h, w, 3) [and int32 stats (n, h, w, 4)] on that device."""
    import torch

    opts = opts or Opts()
    cams = camera_array(cams)
    n = len(cams)
    shp = _out_shape(cams, opts)
    dev = torch.device("cuda", scene.device)
    if out is None:
        out = torch.empty((n, *shp, 3), dtype=torch.float32, device=dev)
    else:
        _check_out(out, (n, *shp, 3), torch.float32, dev, "out")
    st = torch.empty((n, *shp, 4), dtype=torch.int32, device=dev) if stats else None
    s = stream if stream is not None else torch.cuda.current_stream(dev)
    if s.device != dev:
        raise ValueError(f"stream is on {s.device}, the scene on {dev}")
    o = opts.to_c()
    check(lib().ngprt_render(scene.handle, cams, n, C.byref(o), out.data_ptr(),
                             st.data_ptr() if st is not None else None, s.cuda_stream),
          "ngprt_render")
    return (out, st) if stats else out


def render_timing(scene: Scene):
    """(ms in K1 march, ms in K2 shade, kernel launches) of the last profiled render."""
    a, b, n = C.c_float(), C.c_float(), C.c_int()
    check(lib().ngprt_render_timing(scene.handle, C.byref(a), C.byref(b), C.byref(n)),
          "ngprt_render_timing")
    return a.value, b.value, n.value


def render_timing3(scene: Scene):
    """(ms in K0 raygen, ms in K1 march, ms in K2 shade, kernel launches) of the last
    profiled render."""
    z, a, b, n = C.c_float(), C.c_float(), C.c_float(), C.c_int()
    check(lib().ngprt_render_timing3(scene.handle, C.byref(z), C.byref(a), C.byref(b), C.byref(n)),
          "ngprt_render_timing3")
    return z.value, a.value, b.value, n.value


def render_host(scene: Scene, cams, opts: Opts | None = None, out=None, stats=None):
    """Host-buffer render (ngprt_render_host): copies cameras in and RGB out."""
    opts = opts or Opts()
    cams = camera_array(cams)
    n = len(cams)
    shp = _out_shape(cams, opts)
    if out is None:
        out = np.empty((n, *shp, 3), np.float32)
    elif out.dtype != np.float32 or not out.flags.c_contiguous or out.size < n * 3 * int(np.prod(shp)):
        raise ValueError("out must be a C-contiguous float32 array of at least "
                         f"{(n, *shp, 3)} elements")
    if stats is not None and (not stats.flags.c_contiguous or stats.nbytes < 16 * n * int(np.prod(shp))):
        raise ValueError(f"stats must be a C-contiguous array of at least {(n, *shp, 4)} u32")
    o = opts.to_c()
    check(lib().ngprt_render_host(scene.handle, cams, n, C.byref(o), out.ctypes.data,
                                  stats.ctypes.data if stats is not None else None),
          "ngprt_render_host")
    return out


def render_host_async(scene: Scene, cams, out, opts: Opts | None = None, stats=None):
    """Enqueue a host-buffer render (ngprt_render_host_async) and return at once;
    `out` (and `stats`) must stay alive, ideally pinned, until render_host_wait."""
    opts = opts or Opts()
    cams = camera_array(cams)
    need = len(cams) * int(np.prod(_out_shape(cams, opts)))
    if out.dtype != np.float32 or not out.flags.c_contiguous or out.size < 3 * need:
        raise ValueError(f"out must be a C-contiguous float32 array of at least {3 * need} elements")
    if stats is not None and (not stats.flags.c_contiguous or stats.nbytes < 16 * need):
        raise ValueError(f"stats must be a C-contiguous array of at least {16 * need} bytes")
    o = opts.to_c()
    check(lib().ngprt_render_host_async(scene.handle, cams, len(cams), C.byref(o), out.ctypes.data,
                                        stats.ctypes.data if stats is not None else None),
          "ngprt_render_host_async")
    return out


def render_host_wait(scene: Scene) -> None:
    """Block until every enqueued host-buffer frame is in host memory."""
    check(lib().ngprt_render_host_wait(scene.handle), "ngprt_render_host_wait")


def build_pyramid(base_words, base_res: int, stream=None):
    """Levels 1..4 of build_pyramid for a device u64 word tensor (torch.int64)."""
    import torch

    levels = []
    for k in range(1, 5):
        r = base_res >> k
        levels.append(torch.empty(((r ** 3 + 63) // 64,), dtype=torch.int64,
                                  device=base_words.device))
    ptrs = (C.c_void_p * 4)(*[t.data_ptr() for t in levels])
    s = stream if stream is not None else torch.cuda.current_stream(base_words.device)
    check(lib().ngprt_build_pyramid(base_words.data_ptr(), base_res, ptrs, s.cuda_stream),
          "ngprt_build_pyramid")
    return levels


def build_distance_grid(words, res: int, stream=None):
    """build_distance_grid for a device u64 word tensor -> uint8 (res^3) tensor."""
    import torch

    out = torch.empty((res ** 3,), dtype=torch.uint8, device=words.device)
    s = stream if stream is not None else torch.cuda.current_stream(words.device)
    check(lib().ngprt_build_distance_grid(words.data_ptr(), res, out.data_ptr(), s.cuda_stream),
          "ngprt_build_distance_grid")
    return out


def shard_assemble(shards, world: int, n_cams: int, width: int, height: int, tile: int = 32,
                   channels: int = 3, out=None, stream=None):
    """De-interleave gathered compact shard outputs (world x n_cams x P x channels,
    rank-major as an all-gather lays them out) into (n_cams, h, w, channels) frames
    on the same device (ngprt_shard_assemble)."""
    import torch
    if out is None:
        out = torch.empty((n_cams, height, width, channels), dtype=shards.dtype, device=shards.device)
    P = shard_pixels(width, height, world, tile)
    _check_out(shards, (world, n_cams, P, channels), shards.dtype, shards.device, "shards")
    _check_out(out, (n_cams, height, width, channels), shards.dtype, shards.device, "out")
    if shards.element_size() != 4:
        raise ValueError("shards must have 4-byte elements (f32 RGB or u32 counters)")
    s = stream if stream is not None else torch.cuda.current_stream(shards.device)
    with torch.cuda.device(shards.device):  # the kernel launches on the current device
        check(lib().ngprt_shard_assemble(shards.data_ptr(), world, n_cams, width, height, tile,
                                         channels, out.data_ptr(), s.cuda_stream),
              "ngprt_shard_assemble")
    return out
