// render.cuh — launch-parameter types shared by the render kernels and the C ABI.
#pragma once

#include <nvtx3/nvToolsExt.h>

#include <mutex>

#include "device_common.cuh"

namespace ngprt_dev {

// One-time setup per device. Kernel attributes (dynamic shared memory limits,
// carveouts) and the SM-count-derived persistent grids are per device, and the
// ABI renders on any device from any host thread: each value is computed once
// per device under std::call_once, for the device current at the call.
constexpr int kMaxDevices = 64;
inline int current_device() {
    int d = 0;
    cudaGetDevice(&d);
    return (d >= 0 && d < kMaxDevices) ? d : 0;
}
// NVTX ranges around the C-ABI calls and their phases (header-only NVTX v3: a
// no-op unless a profiler's injection library is attached).
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
    NvtxRange(const NvtxRange&) = delete;
    NvtxRange& operator=(const NvtxRange&) = delete;
};

// The C-ABI entry points switch to their scene's device; the caller's current
// device is restored on return (a host thread may interleave calls on several
// devices, and frameworks such as torch keep their own notion of it).
struct DeviceRestore {
    int prev = -1;
    DeviceRestore() {
        if (cudaGetDevice(&prev) != cudaSuccess) {
            prev = -1;
            cudaGetLastError();
        }
    }
    ~DeviceRestore() {
        if (prev >= 0) cudaSetDevice(prev);
    }
    DeviceRestore(const DeviceRestore&) = delete;
    DeviceRestore& operator=(const DeviceRestore&) = delete;
};
struct PerDeviceInt {
    std::once_flag once[kMaxDevices];
    int value[kMaxDevices] = {};
    template <class F>
    int get(F&& init) {
        const int d = current_device();
        std::call_once(once[d], [&] { value[d] = init(d); });
        return value[d];
    }
};

// One camera, pre-flattened: c2w rows (row-major 3x4), intrinsics, image size.
struct CamParams {
    double m[12];
    double fx, fy, cx, cy;
    uint32_t width, height;
};

constexpr int kMaxCamsPerLaunch = 64;  // 64 x 136 B of kernel parameters (CUDA >= 12.1)
constexpr int kTileW = 16, kTileH = 8, kBlock = kTileW * kTileH;
// K1 ray tile: the 32 rays a warp takes at a time (kRayTileW x kRayTileH pixels)
#ifndef NGPRT_RAY_TILE_W
#define NGPRT_RAY_TILE_W 4
#endif
constexpr int kRayTileW = NGPRT_RAY_TILE_W, kRayTileH = 32 / NGPRT_RAY_TILE_W;

struct MarchParams {
    CamParams cams[kMaxCamsPerLaunch];
    int n_cams;
    uint32_t x0, y0, w, h;
    uint32_t tiles_x, tiles_per_cam;  // kRayTileW x kRayTileH ray tiles over the window
    // Interleaved-tile sharding (ngprt_render_opts.shard_*; shard_world == 0: off).
    // Output/ray index space: per camera shard_local tiles of shard_tile^2 pixels.
    uint32_t shard_world, shard_rank, shard_tile, shard_tiles_x, shard_tiles, shard_local;
    uint32_t shard_rt_x, shard_rt_per_tile;  // K1 ray tiles per shard-tile row / per shard tile
    float step;
    int use_grid, max_step_rule, early_stop, keep_level;
    int decode_min, step_burst;  // K1 warp scheduling policy (tunable, see march.cu)
    int fast_color;              // tensor-MLP mode: colour channels with FMA (see march.cu)
    RayAcc* acc;              // n_cams x h x w
    ngprt_ray_stats* stats;   // nullable, n_cams x h x w
    unsigned int* work;       // tile counter (zeroed before launch)
    const float4* rays;       // K0 -> K1: (o, t0), (d, t1) per ray; t1 < 0 = already finished
    uint32_t n_slots;         // rays / acc / stats entries of this launch (bounds checks)
};

// K1: march + gather + fuse + composite. Persistent warps, one ray per lane,
// lanes refilled from a global tile counter.
// K0 (ray generation) then K1; `between` (nullable) is recorded between the two.
void launch_march(const DevScene& sc, const MarchParams& p, cudaStream_t st,
                  cudaEvent_t between = nullptr);
int march_ctas_per_sm(const DevScene& sc);
void launch_probe_codes(const DevScene& sc, uint16_t* out, cudaStream_t st);
// K2 (exact): f32 CUDA-core deferred MLP in the reference's operation order.
void launch_shade_exact(const DevScene& sc, const RayAcc* acc, float* rgb, size_t n_rays,
                        cudaStream_t st);
// psi's biases and 64 -> 3 layer, passed to K2 as a kernel parameter. The
// 64 -> 3 weights are stored as (W2[0][i], W2[1][i]) pairs (one FFMA2 operand)
// followed by W2[2][i].
struct ShadeConsts {
    float b0[64], b1[64], w2p[64][2], w2c[64], b2[4];
};
void shade_consts_from_psi(const float* psi_host_packed, ShadeConsts* out);
// K2 (tensor): tcgen05 deferred MLP, 128 rays per CTA tile.
void launch_shade_tensor(const DevScene& sc, const void* psi_tc, const ShadeConsts& consts,
                         const RayAcc* acc, float* rgb,
                         size_t n_rays, cudaStream_t st);
// Packs psi into the tcgen05 operand layout (done once per scene).
size_t psi_tc_bytes();
void pack_psi_tc(const float* psi_host_packed, void* psi_tc_host);

// K3/K4: occupancy structures.
void launch_pyramid_level(const uint32_t* src, int src_res, uint32_t* dst, cudaStream_t st);
// tmp_a: res^3 x 2 + kDistScratchPad bytes, tmp_b: res^3 x 2 bytes.
constexpr size_t kDistScratchPad = 64;
void launch_distance_grid(const uint32_t* occ, int res, uint16_t* tmp_a, uint16_t* tmp_b,
                          uint8_t* out, cudaStream_t st);
void launch_scatter_coarse(const unsigned long long* keys, const float* rows, size_t n, int w,
                           void* dense, int f16, cudaStream_t st);
void launch_convert_fine(const float* src, void* dst, size_t n, int f16, cudaStream_t st);
void launch_coarse_cells(const void* dense_f16, int L_C, int w, void* cells, cudaStream_t st);

// test hooks
void launch_test_expf(const float* x, float* y, size_t n, cudaStream_t st);
void launch_test_expf_range(uint32_t first, size_t n, uint32_t* y, cudaStream_t st);
void launch_test_march_segments(const DevScene& sc, float step, int use_grid, int max_step_rule,
                                const float* rays8, int n, int max_seg, float* seg, int* nseg,
                                float* samples, int* nsmp, uint32_t* counters, cudaStream_t st);
void launch_test_hash(const DevScene& sc, const int32_t* corners, size_t n, int res,
                      unsigned long long len, int mode, uint32_t mask,
                      unsigned long long* out, cudaStream_t st);

}  // namespace ngprt_dev
