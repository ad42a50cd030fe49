// occupancy.cu — K3 (occupancy pyramid), K4 (distance grid) and the one-off
// scene layout kernels.
//
// K3 restates BitGrid::downsampled2 (occupancy.hpp:40-51) / build_pyramid
// (:114-119): one thread per parent voxel ORs its 8 children; a warp ballot
// assembles 32 parent bits into one little-endian u32 of the u64 word layout.
//
// K4 computes the same grid as build_distance_grid (:136-194) — exact
// Chebyshev distance, G = min(255, max(0, D-1)), all-empty -> 255 — but as a
// separable min-max transform instead of the reference's serial two-pass
// chamfer (which has a loop-carried dependency over the whole grid):
//   D(p) = min_qz max(|pz-qz|, min_qy max(|py-qy|, min_qx |px-qx|)).
// Pass X is a two-sweep 1-D distance per row; passes Y and Z search outward
// with early exit (a candidate at offset k is >= k).
#include "render.cuh"

namespace ngprt_dev {
namespace {

constexpr uint16_t kInf = 0xFFFF;

__device__ __forceinline__ bool get_bit(const uint32_t* g, int res, int x, int y, int z) {
    const size_t i = size_t(x) + size_t(res) * (size_t(y) + size_t(res) * size_t(z));
    return (g[i >> 5] >> (i & 31)) & 1u;
}

__global__ void pyramid_kernel(const uint32_t* __restrict__ src, int rs, uint32_t* __restrict__ dst,
                               int ro) {
    const size_t n = size_t(ro) * ro * ro;
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    bool v = false;
    if (i < n) {
        const int x = int(i % ro), y = int((i / ro) % ro), z = int(i / (size_t(ro) * ro));
#pragma unroll
        for (int c = 0; c < 8; ++c)
            v |= get_bit(src, rs, 2 * x + (c & 1), 2 * y + ((c >> 1) & 1), 2 * z + (c >> 2));
    }
    const unsigned m = __ballot_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && i < n) dst[i >> 5] = m;
}

// Pass X: per row (y, z), distance to the nearest occupied voxel along x.
__global__ void dt_x_kernel(const uint32_t* __restrict__ occ, int r, uint16_t* __restrict__ out) {
    const size_t row = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (row >= size_t(r) * r) return;
    const int y = int(row % r), z = int(row / r);
    uint16_t* o = out + row * r;
    uint32_t d = kInf;
    for (int x = 0; x < r; ++x) {
        d = get_bit(occ, r, x, y, z) ? 0u : (d == kInf ? kInf : d + 1);
        o[x] = uint16_t(d);
    }
    d = kInf;
    for (int x = r - 1; x >= 0; --x) {
        d = (o[x] == 0) ? 0u : (d == kInf ? kInf : d + 1);
        if (d < o[x]) o[x] = uint16_t(d);
    }
}

// Passes Y (axis 1) and Z (axis 2): out(p) = min_k max(|k|, in(p + k e_axis)).
template <int AXIS, bool FINAL>
__global__ void dt_minmax_kernel(const uint16_t* __restrict__ in, int r, uint16_t* __restrict__ out,
                                 uint8_t* __restrict__ out8) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    const size_t n = size_t(r) * r * r;
    if (i >= n) return;
    const size_t stride = AXIS == 1 ? size_t(r) : size_t(r) * r;
    const int c = AXIS == 1 ? int((i / r) % r) : int(i / (size_t(r) * r));
    uint32_t best = in[i];
    for (uint32_t k = 1; k < best && (int(k) <= c || c + int(k) < r); ++k) {
        if (int(k) <= c) {
            const uint32_t v = in[i - k * stride];
            const uint32_t cand = v > k ? v : k;
            if (cand < best) best = cand;
        }
        if (c + int(k) < r) {
            const uint32_t v = in[i + k * stride];
            const uint32_t cand = v > k ? v : k;
            if (cand < best) best = cand;
        }
    }
    if (FINAL) {
        const uint32_t g = best == 0 ? 0u : best - 1u;  // occupancy.hpp:188-192
        out8[i] = uint8_t(g < 255u ? g : 255u);
    } else {
        out[i] = uint16_t(best);
    }
}

template <bool F16>
__global__ void scatter_coarse_kernel(const unsigned long long* __restrict__ keys,
                                      const float* __restrict__ rows, size_t n, int w,
                                      void* __restrict__ dense) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const unsigned long long key = keys[i];
    for (int c = 0; c < w; ++c) {
        const float v = rows[i * w + c];
        if (F16)
            reinterpret_cast<__half*>(dense)[key * 16 + c] = __float2half_rn(v);
        else
            reinterpret_cast<float*>(dense)[key * 16 + c] = v;
    }
}

__global__ void convert_f16_kernel(const float* __restrict__ src, __half* __restrict__ dst,
                                   size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        dst[i] = __float2half_rn(src[i]);
}

unsigned blocks_for(size_t n, unsigned bs) { return unsigned((n + bs - 1) / bs); }

}  // namespace

void launch_pyramid_level(const uint32_t* src, int src_res, uint32_t* dst, cudaStream_t st) {
    const int ro = src_res / 2;
    const size_t n = size_t(ro) * ro * ro;
    pyramid_kernel<<<blocks_for(n, 256), 256, 0, st>>>(src, src_res, dst, ro);
}

void launch_distance_grid(const uint32_t* occ, int r, uint16_t* a, uint16_t* b, uint8_t* out,
                          cudaStream_t st) {
    const size_t rows = size_t(r) * r, n = rows * r;
    dt_x_kernel<<<blocks_for(rows, 128), 128, 0, st>>>(occ, r, a);
    dt_minmax_kernel<1, false><<<blocks_for(n, 256), 256, 0, st>>>(a, r, b, nullptr);
    dt_minmax_kernel<2, true><<<blocks_for(n, 256), 256, 0, st>>>(b, r, nullptr, out);
}

void launch_scatter_coarse(const unsigned long long* keys, const float* rows, size_t n, int w,
                           void* dense, int f16, cudaStream_t st) {
    if (!n) return;
    if (f16)
        scatter_coarse_kernel<true><<<blocks_for(n, 256), 256, 0, st>>>(keys, rows, n, w, dense);
    else
        scatter_coarse_kernel<false><<<blocks_for(n, 256), 256, 0, st>>>(keys, rows, n, w, dense);
}

void launch_convert_fine(const float* src, void* dst, size_t n, int f16, cudaStream_t st) {
    if (f16)
        convert_f16_kernel<<<148 * 8, 256, 0, st>>>(src, reinterpret_cast<__half*>(dst), n);
    else
        cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
}

}  // namespace ngprt_dev
