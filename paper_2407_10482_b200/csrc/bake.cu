// bake.cu — the bake (baking.hpp:107-202) on the GPU: a trained NgpRtModel plus
// its training occupancy -> the render-time BakedScene.
//
//   (1) density cull (:118-134): every occupied training voxel's centre goes
//       through the live decode (decode_point, model.hpp:195-239: 8 corner
//       evaluations, interpolation, attention, fine levels, fuse) and is kept
//       iff 1 - exp(-sigma * cull_step) > cull_alpha_thresh; then dilation
//       (BitGrid::dilated, occupancy.hpp:54-71);
//   (2) the 512 render grid (BitGrid::upsampled, :74-87), its pyramid and the
//       256^3 distance grid (K3/K4, bit-exact with build_pyramid /
//       build_distance_grid);
//   (3) corner retention on the L_C grid (:146-163) and corner evaluation
//       (evaluate_corner, model.hpp:71-87: six coarse hash levels -> 24
//       features -> aux MLP 24 -> 64 -> 8+2L), one thread per retained corner;
//   (4) fine tables, psi and the fusion parameters carried over verbatim.
// Built with -fmad=false: every f32 expression rounds where the reference's
// does, so keys, rows, pyramid and distance grid are bit-identical to the
// reference's bake. The one double-precision transcendental (the cull's
// std::exp, glibc) is evaluated with CUDA's exp; decisions within 1e-12 of the
// threshold are re-evaluated on the host with glibc, so the cull is exact too.
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cmath>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include <cub/device/device_scan.cuh>

#include <mutex>
#include <thread>

#include "baked.hpp"
#include "render.cuh"

namespace ngprt_dev {
namespace {

constexpr int kCoarseLevels = 6;
constexpr int kHiddenUnroll = 64;
#ifndef NGPRT_CORNER_MINB
#define NGPRT_CORNER_MINB 10
#endif

struct DevModel {
    int L, L_C, W;  // W = 8 + 2L
    float lc_h;     // float(L_C) / 2
    int cres[kCoarseLevels];
    float ch[kCoarseLevels];
    int cdirect[kCoarseLevels];
    unsigned long long clen[kCoarseLevels];
    unsigned long long cmask[kCoarseLevels];  // len - 1 for a power-of-two hashed length, else 0
    const float* ctab[kCoarseLevels];
    int fine_res[NGPRT_MAX_FINE_LEVELS];
    float fine_h[NGPRT_MAX_FINE_LEVELS];
    int fine_hashed[NGPRT_MAX_FINE_LEVELS];
    unsigned long long fine_len[NGPRT_MAX_FINE_LEVELS];
    unsigned long long fine_mask[NGPRT_MAX_FINE_LEVELS];
    const float* fine[NGPRT_MAX_FINE_LEVELS];
    int fusion;
    float att_w[2 * NGPRT_MAX_FINE_LEVELS];
    const float* fmlp;  // W0 (64x8L) b0 (64) W1 (8x64) b1 (8)
};

// stencil along one axis (hash_grid.hpp:38-46) with h = float(res)/2.0f
__device__ __forceinline__ void stencil_axis(float x, float h, int res, int& base, float& frac) {
    const float u = (x - (-1.0f)) * h;
    int i = int(floorf(u));
    i = i < res - 1 ? i : res - 1;
    i = i > 0 ? i : 0;
    base = i;
    frac = u - float(i);
}

// HashLevel::hash_index, hash_grid.hpp:83-94 (h % len == h & (len-1) for a power of two)
__device__ __forceinline__ unsigned long long hash_index(int res, unsigned long long len,
                                                         unsigned long long mask, int hashed,
                                                         int x, int y, int z) {
    if (!hashed) {
        const unsigned long long r1 = (unsigned long long)res + 1;
        return (unsigned long long)x + r1 * ((unsigned long long)y + r1 * (unsigned long long)z);
    }
    const unsigned long long h = (unsigned long long)x * 1ull ^
                                 (unsigned long long)y * 2654435761ull ^
                                 (unsigned long long)z * 805459861ull;
    return mask ? (h & mask) : h % len;
}

// HashLevel::interp (hash_grid.hpp:97-104) of a D-wide table at x.
template <int D>
__device__ __forceinline__ void interp(const float* __restrict__ tab, int res, float h,
                                       unsigned long long len, unsigned long long mask, int hashed,
                                       const float x[3], float* out) {
    int b[3];
    float f[3];
    for (int a = 0; a < 3; ++a) stencil_axis(x[a], h, res, b[a], f[a]);
    for (int c = 0; c < D; ++c) out[c] = 0.0f;
    for (int k = 0; k < 8; ++k) {
        const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
        const float w = ((dx ? f[0] : 1.0f - f[0]) * (dy ? f[1] : 1.0f - f[1])) *
                        (dz ? f[2] : 1.0f - f[2]);
        const float4* row = reinterpret_cast<const float4*>(
            tab + hash_index(res, len, mask, hashed, b[0] + dx, b[1] + dy, b[2] + dz) * D);
#pragma unroll
        for (int q = 0; q < D / 4; ++q) {  // rows are 16-byte aligned (D = 4 or 8)
            const float4 v = __ldg(row + q);
            out[4 * q + 0] += w * v.x;
            out[4 * q + 1] += w * v.y;
            out[4 * q + 2] += w * v.z;
            out[4 * q + 3] += w * v.w;
        }
    }
}

// The aux decoder's weights as a kernel parameter (10.5 KB, constant bank 0):
// with the loops below fully unrolled every weight is an FMUL operand read
// from the constant bank, no load instruction per multiply-add.
struct AuxWeights {
    float w0[64 * 24];
    float b0[64];
    float w1[16 * 64];
    float b1[16];
};

// NgpRtModel::evaluate_corner (model.hpp:71-87): encode_coarse at the corner
// position (corner_to_world, hash_grid.hpp:28-31) through the aux MLP.
template <int W>
__device__ __forceinline__ void evaluate_corner(const DevModel& M, const AuxWeights& A, int cx,
                                                int cy, int cz, float* out) {
    const float pos[3] = {-1.0f + 2.0f * (float(cx) / float(M.L_C)),
                          -1.0f + 2.0f * (float(cy) / float(M.L_C)),
                          -1.0f + 2.0f * (float(cz) / float(M.L_C))};
    float feat[24];
#pragma unroll
    for (int k = 0; k < kCoarseLevels; ++k)
        interp<4>(M.ctab[k], M.cres[k], M.ch[k], M.clen[k], M.cmask[k], !M.cdirect[k], pos,
                  feat + 4 * k);
    // TinyMlp::forward (nn.hpp:175-196), hidden unit by unit; the output layer
    // accumulates in the same c-order as the reference's inner loop.
#pragma unroll
    for (int j = 0; j < W; ++j) out[j] = A.b1[j];
    // r unrolled by kHiddenUnroll only: a full unroll (~8 k instructions)
    // overflows the instruction cache (ncu: "no instructions" top stall).
#pragma unroll kHiddenUnroll
    for (int r = 0; r < 64; ++r) {
        float h = A.b0[r];
#pragma unroll
        for (int c = 0; c < 24; ++c) h += A.w0[r * 24 + c] * feat[c];
        h = h < 0.0f ? 0.0f : h;
#pragma unroll
        for (int j = 0; j < W; ++j) out[j] += A.w1[j * 64 + r] * h;
    }
}

// Corner rows evaluated once per distinct corner (the reference's CornerCache,
// model.hpp:113-150): a bitmap of the corners present, the exclusive prefix
// count of each 32-bit word and the rows in key order; rank lookup = 2 loads.
struct CornerTable {
    const uint32_t* marks;
    const uint32_t* offsets;
    const float* rows;
    unsigned long long r1;
    int W;
};

__device__ __forceinline__ const float* corner_row(const CornerTable& T, int x, int y, int z) {
    const unsigned long long key =
        (unsigned long long)x + T.r1 * ((unsigned long long)y + T.r1 * (unsigned long long)z);
    const uint32_t w = __ldg(T.marks + (key >> 5));
    const uint32_t rank = __ldg(T.offsets + (key >> 5)) + __popc(w & ((1u << (key & 31)) - 1u));
    return T.rows + size_t(rank) * T.W;
}

// sigma_pre of decode_point (model.hpp:195-239) at x: only channel 0 of the fuse.
__device__ float decode_sigma_pre(const DevModel& M, const CornerTable& T, const float x[3],
                                  const unsigned long long* tab) {
    int cb[3];
    float cf[3];
    for (int a = 0; a < 3; ++a) stencil_axis(x[a], M.lc_h, M.L_C, cb[a], cf[a]);
    float dec[16];
    for (int i = 0; i < M.W; ++i) dec[i] = 0.0f;
    for (int k = 0; k < 8; ++k) {
        const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
        const float w = ((dx ? cf[0] : 1.0f - cf[0]) * (dy ? cf[1] : 1.0f - cf[1])) *
                        (dz ? cf[2] : 1.0f - cf[2]);
        const float* row = corner_row(T, cb[0] + dx, cb[1] + dy, cb[2] + dz);
        for (int i = 0; i < M.W; ++i) dec[i] += w * __ldg(row + i);
    }
    float fine[NGPRT_MAX_FINE_LEVELS][8];
    for (int l = 0; l < M.L; ++l)
        interp<8>(M.fine[l], M.fine_res[l], M.fine_h[l], M.fine_len[l], M.fine_mask[l],
                  M.fine_hashed[l], x, fine[l]);
    float out0 = dec[0];
    if (M.fusion == NGPRT_FUSION_MLP) {  // fusion.hpp:162-171, channel 0 of the output
        const int IN = 8 * M.L;
        const float* W0 = M.fmlp;
        const float* B0 = W0 + 64 * IN;
        const float* W1 = B0 + 64;
        const float* B1 = W1 + 8 * 64;
        float hat0 = __ldg(B1);
        for (int r = 0; r < 64; ++r) {
            float h = __ldg(B0 + r);
            for (int c = 0; c < IN; ++c) h += __ldg(W0 + r * IN + c) * fine[c / 8][c % 8];
            h = h < 0.0f ? 0.0f : h;
            hat0 += __ldg(W1 + r) * h;
        }
        return out0 + hat0;
    }
    for (int l = 0; l < M.L; ++l) {
        float wo;
        if (M.fusion == NGPRT_FUSION_SEPARATE_ATT_V || M.fusion == NGPRT_FUSION_SHARED_ATT_V)
            wo = activate_sigmoid(dec[8 + 2 * l], tab);  // split_decoder_output, model.hpp:19
        else if (M.fusion == NGPRT_FUSION_SUM)
            wo = 1.0f;
        else
            wo = M.att_w[2 * l];
        out0 += wo * fine[l][0];
    }
    return out0;
}

__device__ __forceinline__ bool bit_at(const uint32_t* g, int res, int x, int y, int z) {
    const size_t i = size_t(x) + size_t(res) * (size_t(y) + size_t(res) * size_t(z));
    return (g[i >> 5] >> (i & 31)) & 1u;
}

// Training-voxel centre (baking.hpp:128-129).
__device__ __forceinline__ void voxel_centre(size_t i, int tres, float c[3]) {
    const int x = int(i % tres), y = int((i / tres) % tres), z = int(i / (size_t(tres) * tres));
    const double vsz = 2.0 / tres;  // Roi::extent / tres
    c[0] = float(-1.0 + (x + 0.5) * vsz);
    c[1] = float(-1.0 + (y + 0.5) * vsz);
    c[2] = float(-1.0 + (z + 0.5) * vsz);
}

// The L_C corners the cull's decodes read: the stencil corners of every
// occupied training-voxel centre.
__global__ void cull_marks_kernel(const DevModel M, const uint32_t* __restrict__ train, int tres,
                                  uint32_t* marks) {
    const size_t n = size_t(tres) * tres * tres;
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n || !((train[i >> 5] >> (i & 31)) & 1u)) return;
    float c[3], f;
    int b[3];
    voxel_centre(i, tres, c);
    for (int a = 0; a < 3; ++a) stencil_axis(c[a], M.lc_h, M.L_C, b[a], f);
    const size_t r1 = size_t(M.L_C) + 1;
    for (int k = 0; k < 8; ++k) {
        const size_t key = size_t(b[0] + (k & 1)) + r1 * (size_t(b[1] + ((k >> 1) & 1)) + r1 * size_t(b[2] + (k >> 2)));
        atomicOr(marks + (key >> 5), 1u << (key & 31));
    }
}

// (1) density cull: one thread per training voxel; 32 voxels -> one ballot word.
__global__ void cull_kernel(const DevModel M, const CornerTable T, const uint32_t* __restrict__ train,
                            int tres, double cull_step, double thresh, uint32_t* __restrict__ culled,
                            unsigned int* amb_n, uint32_t* amb_idx, float* amb_sigma, int amb_cap) {
    __shared__ unsigned long long tab[32];
    load_exp_table(tab);
    __syncthreads();
    const size_t n = size_t(tres) * tres * tres;
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    bool keep = false;
    if (i < n && ((train[i >> 5] >> (i & 31)) & 1u)) {
        float c[3];
        voxel_centre(i, tres, c);
        const float sigma = activate_density(decode_sigma_pre(M, T, c, tab), tab);
        const double e = exp(-double(sigma) * cull_step);
        keep = 1.0 - e > thresh;
        if (fabs(e - (1.0 - thresh)) < 1e-12) {  // glibc exp may decide differently: host re-check
            const unsigned int k = atomicAdd(amb_n, 1u);
            if (int(k) < amb_cap) {
                amb_idx[k] = uint32_t(i);
                amb_sigma[k] = sigma;
            }
        }
    }
    const unsigned m = __ballot_sync(0xffffffffu, keep);
    if ((threadIdx.x & 31) == 0 && i < n) culled[i >> 5] = m;
}

// BitGrid::dilated (occupancy.hpp:54-71): 3^3 OR, clipped at the faces.
__global__ void dilate_kernel(const uint32_t* __restrict__ src, int r, uint32_t* __restrict__ dst) {
    const size_t n = size_t(r) * r * r;
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    bool v = false;
    if (i < n) {
        const int x = int(i % r), y = int((i / r) % r), z = int(i / (size_t(r) * r));
        for (int dz = -1; dz <= 1 && !v; ++dz)
            for (int dy = -1; dy <= 1 && !v; ++dy)
                for (int dx = -1; dx <= 1 && !v; ++dx) {
                    const int nx = x + dx, ny = y + dy, nz = z + dz;
                    if (nx < 0 || ny < 0 || nz < 0 || nx >= r || ny >= r || nz >= r) continue;
                    v = bit_at(src, r, nx, ny, nz);
                }
    }
    const unsigned m = __ballot_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && i < n) dst[i >> 5] = m;
}

// BitGrid::upsampled (occupancy.hpp:74-87): bit replication by `f`.
__global__ void upsample_kernel(const uint32_t* __restrict__ src, int r, int f,
                                uint32_t* __restrict__ dst) {
    const int ro = r * f;
    const size_t n = size_t(ro) * ro * ro;
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    bool v = false;
    if (i < n) {
        const int x = int(i % ro), y = int((i / ro) % ro), z = int(i / (size_t(ro) * ro));
        v = bit_at(src, r, x / f, y / f, z / f);
    }
    const unsigned m = __ballot_sync(0xffffffffu, v);
    if ((threadIdx.x & 31) == 0 && i < n) dst[i >> 5] = m;
}

// corner_marks (baking.hpp:156-163): the 8 corners of every occupied L_C voxel.
__global__ void corner_marks_kernel(const uint32_t* __restrict__ occ, int lc, uint32_t* marks) {
    const size_t n = size_t(lc) * lc * lc;
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n || !((occ[i >> 5] >> (i & 31)) & 1u)) return;
    const int x = int(i % lc), y = int((i / lc) % lc), z = int(i / (size_t(lc) * lc));
    const size_t r1 = size_t(lc) + 1;
    for (int k = 0; k < 8; ++k) {
        const size_t b = size_t(x + (k & 1)) + r1 * (size_t(y + ((k >> 1) & 1)) + r1 * size_t(z + (k >> 2)));
        atomicOr(marks + (b >> 5), 1u << (b & 31));
    }
}

// (3) evaluate_corner for every corner key.
template <int W>
__global__ void __launch_bounds__(128, NGPRT_CORNER_MINB) corner_eval_kernel(const DevModel M,
                                                          const __grid_constant__ AuxWeights A,
                                                          const unsigned long long* __restrict__ keys,
                                                          size_t n, float* __restrict__ rows) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const unsigned long long r1 = (unsigned long long)M.L_C + 1, key = keys[i];
    float row[W];
    evaluate_corner<W>(M, A, int(key % r1), int((key / r1) % r1), int(key / (r1 * r1)), row);
#pragma unroll
    for (int j = 0; j < W; ++j) rows[i * W + j] = row[j];
}

void launch_corner_eval(const DevModel& M, const AuxWeights& A, const unsigned long long* keys,
                        size_t n, float* rows) {
    if (!n) return;
    const unsigned g = unsigned((n + 127) / 128);
    switch (M.W) {
        case 10: corner_eval_kernel<10><<<g, 128>>>(M, A, keys, n, rows); break;
        case 12: corner_eval_kernel<12><<<g, 128>>>(M, A, keys, n, rows); break;
        case 14: corner_eval_kernel<14><<<g, 128>>>(M, A, keys, n, rows); break;
        default: corner_eval_kernel<16><<<g, 128>>>(M, A, keys, n, rows); break;
    }
}

// Retained corner keys in ascending order (== the reference's z,y,x scan,
// baking.hpp:167-175): per-word popcount -> exclusive scan -> scatter.
__global__ void popcount_kernel(const uint32_t* __restrict__ marks, size_t nw, uint32_t* counts) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i < nw) counts[i] = __popc(marks[i]);
    else if (i == nw) counts[i] = 0;
}

__global__ void scatter_keys_kernel(const uint32_t* __restrict__ marks, size_t nw,
                                    const uint32_t* __restrict__ offsets,
                                    unsigned long long* __restrict__ keys) {
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= nw) return;
    uint32_t o = offsets[i];
    for (uint32_t m = marks[i]; m; m &= m - 1) keys[o++] = (i << 5) + unsigned(__ffs(m) - 1);
}

unsigned blocks(size_t n, unsigned bs) { return unsigned((n + bs - 1) / bs); }
size_t words32(size_t res) { return ((res * res * res + 63) / 64) * 2; }

}  // namespace
}  // namespace ngprt_dev

using namespace ngprt_dev;

namespace {

// NGPRT_BAKE_PROFILE=1: per-phase wall times (device synchronised) on stderr.
struct PhaseTimer {
    bool on = std::getenv("NGPRT_BAKE_PROFILE") != nullptr;
    std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
    void mark(const char* name) {
        if (!on) return;
        cudaDeviceSynchronize();
        const auto now = std::chrono::steady_clock::now();
        std::fprintf(stderr, "[bake] %-14s %9.3f ms\n", name,
                     std::chrono::duration<double, std::milli>(now - t).count());
        t = now;
    }
};

// Host <-> device copies of the large arrays (corner rows can be GBs; fine
// tables and coarse tables are 100s of MB) through two pinned staging chunks
// on a blocking stream (ordered with the legacy-stream kernels): the DMA of one
// chunk overlaps a multi-threaded memcpy of the other, so pageable memory
// moves at several times the speed of a plain cudaMemcpy from/to it.
constexpr size_t kChunk = size_t(32) << 20;
constexpr int kMaxThreads = 16;

int copy_threads() {
    static const int t = [] {
        const char* e = std::getenv("NGPRT_COPY_THREADS");
        const int v = e ? std::atoi(e) : 8;
        return v < 1 ? 1 : (v > kMaxThreads ? kMaxThreads : v);
    }();
    return t;
}

void parallel_memcpy(void* dst, const void* src, size_t bytes) {
    const int nt = bytes < (size_t(4) << 20) ? 1 : copy_threads();
    const size_t part = (bytes / nt + 63) & ~size_t(63);
    std::thread th[kMaxThreads - 1];
    auto piece = [=](int t) {
        const size_t a = std::min(bytes, t * part), b = std::min(bytes, (t + 1) * part);
        if (b > a) std::memcpy(static_cast<char*>(dst) + a, static_cast<const char*>(src) + a, b - a);
    };
    for (int t = 1; t < nt; ++t) th[t - 1] = std::thread(piece, t);
    piece(0);
    for (int t = 1; t < nt; ++t) th[t - 1].join();
}

struct Staging {
    std::mutex mu;
    void* buf[2] = {nullptr, nullptr};
    cudaStream_t st = nullptr;
    cudaEvent_t ev[2];
    void init() {
        if (st) return;
        cudaStreamCreate(&st);
        for (int i = 0; i < 2; ++i) {
            cudaMallocHost(&buf[i], kChunk);
            cudaEventCreateWithFlags(&ev[i], cudaEventDisableTiming);
        }
    }
};

// one staging pair per device (its stream and pinned chunks belong to that device)
Staging& staging() {
    static Staging s[kMaxDevices];
    return s[current_device()];
}

void d2h(void* dst, const void* src, size_t bytes) {
    if (bytes < 4 * kChunk) {
        cudaMemcpy(dst, src, bytes, cudaMemcpyDeviceToHost);
        return;
    }
    Staging& S = staging();
    std::lock_guard<std::mutex> lock(S.mu);
    S.init();
    const size_t n = (bytes + kChunk - 1) / kChunk;
    auto len = [&](size_t i) { return std::min(kChunk, bytes - i * kChunk); };
    auto issue = [&](size_t i) {
        cudaMemcpyAsync(S.buf[i & 1], static_cast<const char*>(src) + i * kChunk, len(i),
                        cudaMemcpyDeviceToHost, S.st);
        cudaEventRecord(S.ev[i & 1], S.st);
    };
    issue(0);
    for (size_t i = 0; i < n; ++i) {
        if (i + 1 < n) issue(i + 1);
        cudaEventSynchronize(S.ev[i & 1]);
        parallel_memcpy(static_cast<char*>(dst) + i * kChunk, S.buf[i & 1], len(i));
    }
}

void h2d(void* dst, const void* src, size_t bytes) {
    if (bytes < 4 * kChunk) {
        cudaMemcpy(dst, src, bytes, cudaMemcpyHostToDevice);
        return;
    }
    Staging& S = staging();
    std::lock_guard<std::mutex> lock(S.mu);
    S.init();
    const size_t n = (bytes + kChunk - 1) / kChunk;
    for (size_t i = 0; i < n; ++i) {
        const size_t len = std::min(kChunk, bytes - i * kChunk);
        if (i >= 2) cudaEventSynchronize(S.ev[i & 1]);  // chunk i-2's DMA has drained this buffer
        parallel_memcpy(S.buf[i & 1], static_cast<const char*>(src) + i * kChunk, len);
        cudaMemcpyAsync(static_cast<char*>(dst) + i * kChunk, S.buf[i & 1], len,
                        cudaMemcpyHostToDevice, S.st);
        cudaEventRecord(S.ev[i & 1], S.st);
    }
    cudaStreamSynchronize(S.st);
}

// Stream-ordered scratch from the device's default pool (kept mapped between
// bakes: the release threshold is raised as for the renderer's scratch), all
// freed on scope exit.
struct DeviceBuffers {
    std::vector<void*> ptrs;
    DeviceBuffers(int device) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, device) == cudaSuccess) {
            uint64_t thr = ~uint64_t(0);
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
        }
    }
    ~DeviceBuffers() {
        for (void* p : ptrs) cudaFreeAsync(p, 0);
        cudaStreamSynchronize(0);
    }
    template <class T>
    T* alloc(size_t count) {
        void* p = nullptr;
        const cudaError_t e = cudaMallocAsync(&p, count * sizeof(T) + 16, 0);
        if (e != cudaSuccess) throw std::runtime_error(std::string("bake: cudaMallocAsync: ") + cudaGetErrorString(e));
        cudaMemsetAsync(p, 0, count * sizeof(T) + 16, 0);
        ptrs.push_back(p);
        return static_cast<T*>(p);
    }
    template <class T>
    T* upload(const T* h, size_t count) {
        T* d = alloc<T>(count);
        h2d(d, h, count * sizeof(T));
        return d;
    }
};

void check_cuda(const char* what) {
    const cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) throw std::runtime_error(std::string(what) + ": " + cudaGetErrorString(e));
}

void check_finite(const float* p, size_t n, const std::string& group) {
    const int nt = n < (size_t(1) << 20) ? 1 : copy_threads();
    const size_t part = (n + nt - 1) / nt;
    bool bad[kMaxThreads] = {};
    std::thread th[kMaxThreads - 1];
    auto piece = [&](int t) {
        const size_t a = std::min(n, t * part), b = std::min(n, (t + 1) * part);
        uint32_t acc = 0;  // exponent all-ones <=> inf/nan
        for (size_t i = a; i < b; ++i) {
            uint32_t u;
            std::memcpy(&u, p + i, 4);
            acc |= uint32_t((u & 0x7f800000u) == 0x7f800000u);
        }
        bad[t] = acc != 0;
    };
    for (int t = 1; t < nt; ++t) th[t - 1] = std::thread(piece, t);
    piece(0);
    for (int t = 1; t < nt; ++t) th[t - 1].join();
    for (int t = 0; t < nt; ++t)
        if (bad[t]) throw std::runtime_error("bake: non-finite parameter in group " + group);
}

}  // namespace

extern "C" ngprt_status ngprt_bake(const ngprt_model_desc* md, const uint64_t* train_words,
                                   uint32_t tres, const ngprt_bake_opts* opts, int device,
                                   ngprt_baked** out) {
    if (!md || !train_words || !out) {
        ngprt_host::set_error("ngprt_bake: null argument");
        return NGPRT_EINVAL;
    }
    *out = nullptr;
    try {
        const int L = int(md->L), lc = int(md->L_C), W = 8 + 2 * L;
        if (L < 1 || L > NGPRT_MAX_FINE_LEVELS) throw std::invalid_argument("bake: L out of range");
        if (md->fusion_tag > NGPRT_FUSION_MLP) throw std::invalid_argument("bake: unknown fusion tag");
        const int render_res = 512;
        if (tres == 0 || render_res % int(tres) != 0)
            throw std::invalid_argument("bake: training grid must divide the 512 render grid");
        if (lc % int(tres) != 0 && int(tres) % lc != 0)
            throw std::invalid_argument("bake: L_C and the training grid must nest");
        const double cull_step = (opts && opts->cull_step > 0) ? opts->cull_step : 2.0 * std::sqrt(3.0) / 512.0;
        const double thresh = opts ? opts->cull_alpha_thresh : 0.005;
        const int dilate = opts ? int(opts->dilate_voxels) : 1;

        // parameter checks (baking.hpp:109-112), in GradTape group order
        // (coarse, fine, aux, psi, fusion: model.hpp:44-51)
        for (int k = 0; k < 6; ++k) {
            const uint64_t res = md->coarse_res[k], corners = (res + 1) * (res + 1) * (res + 1);
            check_finite(md->coarse_tables[k], std::min<uint64_t>(corners, md->coarse_table_len) * 4,
                         "coarse_l" + std::to_string(k));
        }
        for (int l = 0; l < L; ++l)
            check_finite(md->fine_tables[l], md->fine_table_len[l] * 8, "fine_l" + std::to_string(l + 1));
        const int aux_w[3] = {24, 64, W}, psi_w[4] = {23, 64, 64, 3}, fm_w[3] = {8 * L, 64, 8};
        for (int k = 0; k < 2; ++k) {
            check_finite(md->aux_w[k], size_t(aux_w[k]) * aux_w[k + 1], "aux.w" + std::to_string(k));
            check_finite(md->aux_b[k], aux_w[k + 1], "aux.b" + std::to_string(k));
        }
        for (int k = 0; k < 3; ++k) {
            check_finite(md->psi_w[k], size_t(psi_w[k]) * psi_w[k + 1], "psi.w" + std::to_string(k));
            check_finite(md->psi_b[k], psi_w[k + 1], "psi.b" + std::to_string(k));
        }
        const bool inv_tag = md->fusion_tag == NGPRT_FUSION_SHARED_ATT_INV ||
                             md->fusion_tag == NGPRT_FUSION_SEPARATE_ATT_INV;
        if (inv_tag) check_finite(md->att_globals, size_t(2) * L, "att_global");
        if (md->fusion_tag == NGPRT_FUSION_MLP)
            for (int k = 0; k < 2; ++k) {
                check_finite(md->fusion_mlp_w[k], size_t(fm_w[k]) * fm_w[k + 1], "fusion_mlp.w" + std::to_string(k));
                check_finite(md->fusion_mlp_b[k], fm_w[k + 1], "fusion_mlp.b" + std::to_string(k));
            }

        // the model on the device
        PhaseTimer pt;
        if (cudaSetDevice(device) != cudaSuccess) throw std::runtime_error("bake: no CUDA device");
        DeviceBuffers db(device);
        DevModel M{};
        M.L = L;
        M.L_C = lc;
        M.W = W;
        M.lc_h = float(lc) / 2.0f;
        for (int k = 0; k < 6; ++k) {
            const uint64_t res = md->coarse_res[k], corners = (res + 1) * (res + 1) * (res + 1);
            const uint64_t len = corners <= md->coarse_table_len ? corners : md->coarse_table_len;
            M.cres[k] = int(res);
            M.ch[k] = float(res) / 2.0f;
            M.cdirect[k] = corners <= md->coarse_table_len;
            M.clen[k] = len;
            M.cmask[k] = (!M.cdirect[k] && (len & (len - 1)) == 0) ? len - 1 : 0;
            M.ctab[k] = db.upload(md->coarse_tables[k], len * 4);
        }
        auto A = std::make_unique<AuxWeights>();
        std::memset(A.get(), 0, sizeof(AuxWeights));
        std::memcpy(A->w0, md->aux_w[0], 64 * 24 * 4);
        std::memcpy(A->b0, md->aux_b[0], 64 * 4);
        std::memcpy(A->w1, md->aux_w[1], size_t(W) * 64 * 4);
        std::memcpy(A->b1, md->aux_b[1], size_t(W) * 4);
        for (int l = 0; l < L; ++l) {
            M.fine_res[l] = int(md->fine_res[l]);
            M.fine_h[l] = float(md->fine_res[l]) / 2.0f;
            M.fine_hashed[l] = md->fine_hashed[l];
            M.fine_len[l] = md->fine_table_len[l];
            M.fine_mask[l] = (M.fine_hashed[l] && (M.fine_len[l] & (M.fine_len[l] - 1)) == 0) ? M.fine_len[l] - 1 : 0;
            M.fine[l] = db.upload(md->fine_tables[l], md->fine_table_len[l] * 8);
        }
        M.fusion = md->fusion_tag;
        const bool inv = M.fusion == NGPRT_FUSION_SHARED_ATT_INV || M.fusion == NGPRT_FUSION_SEPARATE_ATT_INV;
        if (inv)
            for (int i = 0; i < 2 * L; ++i) M.att_w[i] = 1.0f / (1.0f + std::exp(-md->att_globals[i]));
        if (M.fusion == NGPRT_FUSION_MLP) {
            const size_t in = size_t(8) * L;
            std::vector<float> f(64 * in + 64 + 8 * 64 + 8);
            std::memcpy(f.data(), md->fusion_mlp_w[0], 64 * in * 4);
            std::memcpy(f.data() + 64 * in, md->fusion_mlp_b[0], 64 * 4);
            std::memcpy(f.data() + 64 * in + 64, md->fusion_mlp_w[1], 8 * 64 * 4);
            std::memcpy(f.data() + 64 * in + 64 + 512, md->fusion_mlp_b[1], 8 * 4);
            M.fmlp = db.upload(f.data(), f.size());
        }

        pt.mark("upload");
        // marks bitmap -> ascending keys + per-word exclusive counts (rank table)
        auto compact = [&](const uint32_t* marks, size_t nw, uint32_t** offsets_out,
                           unsigned long long** keys_out) -> uint32_t {
            uint32_t* counts = db.alloc<uint32_t>(nw + 1);
            uint32_t* offsets = db.alloc<uint32_t>(nw + 1);
            popcount_kernel<<<blocks(nw + 1, 256), 256>>>(marks, nw, counts);
            size_t scan_bytes = 0;
            cub::DeviceScan::ExclusiveSum(nullptr, scan_bytes, counts, offsets, nw + 1);
            void* scan_tmp = db.alloc<uint8_t>(scan_bytes);
            cub::DeviceScan::ExclusiveSum(scan_tmp, scan_bytes, counts, offsets, nw + 1);
            uint32_t n = 0;
            cudaMemcpy(&n, offsets + nw, 4, cudaMemcpyDeviceToHost);
            check_cuda("bake: corner keys");
            unsigned long long* keys = db.alloc<unsigned long long>(n ? n : 1);
            if (n) scatter_keys_kernel<<<blocks(nw, 256), 256>>>(marks, nw, offsets, keys);
            *offsets_out = offsets;
            *keys_out = keys;
            return n;
        };
        const size_t r1 = size_t(lc) + 1;
        const size_t nw = words32(r1);

        // (1) density cull at the training resolution, exact decisions
        const size_t tn = size_t(tres) * tres * tres;
        CornerTable cull_table{};
        uint32_t* train = db.upload(reinterpret_cast<const uint32_t*>(train_words), words32(tres));
        uint32_t* culled = db.alloc<uint32_t>(words32(tres));
        unsigned int* amb_n = db.alloc<unsigned int>(1);
        const int amb_cap = 1 << 16;
        uint32_t* amb_idx = db.alloc<uint32_t>(amb_cap);
        float* amb_sigma = db.alloc<float>(amb_cap);
        {
            uint32_t* cmarks = db.alloc<uint32_t>(nw);
            cull_marks_kernel<<<blocks(tn, 256), 256>>>(M, train, int(tres), cmarks);
            uint32_t* coffsets;
            unsigned long long* ckeys;
            const uint32_t nc = compact(cmarks, nw, &coffsets, &ckeys);
            float* crows = db.alloc<float>(size_t(nc ? nc : 1) * W);
            launch_corner_eval(M, *A, ckeys, nc, crows);
            check_cuda("bake: cull corners");
            pt.mark("cull_corners");
            cull_table = CornerTable{cmarks, coffsets, crows, (unsigned long long)r1, W};
        }
        cull_kernel<<<blocks(tn, 128), 128>>>(M, cull_table, train, int(tres), cull_step, thresh, culled, amb_n,
                                              amb_idx, amb_sigma, amb_cap);
        check_cuda("bake: cull");
        unsigned int n_amb = 0;
        cudaMemcpy(&n_amb, amb_n, 4, cudaMemcpyDeviceToHost);
        if (n_amb > unsigned(amb_cap)) throw std::runtime_error("bake: too many borderline cull decisions");
        if (n_amb) {  // glibc's exp decides the borderline voxels (baking.hpp:131)
            std::vector<uint32_t> words(words32(tres)), idx(n_amb);
            std::vector<float> sig(n_amb);
            cudaMemcpy(words.data(), culled, words.size() * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(idx.data(), amb_idx, n_amb * 4, cudaMemcpyDeviceToHost);
            cudaMemcpy(sig.data(), amb_sigma, n_amb * 4, cudaMemcpyDeviceToHost);
            for (unsigned k = 0; k < n_amb; ++k) {
                const bool keep = 1.0 - std::exp(-double(sig[k]) * cull_step) > thresh;
                if (keep) words[idx[k] >> 5] |= 1u << (idx[k] & 31);
                else words[idx[k] >> 5] &= ~(1u << (idx[k] & 31));
            }
            cudaMemcpy(culled, words.data(), words.size() * 4, cudaMemcpyHostToDevice);
        }
        pt.mark("cull");
        for (int i = 0; i < dilate; ++i) {
            uint32_t* d2 = db.alloc<uint32_t>(words32(tres));
            dilate_kernel<<<blocks(tn, 256), 256>>>(culled, int(tres), d2);
            culled = d2;
        }
        check_cuda("bake: dilate");

        pt.mark("dilate");
        // (2) render grid, pyramid, distance grid (baking.hpp:137-144)
        const int f = render_res / int(tres);
        uint32_t* levels[NGPRT_PYRAMID_LEVELS];
        levels[0] = db.alloc<uint32_t>(words32(render_res));
        upsample_kernel<<<blocks(size_t(render_res) * render_res * render_res, 256), 256>>>(
            culled, int(tres), f, levels[0]);
        for (int k = 1; k < NGPRT_PYRAMID_LEVELS; ++k) {
            levels[k] = db.alloc<uint32_t>(words32(render_res >> k));
            launch_pyramid_level(levels[k - 1], render_res >> (k - 1), levels[k], nullptr);
        }
        uint8_t* dist = db.alloc<uint8_t>(size_t(256) * 256 * 256);
        uint16_t* ta = db.alloc<uint16_t>(size_t(256) * 256 * 256 + kDistScratchPad / 2);
        uint16_t* tb = db.alloc<uint16_t>(size_t(256) * 256 * 256);
        launch_distance_grid(levels[1], 256, ta, tb, dist, nullptr);
        check_cuda("bake: pyramid / distance grid");

        pt.mark("grids");
        // (3) corner retention on the L_C grid and corner evaluation
        uint32_t* occ_lc = culled;
        int r = int(tres);
        if (lc >= r) {
            if (lc > r) {
                occ_lc = db.alloc<uint32_t>(words32(lc));
                upsample_kernel<<<blocks(size_t(lc) * lc * lc, 256), 256>>>(culled, r, lc / r, occ_lc);
            }
        } else {
            while (r > lc) {  // BitGrid::downsampled2 until res == L_C
                uint32_t* g = db.alloc<uint32_t>(words32(r / 2));
                launch_pyramid_level(occ_lc, r, g, nullptr);
                occ_lc = g;
                r /= 2;
            }
        }
        uint32_t* marks = db.alloc<uint32_t>(nw);
        corner_marks_kernel<<<blocks(size_t(lc) * lc * lc, 256), 256>>>(occ_lc, lc, marks);
        check_cuda("bake: corner marks");
        uint32_t* offsets;
        unsigned long long* dkeys;
        const uint32_t n_keys = compact(marks, nw, &offsets, &dkeys);
        auto b = std::make_unique<ngprt_baked>();
        b->keys.resize(n_keys);
        b->rows.resize(size_t(n_keys) * W);
        pt.mark("keys");
        if (n_keys) {
            float* drows = db.alloc<float>(b->rows.size());
            launch_corner_eval(M, *A, dkeys, n_keys, drows);
            check_cuda("bake: corner evaluation");
            pt.mark("corner_kernel");
            d2h(b->keys.data(), dkeys, size_t(n_keys) * 8);
            d2h(b->rows.data(), drows, b->rows.size() * 4);
        }

        pt.mark("rows_d2h");
        // (4) assemble the BakedScene (verbatim carry-over, baking.hpp:176-200)
        ngprt_scene_desc& d = b->desc;
        d.L = uint32_t(L);
        d.L_C = uint32_t(lc);
        d.fusion_tag = md->fusion_tag;
        for (int l = 0; l < L; ++l) {
            d.fine_res[l] = md->fine_res[l];
            d.fine_table_len[l] = md->fine_table_len[l];
            d.fine_hashed[l] = md->fine_hashed[l];
            b->fine[l].resize(md->fine_table_len[l] * 8);
            parallel_memcpy(b->fine[l].data(), md->fine_tables[l], b->fine[l].size() * 4);
        }
        const int pw[4] = {23, 64, 64, 3};
        for (int k = 0; k < 3; ++k) {
            b->psi_w[k].assign(md->psi_w[k], md->psi_w[k] + size_t(pw[k]) * pw[k + 1]);
            b->psi_b[k].assign(md->psi_b[k], md->psi_b[k] + pw[k + 1]);
        }
        if (inv) b->att.assign(md->att_globals, md->att_globals + 2 * L);
        if (M.fusion == NGPRT_FUSION_MLP) {
            const int fw[3] = {8 * L, 64, 8};
            for (int k = 0; k < 2; ++k) {
                b->fmlp_w[k].assign(md->fusion_mlp_w[k], md->fusion_mlp_w[k] + size_t(fw[k]) * fw[k + 1]);
                b->fmlp_b[k].assign(md->fusion_mlp_b[k], md->fusion_mlp_b[k] + fw[k + 1]);
            }
        }
        for (int k = 0; k < NGPRT_PYRAMID_LEVELS; ++k) {
            const size_t res = size_t(render_res) >> k;
            b->pyramid[k].resize((res * res * res + 63) / 64);
            d2h(b->pyramid[k].data(), levels[k], b->pyramid[k].size() * 8);
        }
        b->dist.resize(size_t(256) * 256 * 256);
        d2h(b->dist.data(), dist, b->dist.size());
        check_cuda("bake: download");
        b->pyramid_base = uint32_t(render_res);
        b->finalize();
        pt.mark("assemble");
        *out = b.release();
        return NGPRT_OK;
    } catch (const std::exception& e) {
        ngprt_host::set_error(e.what());
        return NGPRT_EINVAL;
    }
}
