// occupancy.cu — K3 (occupancy pyramid), K4 (distance grid) and the one-off
// scene layout kernels.
//
// K3 restates BitGrid::downsampled2 (occupancy.hpp:40-51) / build_pyramid
// (:114-119): one thread per output u32 (32 parents along x) ORs the 4 child
// rows' 64-bit words and compacts the bit pairs; levels whose rows are not a
// multiple of 32 voxels take one thread per parent voxel and a warp ballot.
//
// K4 computes the same grid as build_distance_grid (:136-194) — exact
// Chebyshev distance, G = min(255, max(0, D-1)), all-empty -> 255 — but as a
// separable min-max transform instead of the reference's serial two-pass
// chamfer (which has a loop-carried dependency over the whole grid):
//   D(p) = min_qz max(|pz-qz|, min_qy max(|py-qy|, min_qx |px-qx|)).
// Pass X is a two-sweep 1-D distance per row (one warp per row, ballots);
// passes Y and Z take the lower envelope of max(|u - i|, g(i)) per column in
// O(r) (NGPRT_DT_SEARCH: the earlier outward search with early exit).
#include "render.cuh"

namespace ngprt_dev {
namespace {

constexpr uint16_t kInf = 0xFFFF;

// NGPRT_DT_UNSTAGED (experiment): the envelope sweep reads its column through L1
// instead of staging it in shared memory (half the shared memory per column).
#ifndef NGPRT_DT_UNSTAGED
#define NGPRT_DT_UNSTAGED 0
#endif

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

// Word-level K3 (parent rows a multiple of 32 voxels): one thread per output u32,
// i.e. 32 parents along x. Their children are 64 bits (two u32) in each of the 4
// child rows (y, z parity); OR the rows, OR each bit pair, and compact the even
// bits: 8 loads per 32 parents instead of 8 per parent.
__device__ __forceinline__ uint32_t even_bits(uint64_t v) {  // bit 2j -> bit j
    v &= 0x5555555555555555ull;
    v = (v | (v >> 1)) & 0x3333333333333333ull;
    v = (v | (v >> 2)) & 0x0f0f0f0f0f0f0f0full;
    v = (v | (v >> 4)) & 0x00ff00ff00ff00ffull;
    v = (v | (v >> 8)) & 0x0000ffff0000ffffull;
    v = (v | (v >> 16)) & 0x00000000ffffffffull;
    return uint32_t(v);
}
__global__ void pyramid_word_kernel(const uint32_t* __restrict__ src, int rs,
                                    uint32_t* __restrict__ dst, int ro) {
    const size_t nw = size_t(ro) * ro * ro / 32;
    const size_t w = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (w >= nw) return;
    const size_t p0 = w * 32;  // first parent voxel of this word
    const int xw = int(p0 % ro), y = int((p0 / ro) % ro), z = int(p0 / (size_t(ro) * ro));
    uint64_t v = 0;
#pragma unroll
    for (int c = 0; c < 4; ++c) {
        const size_t bit = size_t(2 * xw) + size_t(rs) * (size_t(2 * y + (c & 1)) + size_t(rs) * size_t(2 * z + (c >> 1)));
        const uint2 pr = *reinterpret_cast<const uint2*>(src + (bit >> 5));  // 64-bit aligned: rs % 64 == 0
        v |= uint64_t(pr.x) | (uint64_t(pr.y) << 32);
    }
    dst[w] = even_bits(v | (v >> 1));
}

// Pass X: per row (y, z), distance to the nearest occupied voxel along x. One
// warp per row, 32 voxels per step: a ballot of the occupancy bits gives, per
// lane, the nearest set bit at or before it inside the step (a masked clz) and a
// warp-uniform carry of the last set bit of earlier steps; a backward sweep does
// the same for the nearest set bit after. Loads and u16 stores are coalesced
// (64 B per warp store).
__global__ void dt_x_warp_kernel(const uint32_t* __restrict__ occ, int r, uint16_t* __restrict__ out) {
    const size_t row = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (row >= size_t(r) * r) return;  // warp-uniform
    const size_t base = row * size_t(r);
    uint16_t* o = out + base;
    const int groups = (r + 31) / 32;
    int last = -1;  // last occupied x before the current group (warp-uniform)
    for (int g = 0; g < groups; ++g) {
        const int x = g * 32 + int(lane);
        const size_t i = base + size_t(x);
        const bool in = x < r;
        const bool bit = in && ((occ[i >> 5] >> (i & 31)) & 1u);
        const uint32_t m = __ballot_sync(0xffffffffu, bit);
        const uint32_t le = m & (0xffffffffu >> (31u - lane));  // bits at or before lane
        const int prev = le ? g * 32 + 31 - __clz(le) : last;
        if (in) o[x] = prev < 0 ? kInf : uint16_t(min(x - prev, int(kInf)));
        if (m) last = g * 32 + 31 - __clz(m);
    }
    int next = -1;  // first occupied x after the current group
    for (int g = groups - 1; g >= 0; --g) {
        const int x = g * 32 + int(lane);
        const size_t i = base + size_t(x);
        const bool in = x < r;
        const bool bit = in && ((occ[i >> 5] >> (i & 31)) & 1u);
        const uint32_t m = __ballot_sync(0xffffffffu, bit);
        const uint32_t ge = m & (0xffffffffu << lane);  // bits at or after lane
        const int nx = ge ? g * 32 + __ffs(ge) - 1 : next;
        if (in && nx >= 0) {
            const uint16_t d = uint16_t(min(nx - x, int(kInf)));
            if (d < o[x]) o[x] = d;
        }
        if (m) next = g * 32 + __ffs(m) - 1;
    }
}

// Pass X, one thread per row (the first version; kept for NGPRT_DT_X_SERIAL A/B).
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

// Passes Y and Z in O(r) per column: the lower envelope of the functions
// f_i(u) = max(|u - i|, g(i)) over the column (Meijster, Roerdink & Hesselink's
// separable transform with its chessboard-metric separator), one thread per
// column; consecutive threads take consecutive x, so every load and store of the
// sweep is coalesced. The envelope stacks (s: function index, t: start of its
// interval) live in the thread's local memory (L1). Exact integer arithmetic:
// the same grid as the early-exit search above and the reference's chamfer.
__device__ __forceinline__ int cheb_f(int u, int i, int gi) {
    const int d = u > i ? u - i : i - u;
    return d > gi ? d : gi;
}
__device__ __forceinline__ int cheb_sep(int i, int u, int gi, int gu) {
    const int mid = (i + u) >> 1;  // i < u, both >= 0: floor
    if (gi <= gu) return (i + gu) > mid ? (i + gu) : mid;
    return (u - gi) < mid ? (u - gi) : mid;
}
// The column is first staged in shared memory (independent coalesced loads, all
// in flight at once) and the envelope stacks live in shared memory too (IT =
// u8 indices for r <= 256), so the sequential sweep touches no global or local
// memory: per CTA r x C x (2 + 2 sizeof(IT)) bytes.
template <int AXIS, bool FINAL, typename IT>
__global__ void __launch_bounds__(64) dt_envelope_kernel(const uint16_t* __restrict__ in, int r,
                                                         uint16_t* __restrict__ out,
                                                         uint8_t* __restrict__ out8) {
    extern __shared__ __align__(16) uint16_t colbuf[];  // [r][C] column, then s [r][C], t [r][C]
    const int C = blockDim.x, tid = threadIdx.x;
    IT* s = reinterpret_cast<IT*>(colbuf + (NGPRT_DT_UNSTAGED ? 0 : size_t(r) * C)) + tid;
    IT* t = s + size_t(r) * C;
    const size_t col = blockIdx.x * size_t(C) + tid;
    const bool live = col < size_t(r) * r;
    // AXIS 1 (y): column (x, z), element u at (z * r + u) * r + x
    // AXIS 2 (z): column (x, y), element u at (u * r + y) * r + x
    const size_t x = col % size_t(r), o = col / size_t(r);
    const size_t base = AXIS == 1 ? o * size_t(r) * r + x : o * size_t(r) + x;
    const size_t stride = AXIS == 1 ? size_t(r) : size_t(r) * r;
#if NGPRT_DT_UNSTAGED
    // variant: no column staging; the sweep reads the column through L1 (the next
    // element prefetched one step ahead), the stacks alone take shared memory
    if (!live) return;
    {
    const uint16_t* gcol = in + base;
    auto G = [&](int u) -> int { return __ldg(gcol + size_t(u) * stride); };
    int q = 0, sq = 0, tq = 0;
    s[0] = 0;
    t[0] = 0;
    int gs = G(0);
    int gnext = r > 1 ? G(1) : 0;
    for (int u = 1; u < r; ++u) {
        const int gu = gnext;
        if (u + 1 < r) gnext = G(u + 1);
        while (q >= 0 && cheb_f(tq, sq, gs) > cheb_f(tq, u, gu)) {
            --q;
            if (q >= 0) {
                sq = s[q * C];
                tq = t[q * C];
                gs = G(sq);
            }
        }
        if (q < 0) {
            q = 0;
            sq = u;
            tq = 0;
            s[0] = IT(u);
            t[0] = 0;
            gs = gu;
        } else {
            const int w = 1 + cheb_sep(sq, u, gs, gu);
            if (w < r) {
                ++q;
                sq = u;
                tq = w;
                s[q * C] = IT(u);
                t[q * C] = IT(w);
                gs = gu;
            }
        }
    }
    for (int u = r - 1; u >= 0; --u) {
        const int h = cheb_f(u, sq, gs);
        const size_t i = base + size_t(u) * stride;
        if (FINAL) {
            const int gg = h == 0 ? 0 : h - 1;  // occupancy.hpp:188-192
            out8[i] = uint8_t(gg < 255 ? gg : 255);
        } else {
            out[i] = uint16_t(h < int(kInf) ? h : int(kInf));
        }
        if (u == tq && q > 0) {
            --q;
            sq = s[q * C];
            tq = t[q * C];
            gs = G(sq);
        }
    }
    return;
    }
#endif
    uint16_t* g = colbuf + tid;
    if (r % C == 0 && C % 8 == 0) {
        // the CTA's C columns are C consecutive x of one row: stage the r segments of
        // C u16 cooperatively with 16 B loads (C / 8 threads per segment)
        const size_t x0 = (blockIdx.x * size_t(C)) % size_t(r), o0 = (blockIdx.x * size_t(C)) / size_t(r);
        const size_t b0 = AXIS == 1 ? o0 * size_t(r) * r + x0 : o0 * size_t(r) + x0;
        const int per = C / 8, segs_per_pass = blockDim.x / per;
#pragma unroll 4
        for (int u = tid / per; u < r; u += segs_per_pass) {
            const uint4 v = *reinterpret_cast<const uint4*>(in + b0 + size_t(u) * stride + (tid % per) * 8);
            *reinterpret_cast<uint4*>(colbuf + size_t(u) * C + (tid % per) * 8) = v;
        }
        __syncthreads();
        if (!live) return;
    } else {
        if (!live) return;  // each thread stages and sweeps its own column
#pragma unroll 8
        for (int u = 0; u < r; ++u) g[u * C] = in[base + size_t(u) * stride];
    }
    // stack entry q at s[q * C] / t[q * C]; the top (sq, tq, gs) is kept in registers
    int q = 0, sq = 0, tq = 0;
    s[0] = 0;
    t[0] = 0;
    int gs = g[0];  // g(s[q])
    for (int u = 1; u < r; ++u) {
        const int gu = g[u * C];
        while (q >= 0 && cheb_f(tq, sq, gs) > cheb_f(tq, u, gu)) {
            --q;
            if (q >= 0) {
                sq = s[q * C];
                tq = t[q * C];
                gs = g[sq * C];
            }
        }
        if (q < 0) {
            q = 0;
            sq = u;
            tq = 0;
            s[0] = IT(u);
            t[0] = 0;
            gs = gu;
        } else {
            const int w = 1 + cheb_sep(sq, u, gs, gu);
            if (w < r) {
                ++q;
                sq = u;
                tq = w;
                s[q * C] = IT(u);
                t[q * C] = IT(w);
                gs = gu;
            }
        }
    }
    for (int u = r - 1; u >= 0; --u) {
        const int h = cheb_f(u, sq, gs);
        const size_t i = base + size_t(u) * stride;
        if (FINAL) {
            const int gg = h == 0 ? 0 : h - 1;  // occupancy.hpp:188-192
            out8[i] = uint8_t(gg < 255 ? gg : 255);
        } else {
            out[i] = uint16_t(h < int(kInf) ? h : int(kInf));
        }
        if (u == tq && q > 0) {
            --q;
            sq = s[q * C];
            tq = t[q * C];
            gs = g[sq * C];
        }
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
    if (ro % 32 == 0)  // every output word is 32 parents of one row
        pyramid_word_kernel<<<blocks_for(n / 32, 256), 256, 0, st>>>(src, src_res, dst, ro);
    else
        pyramid_kernel<<<blocks_for(n, 256), 256, 0, st>>>(src, src_res, dst, ro);
}

void launch_distance_grid(const uint32_t* occ, int r, uint16_t* a, uint16_t* b, uint8_t* out,
                          cudaStream_t st) {
    const size_t rows = size_t(r) * r, n = rows * r;
#ifdef NGPRT_DT_X_SERIAL
    dt_x_kernel<<<blocks_for(rows, 128), 128, 0, st>>>(occ, r, a);
#else
    dt_x_warp_kernel<<<blocks_for(rows * 32, 256), 256, 0, st>>>(occ, r, a);
#endif
#ifdef NGPRT_DT_SEARCH
    dt_minmax_kernel<1, false><<<blocks_for(n, 256), 256, 0, st>>>(a, r, b, nullptr);
    dt_minmax_kernel<2, true><<<blocks_for(n, 256), 256, 0, st>>>(b, r, nullptr, out);
#else
    static PerDeviceInt attrs;  // opt in to > 48 KB of dynamic shared memory, once per device
    attrs.get([](int) {
        cudaFuncSetAttribute(dt_envelope_kernel<1, false, uint8_t>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 64 * 4);
        cudaFuncSetAttribute(dt_envelope_kernel<2, true, uint8_t>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 64 * 4);
        cudaFuncSetAttribute(dt_envelope_kernel<1, false, uint16_t>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 16 * 6);
        cudaFuncSetAttribute(dt_envelope_kernel<2, true, uint16_t>,
                             cudaFuncAttributeMaxDynamicSharedMemorySize, 1024 * 16 * 6);
        return 1;
    });
    if (r <= 256) {  // 64 columns per CTA, u8 stack indices: r x 64 x 4 B (<= 64 KB)
        const size_t sm = size_t(r) * 64 * (NGPRT_DT_UNSTAGED ? 2 : 4);
        dt_envelope_kernel<1, false, uint8_t><<<blocks_for(rows, 64), 64, sm, st>>>(a, r, b, nullptr);
        dt_envelope_kernel<2, true, uint8_t><<<blocks_for(rows, 64), 64, sm, st>>>(b, r, nullptr, out);
    } else if (r <= 1024) {  // 16 columns per CTA, u16 stack indices: r x 16 x 6 B (<= 96 KB)
        const size_t sm = size_t(r) * 16 * (NGPRT_DT_UNSTAGED ? 4 : 6);
        dt_envelope_kernel<1, false, uint16_t><<<blocks_for(rows, 16), 16, sm, st>>>(a, r, b, nullptr);
        dt_envelope_kernel<2, true, uint16_t><<<blocks_for(rows, 16), 16, sm, st>>>(b, r, nullptr, out);
    } else {  // beyond the envelope stacks' size: the outward search
        dt_minmax_kernel<1, false><<<blocks_for(n, 256), 256, 0, st>>>(a, r, b, nullptr);
        dt_minmax_kernel<2, true><<<blocks_for(n, 256), 256, 0, st>>>(b, r, nullptr, out);
    }
#endif
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
