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
#include <stdlib.h>

#include "render.cuh"

namespace ngprt_dev {
namespace {

constexpr uint16_t kInf = 0xFFFF;

// NGPRT_DT_UNSTAGED (experiment): the envelope sweep reads its column through L1
// instead of staging it in shared memory (half the shared memory per column).
#ifndef NGPRT_DT_UNSTAGED
#define NGPRT_DT_UNSTAGED 0
#endif
// NGPRT_DT_U16=1: the u16 passes for every r (A/B against the u8 passes, r <= 256)
#ifndef NGPRT_DT_U16
#define NGPRT_DT_U16 0
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
// OT = uint16_t: distances with kInf for a row without occupied voxels; OT =
// uint8_t (r <= 256): distances saturated at 255 (see dt_deque_kernel), and
// `nonempty` (nullable) set once any row holds an occupied voxel.
template <class OT>
__global__ void dt_x_warp_kernel(const uint32_t* __restrict__ occ, int r, OT* __restrict__ out,
                                 uint32_t* __restrict__ nonempty) {
    constexpr int kSat = sizeof(OT) == 1 ? 255 : int(kInf);
    const size_t row = (blockIdx.x * size_t(blockDim.x) + threadIdx.x) >> 5;
    const uint32_t lane = threadIdx.x & 31u;
    if (row >= size_t(r) * r) return;  // warp-uniform
    const size_t base = row * size_t(r);
    OT* o = out + base;
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
        if (in) o[x] = OT(prev < 0 ? kSat : min(x - prev, kSat));
        if (m) last = g * 32 + 31 - __clz(m);
    }
    if (nonempty && last >= 0 && lane == 0 &&
        *reinterpret_cast<volatile uint32_t*>(nonempty) == 0)
        atomicOr(nonempty, 1u);
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
            const OT d = OT(min(nx - x, kSat));
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

// Passes Y and Z for r <= 256 on u8 values saturated at 255. Saturation
// commutes with every pass: with S(v) = min(v, 255) and |u - i| <= 255,
//   min_i max(|u - i|, S(g_i)) = min(min_i max(|u - i|, g_i), 255),
// so the u8 passes give S(D). D itself is <= 255 whenever any voxel is occupied
// (two voxels of a 256^3 grid are at most 255 apart), so G = max(0, D - 1)
// follows from S(D) except for the all-empty grid, which `nonempty` (set by
// pass X) maps to 255.
//
// Per column, D(u) = min(F_L(u), F_R(u)) with F_L(u) = min_{i <= u} max(u - i, g_i)
// (F_R mirrored). A forward sweep keeps F_L's candidates in a monotone deque: a
// new i retires every older candidate with g >= g_i (it is nearer and no
// higher, so never worse again), so g rises from front to back; the front
// retires once the next entry is no worse — the front is then on its rising
// part (u - i >= g_front, else it would beat the higher-g entry), grows by 1 per
// step, and the next entry grows by at most 1, so it never wins again. F_L(u) is
// the front's value. The backward sweep runs the same on the reversed column
// and takes the minimum with the stored F_L. O(r) per column, integer, exact.
// The deques are short on scene data (<= 5 entries on the c3 grid's columns;
// a long deque needs g rising ~1 per voxel over a long run, e.g. next to a
// diagonal wall): each thread keeps a ring of `ring` u16 entries (index, g) in
// shared memory, and a column whose deque outgrows it is redone with its deque
// in global scratch (`spill`, r entries per column, column-interleaved), which
// cannot overflow. No column staging: the sweeps read their column directly
// (consecutive threads take consecutive x, so each load and store is one
// coalesced 32 B access per warp), eight steps' loads issued together.
constexpr int kDequeBlock = 256;
struct SmemRing {
    uint16_t* base;  // this thread's entry 0; entries kDequeBlock apart
    int mask;
    __device__ uint16_t get(int k) const { return base[(k & mask) * kDequeBlock]; }
    __device__ void set(int k, uint16_t v) const { base[(k & mask) * kDequeBlock] = v; }
    __device__ bool full(int len) const { return len > mask; }
};
struct GlobalDeque {
    uint16_t* base;  // spill + column; entry k at base[k * ncols]
    uint32_t stride;
    __device__ uint16_t get(int k) const { return base[uint32_t(k) * stride]; }
    __device__ void set(int k, uint16_t v) const { base[uint32_t(k) * stride] = v; }
    __device__ bool full(int) const { return false; }
};

// One sweep over the column in step order p = 0..r-1 (element u = REV ? r-1-p : p,
// at in/out[base + u * stride]; r^3 <= 2^24, so 32-bit offsets). Deque entries
// pack (p, g) as p | g << 8 in [head, tail); the front (fp, fg) and the back's g
// stay in registers. Forward: out[u] = F_L(u). Reverse: out[u] =
// final(min(out[u], F_R(u))). Returns false if the deque outgrew Q.
template <bool REV, bool FINAL, class Q>
__device__ __forceinline__ bool dt_sweep(const Q& q, const uint8_t* __restrict__ in,
                                         uint8_t* __restrict__ out, uint32_t base,
                                         uint32_t stride, int r, bool empty) {
    int head = 0, tail = 0, fp = 0, fg = 0, bg = 0;
    const int32_t step = REV ? -int32_t(stride) : int32_t(stride);
    uint32_t off = REV ? base + uint32_t(r - 1) * stride : base;
    for (int p0 = 0; p0 < r; p0 += 8, off += 8 * step) {
        int gv[8], fl[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const uint32_t o = off + j * step;
            gv[j] = p0 + j < r ? int(in[o]) : 0;
            if (REV) fl[j] = p0 + j < r ? int(out[o]) : 0;
        }
#pragma unroll
        for (int j = 0; j < 8; ++j) {
            const int p = p0 + j;
            if (p >= r) break;
            const int gp = gv[j];
            // retire older candidates that are no nearer and no lower
            while (tail > head && bg >= gp) {
                --tail;
                if (tail > head) bg = q.get(tail - 1) >> 8;
            }
            if (tail == head) {
                fp = p;
                fg = gp;
            } else if (q.full(tail - head)) {
                return false;
            }
            q.set(tail++, uint16_t(p | (gp << 8)));
            bg = gp;
            // retire the front while the next entry is no worse
            int v0 = max(p - fp, fg);
            while (tail - head >= 2) {
                const int e1 = q.get(head + 1);
                const int v1 = max(p - (e1 & 0xFF), e1 >> 8);
                if (v0 < v1) break;
                ++head;
                fp = e1 & 0xFF;
                fg = e1 >> 8;
                v0 = v1;
            }
            int h = v0;
            if (REV) {
                h = min(h, fl[j]);
                if (FINAL) h = empty ? 255 : (h == 0 ? 0 : h - 1);  // occupancy.hpp:188-192
            }
            out[off + j * step] = uint8_t(h);
        }
    }
    return true;
}

template <int AXIS, bool FINAL>
__global__ void __launch_bounds__(kDequeBlock) dt_deque_kernel(const uint8_t* __restrict__ in,
                                                               int r, int ring,
                                                               uint8_t* __restrict__ out,
                                                               uint16_t* __restrict__ spill,
                                                               const uint32_t* __restrict__ nonempty) {
    extern __shared__ uint16_t rings[];  // [ring][kDequeBlock]
    const uint32_t ncols = uint32_t(r) * r;
    const uint32_t col = blockIdx.x * kDequeBlock + threadIdx.x;
    if (col >= ncols) return;
    const uint32_t x = col % uint32_t(r), o = col / uint32_t(r);
    // AXIS 1 (y): column (x, z), element u at (z * r + u) * r + x
    // AXIS 2 (z): column (x, y), element u at (u * r + y) * r + x
    const uint32_t base = AXIS == 1 ? o * ncols + x : o * uint32_t(r) + x;
    const uint32_t stride = AXIS == 1 ? uint32_t(r) : ncols;
    const bool empty = FINAL && *nonempty == 0;
    const SmemRing sq{rings + threadIdx.x, ring - 1};
    if (dt_sweep<false, FINAL>(sq, in, out, base, stride, r, empty) &&
        dt_sweep<true, FINAL>(sq, in, out, base, stride, r, empty))
        return;
    const GlobalDeque gq{spill + col, ncols};  // the deque outgrew the ring: redo the column
    dt_sweep<false, FINAL>(gq, in, out, base, stride, r, empty);
    dt_sweep<true, FINAL>(gq, in, out, base, stride, r, empty);
}

// Passes Y and Z for r a multiple of 32 (<= 256), data-parallel: with
// P_u(d) = [min(g[u-d .. u+d]) <= d] (monotone in d), D(u) = min{d : P_u(d)} —
// the window test is one range-minimum query on a per-column sparse table
// (levels 0..7, u16 entries so a level is built with packed VIMNMX.U16x2 on
// 16 B rows). D is 1-Lipschitz along the column, so a lane binary-searches only
// its first element (<= 8 queries) and steps each next one from D(u-1) in
// {D-1, D, D+1} (one query plus two table reads). D is also 1-Lipschitz
// across x, so only a warp's first column runs the per-lane chains: a CTA
// stages 32 columns (consecutive x) transposed into shared memory, its 8 warps
// take 4 adjacent columns each, every element of the next columns steps
// independently from the previous column's D at the same u, and the
// results go back through the same tile as 16 B stores. FROM_BITS (pass Y):
// the tile is pass X itself — each thread takes one row's occupancy words and
// writes the 32 x-distances of the tile's x range (nearest set bit at or
// before / at or after, within the row's word or from the row's other words),
// so pass X needs no kernel or buffer of its own. Exact integer arithmetic,
// same values as the deque sweeps and the reference.
// a[i] = bytes 0..3 of column i (4 rows) <-> a[j] = bytes 0..3 of row j (4 columns)
__device__ __forceinline__ void transpose4x4(uint32_t a[4]) {
    const uint32_t t0 = __byte_perm(a[0], a[1], 0x5140), t1 = __byte_perm(a[2], a[3], 0x5140);
    const uint32_t t2 = __byte_perm(a[0], a[1], 0x7362), t3 = __byte_perm(a[2], a[3], 0x7362);
    a[0] = __byte_perm(t0, t1, 0x5410);
    a[1] = __byte_perm(t0, t1, 0x7632);
    a[2] = __byte_perm(t2, t3, 0x5410);
    a[3] = __byte_perm(t2, t3, 0x7632);
}
// Levels 0..7: a window of up to 2^8 = 256 >= r entries is covered by two level-7 rows.
constexpr int kRmqCols = 32, kRmqThreads = 256, kRmqPitch = 260, kRmqLevels = 8;
template <int AXIS, bool FINAL, bool FROM_BITS>
__global__ void __launch_bounds__(kRmqThreads) dt_rmq_kernel(const uint8_t* __restrict__ in,
                                                             const uint32_t* __restrict__ occ,
                                                             int r, uint8_t* __restrict__ out,
                                                             uint32_t* __restrict__ nonempty) {
    __shared__ __align__(16) uint8_t tile[kRmqCols * kRmqPitch];               // [column][u]
    __shared__ __align__(16) uint16_t tabs[kRmqThreads / 32][kRmqLevels * 256];  // per warp
    __shared__ uint8_t dbufs[kRmqThreads / 32][256];  // per warp: first column's D
    const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
    const uint32_t ncols = uint32_t(r) * r, col0 = blockIdx.x * kRmqCols;
    const uint32_t x0 = col0 % uint32_t(r), o = col0 / uint32_t(r);
    // AXIS 1 (y): element (x, u) of slice z = o at (o * r + u) * r + x
    // AXIS 2 (z): element (x, u) of row y = o at (u * r + o) * r + x
    const uint32_t base0 = AXIS == 1 ? o * ncols + x0 : o * uint32_t(r) + x0;
    const uint32_t stride = AXIS == 1 ? uint32_t(r) : ncols;
    if constexpr (FROM_BITS) {
        bool any = false;
        for (int y = tid; y < r; y += kRmqThreads) {  // row (y, z = o): r / 32 words
            const uint32_t* row = occ + (size_t(o) * r + y) * (r >> 5);
            const int nw = r >> 5, wx = int(x0 >> 5);
            int lp = -1, fn = -1;  // last set bit before / first after the tile's word
            uint32_t W = 0;
            for (int w = 0; w < nw; ++w) {
                const uint32_t v = row[w];
                any |= v != 0;
                if (w < wx && v) lp = w * 32 + 31 - __clz(v);
                if (w == wx) W = v;
                if (w > wx && v && fn < 0) fn = w * 32 + __ffs(v) - 1;
            }
#pragma unroll 8
            for (int bpos = 0; bpos < 32; ++bpos) {
                const int x = int(x0) + bpos;
                const uint32_t le = W & (0xffffffffu >> (31 - bpos)), ge = W & (0xffffffffu << bpos);
                const int prev = le ? int(x0) + 31 - __clz(le) : lp;
                const int next = ge ? int(x0) + __ffs(ge) - 1 : fn;
                const int dp = prev >= 0 ? x - prev : 255, dn = next >= 0 ? next - x : 255;
                tile[bpos * kRmqPitch + y] = uint8_t(min(min(dp, dn), 255));
            }
        }
        if (__syncthreads_or(any) && tid == 0 && *reinterpret_cast<volatile uint32_t*>(nonempty) == 0)
            atomicOr(nonempty, 1u);
    } else {
        // 4 x 4 byte blocks: 4 rows of 4 columns in (coalesced: 8 threads per 32 B
        // row), transposed in registers, 4 column words out (conflict-free: pitch
        // 65 words)
        for (int blk = tid; blk < 8 * (r >> 2); blk += kRmqThreads) {
            const int cg = blk & 7, u = (blk >> 3) * 4;
            uint32_t a[4];
#pragma unroll
            for (int j = 0; j < 4; ++j)
                a[j] = *reinterpret_cast<const uint32_t*>(in + base0 + (u + j) * stride + cg * 4);
            transpose4x4(a);
#pragma unroll
            for (int i = 0; i < 4; ++i)
                *reinterpret_cast<uint32_t*>(tile + (cg * 4 + i) * kRmqPitch + u) = a[i];
        }
        __syncthreads();
    }
    const bool empty = FINAL && *reinterpret_cast<volatile uint32_t*>(nonempty) == 0;
    uint16_t* T = tabs[warp];
    const int E = r >> 5;  // elements per lane
    const bool builder = lane * 8 < r;  // table rows: 8 entries (16 B) per lane
    constexpr int kColsPerWarp = kRmqCols / (kRmqThreads / 32);
    uint8_t* dbuf = dbufs[warp];
    int dv[8];  // D(32 e + lane) of the previous column
    for (int j = 0; j < kColsPerWarp; ++j) {
        const int c = warp * kColsPerWarp + j;  // adjacent x: D is 1-Lipschitz across them too
        uint8_t* colv = tile + c * kRmqPitch;
        if (builder) {
            const uint32_t* cw = reinterpret_cast<const uint32_t*>(colv + lane * 8);  // 4 B aligned
            const uint2 v = make_uint2(cw[0], cw[1]);
            *reinterpret_cast<uint4*>(T + lane * 8) =
                make_uint4(__byte_perm(v.x, 0, 0x4140), __byte_perm(v.x, 0, 0x4342),
                           __byte_perm(v.y, 0, 0x4140), __byte_perm(v.y, 0, 0x4342));
        }
        __syncwarp();
        // level k: T_k[i] = min(T_{k-1}[i], T_{k-1}[i + 2^(k-1)]), valid for i <= r - 2^k
        // (entries past that read the next rows: garbage, never queried)
        for (int k = 1; k < kRmqLevels && (1 << k) <= r; ++k) {
            const uint16_t* prev = T + (k - 1) * 256;
            const int off = 1 << (k - 1);
            if (builder) {
                const uint4 a = *reinterpret_cast<const uint4*>(prev + lane * 8);
                uint4 b;
                if (off >= 8) {
                    b = *reinterpret_cast<const uint4*>(prev + lane * 8 + off);
                } else {
                    const uint32_t* pw = reinterpret_cast<const uint32_t*>(prev + lane * 8 + (off & ~1));
                    uint32_t w[5];
#pragma unroll
                    for (int q = 0; q < 5; ++q) w[q] = pw[q];
                    if (off & 1) {
                        b = make_uint4(__funnelshift_r(w[0], w[1], 16), __funnelshift_r(w[1], w[2], 16),
                                       __funnelshift_r(w[2], w[3], 16), __funnelshift_r(w[3], w[4], 16));
                    } else {
                        b = make_uint4(w[0], w[1], w[2], w[3]);
                    }
                }
                *reinterpret_cast<uint4*>(T + k * 256 + lane * 8) =
                    make_uint4(__vminu2(a.x, b.x), __vminu2(a.y, b.y), __vminu2(a.z, b.z),
                               __vminu2(a.w, b.w));
            }
            __syncwarp();
        }
        auto rmq = [&](int lo, int hi) {  // min(g[lo .. hi]), lo <= hi
            const int k = min(31 - __clz(hi - lo + 1), kRmqLevels - 1);
            const uint16_t* row = T + k * 256;
            return int(min(row[lo], row[hi - (1 << k) + 1]));
        };
        // D(u) from a neighbour's value d (D(u-1), or D(u) of the previous column):
        // D(u) in {d-1, d, d+1}. The radius-d window's minimum is the radius-(d-1)
        // window's (one query) with g[u-d] and g[u+d] added (clamped to the
        // column: a clipped side's end is already inside the smaller window).
        // Branch-free, so the warp stays converged.
        auto step = [&](int u, int d) {
            // (d == 0: the radius -1 window is empty; query [u, u] and discard it)
            const int q1 = rmq(max(0, u - max(d - 1, 0)), min(r - 1, u + max(d - 1, 0)));
            const int m1 = d >= 1 ? q1 : 0xFFFF;
            const int m2 = min(m1, int(min(T[max(u - d, 0)], T[min(u + d, r - 1)])));
            return m1 <= d - 1 ? d - 1 : (m2 <= d ? d : d + 1);
        };
        if (j == 0) {
            // first column: a chain per lane over u0 .. u0+E-1. D(u0) = min{d :
            // min(g[u0-d .. u0+d]) <= d} <= g[u0] <= 255 by the same 8 bisection
            // steps in every lane (the predicate is monotone in d), then steps
            const int u0 = lane * E;
            int d = 0;
#pragma unroll
            for (int bit = 128; bit >= 1; bit >>= 1) {
                const int m = d + bit - 1;
                if (rmq(max(0, u0 - m), min(r - 1, u0 + m)) > m) d += bit;
            }
#pragma unroll 8
            for (int e = 0; e < E; ++e) {
                const int u = u0 + e;
                if (e > 0) d = step(u, d);
                colv[u] = uint8_t(FINAL ? (empty ? 255 : max(d - 1, 0)) : d);  // occupancy.hpp:188-192
                dbuf[u] = uint8_t(d);
            }
            __syncwarp();
#pragma unroll
            for (int e = 0; e < 8; ++e)
                if (e < E) dv[e] = dbuf[32 * e + lane];
        } else {
            // next columns: every element steps from the previous column's D at the
            // same u (independent steps; lanes take consecutive u, so the table
            // reads of a warp spread over the banks)
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                if (e < E) {
                    const int u = 32 * e + lane;
                    dv[e] = step(u, dv[e]);
                    colv[u] = uint8_t(FINAL ? (empty ? 255 : max(dv[e] - 1, 0)) : dv[e]);
                }
            }
        }
        __syncwarp();
    }
    __syncthreads();
    for (int blk = tid; blk < 8 * (r >> 2); blk += kRmqThreads) {
        const int cg = blk & 7, u = (blk >> 3) * 4;
        uint32_t a[4];
#pragma unroll
        for (int i = 0; i < 4; ++i)
            a[i] = *reinterpret_cast<const uint32_t*>(tile + (cg * 4 + i) * kRmqPitch + u);
        transpose4x4(a);
#pragma unroll
        for (int j = 0; j < 4; ++j)
            *reinterpret_cast<uint32_t*>(out + base0 + (u + j) * stride + cg * 4) = a[j];
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

// Cell-brick copy of the fp16 coarse grid (NGPRT_COARSE_CELLS): thread = (cell,
// corner k, word j) copies word j of corner k's row into the cell's record.
__global__ void coarse_cells_kernel(const uint32_t* __restrict__ dense, int lc, int w2,
                                    uint32_t* __restrict__ cells, size_t n) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const size_t per_cell = size_t(8) * w2;
        const size_t cell = i / per_cell;
        const int r = int(i - cell * per_cell), k = r / w2, j = r - k * w2;
        const size_t cx = cell % lc, cy = (cell / lc) % lc, cz = cell / (size_t(lc) * lc);
        const size_t r1 = size_t(lc) + 1;
        const size_t key = (cx + (k & 1)) + r1 * ((cy + ((k >> 1) & 1)) + r1 * (cz + (k >> 2)));
        cells[i] = dense[key * 8 + j];  // a row is 16 fp16 = 8 words
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
#if !defined(NGPRT_DT_X_SERIAL) && !defined(NGPRT_DT_SEARCH) && !NGPRT_DT_U16
    if (r <= 256) {  // u8 passes (dt_deque_kernel)
        // b (2n bytes) holds the x and y results (n bytes each), a (2n + 64 bytes,
        // kDistScratchPad) the deque spill space (r u16 entries per column) and
        // `nonempty` after it
        uint8_t* x8 = reinterpret_cast<uint8_t*>(b);
        uint8_t* y8 = x8 + n;
        uint32_t* nonempty =
            reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(a) + ((2 * n + 15) & ~size_t(15)));
        cudaMemsetAsync(nonempty, 0, sizeof(uint32_t), st);
        const char* env = getenv("NGPRT_DT_RING");  // test hook: the deque kernel, ring size
        if (r % 32 == 0 && !env) {  // pass X fused into pass Y's tile staging
            dt_rmq_kernel<1, false, true><<<unsigned(rows / kRmqCols), kRmqThreads, 0, st>>>(
                nullptr, occ, r, y8, nonempty);
            dt_rmq_kernel<2, true, false><<<unsigned(rows / kRmqCols), kRmqThreads, 0, st>>>(
                y8, nullptr, r, out, nonempty);
            return;
        }
        dt_x_warp_kernel<uint8_t><<<blocks_for(rows * 32, 256), 256, 0, st>>>(occ, r, x8, nonempty);
        int ring = 16;
        if (env) {
            const int want = atoi(env);
            ring = 1;
            while (ring < want && ring < 256) ring *= 2;
        }
        const size_t sm = size_t(ring) * kDequeBlock * sizeof(uint16_t);
        static PerDeviceInt attrs8;  // > 48 KB only for forced large rings
        attrs8.get([](int) {
            cudaFuncSetAttribute(dt_deque_kernel<1, false>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 256 * 2);
            cudaFuncSetAttribute(dt_deque_kernel<2, true>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, 256 * 256 * 2);
            return 1;
        });
        dt_deque_kernel<1, false><<<blocks_for(rows, kDequeBlock), kDequeBlock, sm, st>>>(x8, r, ring, y8, a, nullptr);
        dt_deque_kernel<2, true><<<blocks_for(rows, kDequeBlock), kDequeBlock, sm, st>>>(y8, r, ring, out, a, nonempty);
        return;
    }
#endif
#ifdef NGPRT_DT_X_SERIAL
    dt_x_kernel<<<blocks_for(rows, 128), 128, 0, st>>>(occ, r, a);
#else
    dt_x_warp_kernel<uint16_t><<<blocks_for(rows * 32, 256), 256, 0, st>>>(occ, r, a, nullptr);
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

void launch_coarse_cells(const void* dense_f16, int L_C, int w, void* cells, cudaStream_t st) {
    const size_t n = size_t(L_C) * L_C * L_C * 8 * (w / 2);
    coarse_cells_kernel<<<148 * 16, 256, 0, st>>>(static_cast<const uint32_t*>(dense_f16), L_C, w / 2,
                                                  static_cast<uint32_t*>(cells), n);
}

void launch_convert_fine(const float* src, void* dst, size_t n, int f16, cudaStream_t st) {
    if (f16)
        convert_f16_kernel<<<148 * 8, 256, 0, st>>>(src, reinterpret_cast<__half*>(dst), n);
    else
        cudaMemcpyAsync(dst, src, n * sizeof(float), cudaMemcpyDeviceToDevice, st);
}

}  // namespace ngprt_dev
