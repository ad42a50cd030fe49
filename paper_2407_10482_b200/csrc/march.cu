// march.cu — K1: ray generation, empty-space-skipping march, per-sample gather
// of baked coarse rows and fine hash features, attention fusion and
// front-to-back compositing with early stop.
//
// Execution model: persistent warps, one ray per lane. Rays come in 4x8 pixel
// tiles (kRayTileW x kRayTileH) from a global counter; a lane whose ray finishes is refilled from the
// warp's current tile. Lanes march independently, but a lane that reaches an
// occupied point parks there until enough lanes of the warp are parked
// (MarchParams::decode_min) or no lane can step: the expensive sample decode then runs
// with most lanes converged instead of serialising against cheap empty steps.
//
// Parity: built with -fmad=false and every float/double operation is the
// reference's, in its order. Restructurings that are
// exact by construction are documented inline: (1) pyramid voxel indices at
// level k are the level-0 index >> k (power-of-two scaling commutes with
// rounding), (2) division by a power-of-two resolution is multiplication by
// its exact reciprocal, (3) voxel_exit_step divides only for the axis with the
// smallest exact ratio, (4) the unclamped point's voxel equals the clamped
// point's. In tensor-MLP mode (FC) the colour-only channels use FMA and the
// beta sigmoids a fast exp; everything that reaches density, transmittance,
// early stop or the counters stays exact. Reference citations are relative to
// /root/reference/proj/include/ngprt/.
#include <cstdlib>

#include "render.cuh"

namespace ngprt_dev {
namespace {

constexpr unsigned kFull = 0xffffffffu;
// MarchParams::decode_min: parked lanes that trigger a warp-wide decode (default 4)
// MarchParams::step_burst: marching points a stepping lane takes per round (default 6)
// CTAs per SM the register allocation targets: 6 (80 registers, 24 warps) for
// L <= 2, 5 (96 registers) for L = 3, 4, whose wider decode would spill at 80.
// NGPRT_K1_MIN_BLOCKS overrides both.
// f32 storage (twice the gathered words per sample, fine level 0 gathered with the
// coarse rows) takes 4 (128 registers): 4.89 -> 4.76 ms at config 3 vs 5 CTAs
// without the fine prefetch.
#ifdef NGPRT_K1_MIN_BLOCKS
template <int L, bool F16> constexpr int kMinBlocks = NGPRT_K1_MIN_BLOCKS;
#else
template <int L, bool F16> constexpr int kMinBlocks = F16 ? (L <= 2 ? 6 : 5) : 4;
#endif

struct Ray {
    float o[3], d[3];
    float tn, tf;
};

// generate_rays<float>, scene.hpp:211-228: f64 direction, c2w_rotate (:203-206),
// normalized() (common.hpp:30-35), clip_to_roi<double> with t in [0, 1e9].
__device__ __forceinline__ bool generate_ray(const CamParams& c, double u, double v, Ray& r) {
    const double dcx = (u - c.cx) / c.fx, dcy = (v - c.cy) / c.fy, dcz = 1.0;
    double w[3];
    w[0] = c.m[0] * dcx + c.m[1] * dcy + c.m[2] * dcz;
    w[1] = c.m[4] * dcx + c.m[5] * dcy + c.m[6] * dcz;
    w[2] = c.m[8] * dcx + c.m[9] * dcy + c.m[10] * dcz;
    const double n = sqrt(w[0] * w[0] + w[1] * w[1] + w[2] * w[2]);
    w[0] = w[0] / n;
    w[1] = w[1] / n;
    w[2] = w[2] / n;
    const double o[3] = {c.m[3], c.m[7], c.m[11]};
    double t0 = 0.0, t1 = 1e9;
    for (int a = 0; a < 3; ++a) {
        if (w[a] == 0.0) {
            if (o[a] < -1.0 || o[a] > 1.0) return false;
            continue;
        }
        double ta = (-1.0 - o[a]) / w[a], tb = (1.0 - o[a]) / w[a];
        if (ta > tb) {
            const double tmp = ta;
            ta = tb;
            tb = tmp;
        }
        t0 = (t0 < ta) ? ta : t0;
        t1 = (tb < t1) ? tb : t1;
    }
    if (!(t0 < t1)) return false;
    for (int a = 0; a < 3; ++a) {
        r.o[a] = float(o[a]);
        r.d[a] = float(w[a]);
    }
    r.tn = float(t0 < 0.0 ? 0.0 : t0);
    r.tf = float(t1);
    return r.tn < r.tf;
}

// clip_to_roi<float>, occupancy.hpp:279-297
__device__ __forceinline__ bool clip_f(const Ray& r, float& t0, float& t1) {
    t0 = r.tn;
    t1 = r.tf;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float d = r.d[a], o = r.o[a];
        if (d == 0.0f) {
            if (o < -1.0f || o > 1.0f) return false;
            continue;
        }
        float ta = (-1.0f - o) / d, tb = (1.0f - o) / d;
        if (ta > tb) {
            const float tmp = ta;
            ta = tb;
            tb = tmp;
        }
        t0 = (t0 < ta) ? ta : t0;
        t1 = (tb < t1) ? tb : t1;
    }
    return t0 < t1;
}

// voxel_of along one axis (occupancy.hpp:94-102) with h = float(res)/2.0f,
// i.e. to_grid_coord (hash_grid.hpp:23-26) then floor and clamp.
__device__ __forceinline__ int voxel_1d(float x, float h, int res) {
    const int i = __float2int_rd((x - (-1.0f)) * h);  // == int(floor(u)) for finite u
    return i < 0 ? 0 : (i > res - 1 ? res - 1 : i);
}
// Same for a point already clamped to [-1, 1]: u = (x + 1) * h >= +0, so only
// the upper clamp (x == 1 -> u == res) can apply.
// NGPRT_MAGIC_FLOOR: floor of a u in [0, 2^23) as the low mantissa bits of
// RD(u + 2^23) (FADD.RM + IADD at full rate) instead of F2I / I2F conversions
// (quarter-rate pipe); the float of a clamped index the same way. Exact.
#ifndef NGPRT_MAGIC_FLOOR
#define NGPRT_MAGIC_FLOOR 0
#endif
constexpr float kTwo23 = 8388608.0f;
__device__ __forceinline__ int floor_nonneg(float u) {  // u in [0, 2^23)
#if NGPRT_MAGIC_FLOOR
    return __float_as_int(__fadd_rd(u, kTwo23)) - 0x4B000000;
#else
    return __float2int_rd(u);
#endif
}
__device__ __forceinline__ float float_of_index(int i) {  // i in [0, 2^23)
#if NGPRT_MAGIC_FLOOR
    return __int_as_float(i + 0x4B000000) - kTwo23;
#else
    return float(i);
#endif
}
__device__ __forceinline__ int voxel_1d_clamped(float x, float h, int res) {
    const int i = floor_nonneg((x - (-1.0f)) * h);  // x in [-1, 1]: u in [0, res]
    return i > res - 1 ? res - 1 : i;
}

// Stencil along one axis: base index and fractional offset (hash_grid.hpp:38-46).
__device__ __forceinline__ void stencil_axis(float x, float h, int res, int& base, float& frac) {
    const float u = (x - (-1.0f)) * h;
#if NGPRT_MAGIC_FLOOR
    // (u clamped to [0, 2^22] for the floor only: outside [0, res) the index
    // clamps to 0 or res - 1 either way; frac uses u itself)
    int i = floor_nonneg(fminf(fmaxf(u, 0.0f), 4194304.0f));
    i = i < res - 1 ? i : res - 1;
    base = i;
    frac = u - float_of_index(i);
#else
    int i = __float2int_rd(u);
    i = i < res - 1 ? i : res - 1;
    i = i > 0 ? i : 0;
    base = i;
    frac = u - float(i);
#endif
}

// L1 allocation policy of the fine-row and probe-code gathers (tuning;
// 0 default, 1 L1::no_allocate, 2 L1::evict_first, 3 L1::evict_last).
#ifndef NGPRT_FINE_L1
#define NGPRT_FINE_L1 0
#endif
#ifndef NGPRT_COARSE_L1
#define NGPRT_COARSE_L1 0
#endif
#ifndef NGPRT_PROBE_L1
#define NGPRT_PROBE_L1 0
#endif
#define NGPRT_L1Q_0 ""
#define NGPRT_L1Q_1 ".L1::no_allocate"
#define NGPRT_L1Q_2 ".L1::evict_first"
#define NGPRT_L1Q_3 ".L1::evict_last"
#define NGPRT_L1Q_(n) NGPRT_L1Q_##n
#define NGPRT_L1Q(n) NGPRT_L1Q_(n)
__device__ __forceinline__ uint4 ldg_fine(const uint4* p) {
#if NGPRT_FINE_L1 == 0
    return __ldg(p);
#else
    uint4 r;
    asm("ld.global.nc" NGPRT_L1Q(NGPRT_FINE_L1) ".v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
    return r;
#endif
}
__device__ __forceinline__ uint32_t ldg_probe(const uint16_t* p) {
#if NGPRT_PROBE_L1 == 0
    return __ldg(p);
#else
    unsigned short r;
    asm("ld.global.nc" NGPRT_L1Q(NGPRT_PROBE_L1) ".u16 %0, [%1];" : "=h"(r) : "l"(p));
    return r;
#endif
}

// One 32 B fp16 coarse row (one sector) in a single 256-bit load (sm_100
// ld.global.v8.b32 -> LDG.E.256). NGPRT_COARSE_L2_HINT selects the L2 eviction
// priority: 0 normal, 1 evict_first, 2 evict_last.
#ifndef NGPRT_COARSE_L2_HINT
#define NGPRT_COARSE_L2_HINT 0
#endif
__device__ __forceinline__ void ldg256(const void* p, uint32_t (&r)[8]) {
#if NGPRT_COARSE_L2_HINT == 1
    asm volatile("ld.global.nc.L2::evict_first.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#elif NGPRT_COARSE_L2_HINT == 2
    asm volatile("ld.global.nc.L2::evict_last.v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#else
    asm volatile("ld.global.nc" NGPRT_L1Q(NGPRT_COARSE_L1) ".v8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
#endif
                 : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]),
                   "=r"(r[6]), "=r"(r[7])
                 : "l"(p));
}

// The N leading words of an f32 coarse row (16 floats, 64 B = two sectors) with
// the fewest wide loads: 256 bits, then 128 / 64 as needed (N = 8 + 2L).
template <int N>
__device__ __forceinline__ void load_coarse_f32_raw(const void* __restrict__ base,
                                                    unsigned long long row, uint32_t* r) {
    const uint4* p = reinterpret_cast<const uint4*>(base) + row * 4;
    uint32_t a[8];
    ldg256(p, a);
#pragma unroll
    for (int i = 0; i < 8; ++i) r[i] = a[i];
    if constexpr (N > 12) {
        uint32_t b[8];
        ldg256(p + 2, b);
#pragma unroll
        for (int i = 0; i < N - 8; ++i) r[8 + i] = b[i];
    } else if constexpr (N > 8) {
        const uint4 b = __ldg(p + 2);
        r[8] = b.x; r[9] = b.y; r[10] = b.z; r[11] = b.w;
    }
}

// Row loads: N leading elements of a 16-element row, converted to f32 (exact).
template <int N, bool F16>
__device__ __forceinline__ void load_coarse_row(const void* __restrict__ base,
                                                unsigned long long row, float* out) {
    if constexpr (F16) {
        uint32_t r[8];
        ldg256(reinterpret_cast<const uint4*>(base) + row * 2, r);
#pragma unroll
        for (int i = 0; i < N / 2; ++i) {
            const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&r[i]));
            out[2 * i] = f.x;
            out[2 * i + 1] = f.y;
        }
    } else {
        uint32_t r[16];
        load_coarse_f32_raw<N>(base, row, r);
#pragma unroll
        for (int i = 0; i < N; ++i) out[i] = __uint_as_float(r[i]);
    }
}

template <bool F16>
__device__ __forceinline__ void load_fine_row(const void* __restrict__ base,
                                              unsigned long long row, float* out) {
    if constexpr (F16) {
        const uint4 a = ldg_fine(reinterpret_cast<const uint4*>(base) + row);
        const __half2* h = reinterpret_cast<const __half2*>(&a);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h[i]);
            out[2 * i] = f.x;
            out[2 * i + 1] = f.y;
        }
    } else {
        // an f32 row is 32 B: one sector, one 256-bit load
        uint32_t r[8];
        ldg256(reinterpret_cast<const uint4*>(base) + row * 2, r);
#pragma unroll
        for (int i = 0; i < 8; ++i) out[i] = __uint_as_float(r[i]);
    }
}

// The 8 fp16 corner rows of a power-of-two hashed fine level with x-adjacent
// pairs fetched together (NGPRT_FINE_PAIR). The x prime is 1 (hash_grid.hpp:8):
// for an even base x the corners x and x + 1 of one (y, z) hash to rows h and
// h ^ 1, the two halves of one 32 B sector, so one 256-bit load brings both
// (and the pair swaps when h is odd); an odd base x takes two 128-bit loads.
// Rows come out in corner order k, so the interpolation is unchanged.
// NGPRT_FINE_PAIR bit 0: the fine levels gathered with the coarse rows; bit 1:
// the levels gathered in their own round trip (fine_level).
#ifndef NGPRT_FINE_PAIR
#define NGPRT_FINE_PAIR 0
#endif
__device__ __forceinline__ void fine_rows_paired(const uint4* __restrict__ table, int bx,
                                                 const uint32_t hy[2], const uint32_t hz[2],
                                                 uint32_t mask, uint32_t (&rows)[8][4]) {
    const bool even = (bx & 1) == 0;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
        const uint32_t c = hy[j & 1] ^ hz[j >> 1];
        const uint32_t h0 = (uint32_t(bx) ^ c) & mask, h1 = (uint32_t(bx + 1) ^ c) & mask;
        uint32_t r[8];
        if (even) {
            ldg256(table + (h0 & ~1u), r);
        } else {
            const uint4 a = ldg_fine(table + h0), b = ldg_fine(table + h1);
            r[0] = a.x; r[1] = a.y; r[2] = a.z; r[3] = a.w;
            r[4] = b.x; r[5] = b.y; r[6] = b.z; r[7] = b.w;
        }
        const bool swap = even && (h0 & 1u);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            rows[2 * j][i] = swap ? r[4 + i] : r[i];
            rows[2 * j + 1][i] = swap ? r[i] : r[4 + i];
        }
    }
}

// HashLevel::hash_index, hash_grid.hpp:83-94 (primes :8-10)
__device__ __forceinline__ unsigned long long fine_index(const DevScene& sc, int l, int x, int y,
                                                         int z) {
    const int mode = sc.fine_mode[l];
    if (mode == 1) {  // power-of-two table: u64 mod 2^k == u32 wrap & mask
        return (uint32_t(x) ^ (uint32_t(y) * 2654435761u) ^ (uint32_t(z) * 805459861u)) &
               sc.fine_mask[l];
    }
    if (mode == 2) {
        const unsigned long long h = (unsigned long long)x ^
                                     (unsigned long long)y * 2654435761ull ^
                                     (unsigned long long)z * 805459861ull;
        return h % sc.fine_len[l];
    }
    const unsigned long long r1 = (unsigned long long)sc.fine_res[l] + 1;
    return (unsigned long long)x + r1 * ((unsigned long long)y + r1 * (unsigned long long)z);
}

// Multiply-accumulate of one channel: exact (separate f32 multiply and add,
// the reference's -ffp-contract=off rounding) or, for the colour channels in
// tensor-MLP mode (FC), one FMA. Channels that feed density, attention
// weights or transmittance are always exact, so marching, early stop and the
// per-ray counters are bit-identical in both modes.
// (`fma` is a compile-time constant at every call site after unrolling.)
__device__ __forceinline__ float mac(bool fma, float acc, float w, float v) {
    return fma ? __fmaf_rn(w, v, acc) : acc + w * v;
}

// Two exact channels (a0 += w0 * v0, a1 += w1 * v1, product and sum each
// rounded like the reference's FMUL and FADD) as two packed sm_100
// instructions. The product is FFMA2(w, v, +0): RN(w*v + 0) is RN(w*v) except
// that a -0 product becomes +0, and ptxas does not fold it into the add (it
// contracts mul.f32x2 + add.f32x2, or an addend of -0, into one FFMA2). The
// zero sign never shows: every accumulator here starts at +0 and a sum that
// starts at +0 is never -0 under round-to-nearest (+0 + -0 = +0, exact
// cancellation gives +0), so adding +0 instead of -0 leaves it unchanged.
#ifndef NGPRT_PACKED_EXACT
#define NGPRT_PACKED_EXACT 1
#endif
__device__ __forceinline__ void mac2x(float& a0, float& a1, float w0, float w1, float v0,
                                      float v1) {
#if NGPRT_PACKED_EXACT
    unsigned long long acc, v, ww, prod;
    asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(v0), "f"(v1));
    asm("mov.b64 %0, {%1, %2};" : "=l"(ww) : "f"(w0), "f"(w1));
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(prod) : "l"(ww), "l"(v), "l"(0ull));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(acc) : "l"(prod));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
#else
    a0 = mac(false, a0, w0, v0);
    a1 = mac(false, a1, w1, v1);
#endif
}

// A pair of channels: with fma (both channels FMA-allowed) one sm_100 FFMA2
// (packed f32x2; each half rounds exactly like a scalar FMA), else mac2x.
__device__ __forceinline__ void mac2(bool fma, float& a0, float& a1, float w, float v0, float v1) {
    if (fma) {
        unsigned long long acc, v, ww;
        asm("mov.b64 %0, {%1, %2};" : "=l"(acc) : "f"(a0), "f"(a1));
        asm("mov.b64 %0, {%1, %2};" : "=l"(v) : "f"(v0), "f"(v1));
        asm("mov.b64 %0, {%1, %1};" : "=l"(ww) : "f"(w));
        asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(ww), "l"(v));
        asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(acc));
    } else {
        mac2x(a0, a1, w, w, v0, v1);
    }
}

// NGPRT_FHFMA (tensor-MLP mode, fp16 rows): a pair of colour channels takes
// sm_100's mixed-precision FFMA (FHFMA: f32 += f16 x f16) straight on the raw
// half2 row word with the trilinear weight rounded to f16: no f16 -> f32
// conversions; the products are exact, so the only change is the weight's
// rounding (relative 2^-11). Exact channels keep the f32 path.
#ifndef NGPRT_FHFMA
#define NGPRT_FHFMA 0
#endif
__device__ __forceinline__ uint16_t weight_f16(float w) { return __half_as_ushort(__float2half_rn(w)); }
__device__ __forceinline__ void fhfma_pair(float& a0, float& a1, uint32_t raw, uint16_t w16) {
    uint16_t lo, hi;
    asm("mov.b32 {%0, %1}, %2;" : "=h"(lo), "=h"(hi) : "r"(raw));
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a0) : "h"(lo), "h"(w16));
    asm("fma.rn.f32.f16 %0, %1, %2, %0;" : "+f"(a1) : "h"(hi), "h"(w16));
}

// Coarse decoder channels that must stay exact: sigma_pre (0) and the omega
// logits (8 + 2l), which set the density fuse weights of the variant modes.
__device__ __forceinline__ constexpr bool exact_channel(int c) {
    return c == 0 || (c >= 8 && ((c - 8) & 1) == 0);
}

// Trilinear weights in corner order k (bit0 x, bit1 y, bit2 z): w_k = (wx*wy)*wz
// (hash_grid.hpp:50-54); the wx*wy products are shared, the values are identical.
// NGPRT_PACKED_WEIGHTS: the 12 products as 6 FMUL2 (each half rounds like FMUL;
// the products only feed multiplies, so nothing can contract them).
#ifndef NGPRT_PACKED_WEIGHTS
#define NGPRT_PACKED_WEIGHTS 1
#endif
__device__ __forceinline__ unsigned long long mul_f32x2(unsigned long long a, float b0, float b1) {
    unsigned long long b, r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(b) : "f"(b0), "f"(b1));
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(r) : "l"(a), "l"(b));
    return r;
}
__device__ __forceinline__ void corner_weights(const float f[3], float w[8]) {
    const float wx[2] = {1.0f - f[0], f[0]}, wy[2] = {1.0f - f[1], f[1]},
                wz[2] = {1.0f - f[2], f[2]};
#if NGPRT_PACKED_WEIGHTS
    unsigned long long x;
    asm("mov.b64 %0, {%1, %2};" : "=l"(x) : "f"(wx[0]), "f"(wx[1]));
    const unsigned long long a = mul_f32x2(x, wy[0], wy[0]);  // (wxy0, wxy1)
    const unsigned long long b = mul_f32x2(x, wy[1], wy[1]);  // (wxy2, wxy3)
    const unsigned long long p[4] = {mul_f32x2(a, wz[0], wz[0]), mul_f32x2(b, wz[0], wz[0]),
                                     mul_f32x2(a, wz[1], wz[1]), mul_f32x2(b, wz[1], wz[1])};
#pragma unroll
    for (int q = 0; q < 4; ++q)
        asm("mov.b64 {%0, %1}, %2;" : "=f"(w[2 * q]), "=f"(w[2 * q + 1]) : "l"(p[q]));
#else
    float wxy[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) wxy[j] = wx[j & 1] * wy[j >> 1];
#pragma unroll
    for (int k = 0; k < 8; ++k) w[k] = wxy[k & 3] * wz[k >> 2];
#endif
}

// Interpolate fine level l at x (hash_grid.hpp:97-106: out[c] = sum_k w_k row_k[c],
// corner order k = 0..7 from a zero start). Power-of-two hashed tables take the
// unrolled path; direct / generic-length levels a compact loop (rare).
template <bool F16, bool FC = false>
__device__ __forceinline__ void fine_level(const DevScene& sc, int l, const float x[3],
                                           float fine[8]) {
    int b[3];
    float f[3];
    const float h = sc.fine_h[l];
    const int res = sc.fine_res[l];
#pragma unroll
    for (int a = 0; a < 3; ++a) stencil_axis(x[a], h, res, b[a], f[a]);
    const void* table = sc.fine[l];
#pragma unroll
    for (int c = 0; c < 8; ++c) fine[c] = 0.0f;
    if (sc.fine_mode[l] == 1) {
        float w[8];
        corner_weights(f, w);
        const uint32_t mask = sc.fine_mask[l];
        const uint32_t hy[2] = {uint32_t(b[1]) * 2654435761u, uint32_t(b[1] + 1) * 2654435761u};
        const uint32_t hz[2] = {uint32_t(b[2]) * 805459861u, uint32_t(b[2] + 1) * 805459861u};
        if constexpr (F16 && FC && NGPRT_FHFMA) {
            uint4 raw[8];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t row = (uint32_t(b[0] + (k & 1)) ^ hy[(k >> 1) & 1] ^ hz[k >> 2]) & mask;
                NG_BOUNDS(row < sc.fine_len[l]);
                raw[k] = ldg_fine(reinterpret_cast<const uint4*>(table) + row);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const float2 v0 = __half22float2(*reinterpret_cast<const __half2*>(&raw[k].x));
                mac2x(fine[0], fine[1], w[k], w[k], v0.x, v0.y);
                const uint16_t w16 = weight_f16(w[k]);
                fhfma_pair(fine[2], fine[3], raw[k].y, w16);
                fhfma_pair(fine[4], fine[5], raw[k].z, w16);
                fhfma_pair(fine[6], fine[7], raw[k].w, w16);
            }
            return;
        }
        float frow[8][8];
#if NGPRT_FINE_PAIR & 2
        if constexpr (F16) {
            uint32_t raw[8][4];
            fine_rows_paired(reinterpret_cast<const uint4*>(table), b[0], hy, hz, mask, raw);
#pragma unroll
            for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int i = 0; i < 4; ++i) {
                    const float2 f2 = __half22float2(*reinterpret_cast<const __half2*>(&raw[k][i]));
                    frow[k][2 * i] = f2.x;
                    frow[k][2 * i + 1] = f2.y;
                }
        } else
#endif
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t row = (uint32_t(b[0] + (k & 1)) ^ hy[(k >> 1) & 1] ^ hz[k >> 2]) & mask;
            NG_BOUNDS(row < sc.fine_len[l]);
            load_fine_row<F16>(table, row, frow[k]);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            mac2x(fine[0], fine[1], w[k], w[k], frow[k][0], frow[k][1]);
#pragma unroll
            for (int c = 2; c < 8; c += 2)
                mac2(FC, fine[c], fine[c + 1], w[k], frow[k][c], frow[k][c + 1]);
        }
    } else {
#pragma unroll 1
        for (int k = 0; k < 8; ++k) {
            const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            const float wk = ((dx ? f[0] : 1.0f - f[0]) * (dy ? f[1] : 1.0f - f[1])) *
                             (dz ? f[2] : 1.0f - f[2]);
            float row[8];
            const unsigned long long fi = fine_index(sc, l, b[0] + dx, b[1] + dy, b[2] + dz);
            NG_BOUNDS(fi < sc.fine_len[l]);
            load_fine_row<F16>(table, fi, row);
#pragma unroll
            for (int c = 0; c < 8; ++c) fine[c] = mac(FC && c != 0, fine[c], wk, row[c]);
        }
    }
}

// decode_point_baked (baking.hpp:68-91) + split_decoder_output (model.hpp:13-22)
// + level_masked_fine (fusion.hpp:198-209) + fuse (fusion.hpp:107-173).
// The weighted fuse adds level l's contribution right after that level is
// interpolated; levels are visited in order, so every sum is formed in the
// reference's order. `scr` is this thread's column of a [rows][kBlock] shared
// scratch (element j at scr[j * kBlock], so a warp's accesses hit 32 banks).
// MLPF: the MLP-fusion ablation (fusion.hpp:162-171) instead of attention.
template <int L, bool F16, bool MLPF>
__device__ __forceinline__ void decode_point(const DevScene& sc, const float x[3], int keep_level,
                                             const unsigned long long* tab, float* scr,
                                             float out[8]) {
    constexpr int W = 8 + 2 * L;
    // coarse: stencil at L_C, 8 corner rows, interpolation in corner order
    // k = 0..7 from a zero start (baking.hpp:72-78; absent corners are zero rows)
    float dec[W];
    {
        int cb[3];
        float cf[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) stencil_axis(x[a], sc.coarse_h, sc.L_C, cb[a], cf[a]);
        float w[8];
        corner_weights(cf, w);
        const uint32_t r1 = uint32_t(sc.L_C) + 1;
#pragma unroll
        for (int i = 0; i < W; ++i) dec[i] = 0.0f;
        if (sc.coarse_u32) {
            const uint32_t key0 = uint32_t(cb[0]) + r1 * (uint32_t(cb[1]) + r1 * uint32_t(cb[2]));
            const uint32_t sy = r1, sz = r1 * r1;
            float rows[8][W];
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const uint32_t key = key0 + (k & 1) + ((k >> 1) & 1) * sy + (k >> 2) * sz;
                NG_BOUNDS(key < uint64_t(r1) * r1 * r1);
                load_coarse_row<W, F16>(sc.coarse, key, rows[k]);
            }
#pragma unroll
            for (int k = 0; k < 8; ++k)
#pragma unroll
                for (int i = 0; i < W; ++i) dec[i] += w[k] * rows[k][i];
        } else {
            const unsigned long long R1 = r1;
#pragma unroll 1
            for (int k = 0; k < 8; ++k) {
                const unsigned long long key =
                    (unsigned long long)(cb[0] + (k & 1)) +
                    R1 * ((unsigned long long)(cb[1] + ((k >> 1) & 1)) +
                          R1 * (unsigned long long)(cb[2] + (k >> 2)));
                float row[W];
                NG_BOUNDS(key < R1 * R1 * R1);
                load_coarse_row<W, F16>(sc.coarse, key, row);
                const float wk = (((k & 1) ? cf[0] : 1.0f - cf[0]) *
                                  (((k >> 1) & 1) ? cf[1] : 1.0f - cf[1])) *
                                 ((k >> 2) ? cf[2] : 1.0f - cf[2]);
#pragma unroll
                for (int i = 0; i < W; ++i) dec[i] += wk * row[i];
            }
        }
    }
    if constexpr (MLPF) {
        // fuse, MLP mode (fusion.hpp:162-171): concatenated (masked) fine features
        // through TinyMlp {8L, 64, 8} (nn.hpp:175-196), added to the coarse feature.
        constexpr int IN = 8 * L;
#pragma unroll 1
        for (int l = 0; l < L; ++l) {
            float fine[8];
            fine_level<F16>(sc, l, x, fine);
            if (keep_level > 0 && l + 1 != keep_level) {
#pragma unroll
                for (int c = 1; c < 8; ++c) fine[c] = 0.0f;
            }
#pragma unroll
            for (int c = 0; c < 8; ++c) scr[(8 * l + c) * kBlock] = fine[c];
        }
        float in[IN];
#pragma unroll
        for (int c = 0; c < IN; ++c) in[c] = scr[c * kBlock];
        const float* W0 = sc.fmlp;
        const float* B0 = W0 + 64 * IN;
        const float* W1 = B0 + 64;
        const float* B1 = W1 + 8 * 64;
        float hat[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) hat[j] = __ldg(B1 + j);
        // hidden unit by unit; the output layer accumulates in the reference's c-order
#pragma unroll 1
        for (int r = 0; r < 64; ++r) {
            float h = __ldg(B0 + r);
            const float4* wr = reinterpret_cast<const float4*>(W0 + r * IN);
#pragma unroll
            for (int q = 0; q < IN / 4; ++q) {
                const float4 wq = __ldg(wr + q);
                h += wq.x * in[4 * q];
                h += wq.y * in[4 * q + 1];
                h += wq.z * in[4 * q + 2];
                h += wq.w * in[4 * q + 3];
            }
            h = h < 0.0f ? 0.0f : h;
#pragma unroll
            for (int j = 0; j < 8; ++j) hat[j] += __ldg(W1 + j * 64 + r) * h;
        }
#pragma unroll
        for (int i = 0; i < 8; ++i) out[i] = dec[i] + hat[i];
        return;
    }
    // post-sigmoid attention (split_decoder_output, model.hpp:18-21) for the
    // spatially variant modes: one sigmoid loop over the 2L logits in scratch
    const int mode = sc.fusion;
    const bool variant = mode == NGPRT_FUSION_SEPARATE_ATT_V || mode == NGPRT_FUSION_SHARED_ATT_V;
    if (variant) {
#pragma unroll
        for (int j = 0; j < 2 * L; ++j) scr[j * kBlock] = dec[8 + j];
        const int jstep = mode == NGPRT_FUSION_SHARED_ATT_V ? 2 : 1;
        // two independent sigmoid chains per iteration (ILP across the expf latency)
#pragma unroll 1
        for (int j = 0; j < 2 * L; j += 2 * jstep) {
            const int j2 = j + jstep;
            const bool two = j2 < 2 * L;
            const float y0 = activate_sigmoid(scr[j * kBlock], tab);
            const float y1 = activate_sigmoid(two ? scr[j2 * kBlock] : 0.0f, tab);
            scr[j * kBlock] = y0;
            if (two) scr[j2 * kBlock] = y1;
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = dec[i];
    // fine levels, fused in order (fusion.hpp:143-154, effective_weights :107-137)
#pragma unroll 1
    for (int l = 0; l < L; ++l) {
        float fine[8];
        fine_level<F16>(sc, l, x, fine);
        if (keep_level > 0 && l + 1 != keep_level) {
#pragma unroll
            for (int c = 1; c < 8; ++c) fine[c] = 0.0f;
        }
        float wo, wb;
        if (variant) {
            wo = scr[2 * l * kBlock];
            wb = mode == NGPRT_FUSION_SEPARATE_ATT_V ? scr[(2 * l + 1) * kBlock] : wo;
        } else if (mode == NGPRT_FUSION_SUM) {
            wo = wb = 1.0f;
        } else {
            wo = sc.att_w[2 * l];
            wb = mode == NGPRT_FUSION_SHARED_ATT_INV ? wo : sc.att_w[2 * l + 1];
        }
        out[0] += wo * fine[0];
#pragma unroll
        for (int c = 1; c < 8; ++c) out[c] += wb * fine[c];
    }
}

// Fast-path decode (fp16 storage, power-of-two hashed fine levels, 32-bit
// coarse keys): the coarse rows and the rows of the first P fine levels are
// requested before any of them is consumed (one dependent gather round trip for
// them); the next A levels are requested with them too but land in shared
// memory (cp.async, no registers held); any further level is one round trip
// each. Arithmetic and its order are exactly decode_point's (same per-corner
// accumulation, same in-order fuse). At L <= 2 (6 CTAs per SM) level 1 takes
// its own round trip (A = 0): the 16 KB staging buffer per CTA costs more L1
// than the extra trip costs latency; at L = 3, 4 (5 CTAs) one level is staged.
#ifndef NGPRT_FINE_PREFETCH
#define NGPRT_FINE_PREFETCH 1
#endif
template <int L> constexpr int kFineP = NGPRT_FINE_PREFETCH < L ? NGPRT_FINE_PREFETCH : L;
#ifdef NGPRT_FINE_ASYNC_LEVELS
template <int L> constexpr int kFineAsync = NGPRT_FINE_ASYNC_LEVELS;
#else
template <int L> constexpr int kFineAsync = L <= 2 ? 0 : 1;
#endif
template <int L> constexpr int kFineA = (L - kFineP<L>) < kFineAsync<L> ? (L - kFineP<L>) : kFineAsync<L>;
// F16 = false: f32 storage (any scene whose values are not fp16-exact, e.g. a
// real bake or a reference .ngrt): the same arithmetic on f32 rows (a 64 B
// coarse row in a 256-bit + 128/256-bit load, a 32 B fine row in one 256-bit
// load); the rows are twice as wide, so the coarse rows take their own round
// trip, and NGPRT_F32_FINE_PREFETCH fine levels ride along (default 1).
#ifndef NGPRT_F32_FINE_PREFETCH
#define NGPRT_F32_FINE_PREFETCH 1
#endif
template <int L, bool FC, bool F16 = true>
__device__ __forceinline__ void decode_point_fast(const DevScene& sc, const float x[3],
                                                  int keep_level, const unsigned long long* tab,
                                                  float* scr, uint4* stage, float out[8]) {
    constexpr int W = 8 + 2 * L;
    constexpr int P = F16 ? kFineP<L> : (NGPRT_F32_FINE_PREFETCH < L ? NGPRT_F32_FINE_PREFETCH : L);
    // fine levels P .. P+A-1 go to shared memory with cp.async (no registers held
    // while in flight), issued together with the coarse and register-held rows
    constexpr int A = F16 ? kFineA<L> : 0;
#ifndef NGPRT_COARSE_FULL_ROW
#define NGPRT_COARSE_FULL_ROW 1
#endif
    // u32 words of a coarse row actually loaded (W <= 12: 128+64-bit loads, else one 256-bit)
#if defined(NGPRT_COARSE_CELLS) && NGPRT_COARSE_CELLS
    constexpr bool kCells = F16;  // fp16: the cell's 8 corner rows back to back (16 W bytes)
#else
    constexpr bool kCells = false;
#endif
    constexpr int CW = !F16 ? W : (kCells ? W / 2 : ((W <= 12 && !NGPRT_COARSE_FULL_ROW) ? 6 : 8));
    // ---- issue: coarse rows ----
    int cb[3];
    float cf[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) stencil_axis(x[a], sc.coarse_h, sc.L_C, cb[a], cf[a]);
    const uint32_t r1 = uint32_t(sc.L_C) + 1;
    const uint32_t key0 = uint32_t(cb[0]) + r1 * (uint32_t(cb[1]) + r1 * uint32_t(cb[2]));
    uint32_t craw[8][CW];
    if constexpr (kCells) {
        const uint32_t lc = uint32_t(sc.L_C);
        const uint32_t cell = uint32_t(cb[0]) + lc * (uint32_t(cb[1]) + lc * uint32_t(cb[2]));
        const uint4* rec = reinterpret_cast<const uint4*>(sc.coarse_cells) + size_t(cell) * W;
        uint32_t cw[W / 2][8];
#pragma unroll
        for (int q = 0; q < W / 2; ++q) ldg256(rec + 2 * q, cw[q]);
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int i = 0; i < W / 2; ++i) {
                const int wi = k * (W / 2) + i;
                craw[k][i] = cw[wi >> 3][wi & 7];
            }
    } else
#pragma unroll
    for (int k = 0; k < 8; ++k) {
        const uint32_t key = key0 + (k & 1) + ((k >> 1) & 1) * r1 + (k >> 2) * r1 * r1;
        NG_BOUNDS(key < uint64_t(r1) * r1 * r1);
        const uint4* p = reinterpret_cast<const uint4*>(sc.coarse) + size_t(key) * 2;
        if constexpr (!F16) {
            load_coarse_f32_raw<W>(sc.coarse, key, craw[k]);
        } else if constexpr (CW == 8) {
            uint32_t r[8];
            ldg256(p, r);
#pragma unroll
            for (int i = 0; i < 8; ++i) craw[k][i] = r[i];
        } else {
            const uint4 a = __ldg(p);
            const uint2 b = __ldg(reinterpret_cast<const uint2*>(p + 1));
            craw[k][0] = a.x; craw[k][1] = a.y; craw[k][2] = a.z; craw[k][3] = a.w;
            craw[k][4] = b.x; craw[k][5] = b.y;
        }
    }
    // ---- issue: fine levels P..P+A-1 -> shared memory (cp.async), weights kept ----
    float fa[A > 0 ? A : 1][3];
#pragma unroll
    for (int j = 0; j < A; ++j) {
        const int l = P + j;
        int b[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) stencil_axis(x[a], sc.fine_h[l], sc.fine_res[l], b[a], fa[j][a]);
        const uint32_t mask = sc.fine_mask[l];
        const uint32_t hy[2] = {uint32_t(b[1]) * 2654435761u, uint32_t(b[1] + 1) * 2654435761u};
        const uint32_t hz[2] = {uint32_t(b[2]) * 805459861u, uint32_t(b[2] + 1) * 805459861u};
        const uint4* table = reinterpret_cast<const uint4*>(sc.fine[l]);
        const uint32_t s0 = uint32_t(__cvta_generic_to_shared(stage + j * 8 * kBlock));
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t row = (uint32_t(b[0] + (k & 1)) ^ hy[(k >> 1) & 1] ^ hz[k >> 2]) & mask;
            NG_BOUNDS(row < sc.fine_len[l]);
            const uint4* src = table + row;
            asm volatile("cp.async.ca.shared.global [%0], [%1], 16;"
                         :: "r"(s0 + uint32_t(k * kBlock * 16)), "l"(src) : "memory");
        }
    }
    if constexpr (A > 0) asm volatile("cp.async.commit_group;" ::: "memory");
    // ---- issue: fine levels 0..P-1 ----
    uint32_t fraw[P > 0 ? P : 1][8][F16 ? 4 : 8];
    float ff[P > 0 ? P : 1][3];
#pragma unroll
    for (int l = 0; l < P; ++l) {
        int b[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) stencil_axis(x[a], sc.fine_h[l], sc.fine_res[l], b[a], ff[l][a]);
        const uint32_t mask = sc.fine_mask[l];
        const uint32_t hy[2] = {uint32_t(b[1]) * 2654435761u, uint32_t(b[1] + 1) * 2654435761u};
        const uint32_t hz[2] = {uint32_t(b[2]) * 805459861u, uint32_t(b[2] + 1) * 805459861u};
        const uint4* table = reinterpret_cast<const uint4*>(sc.fine[l]);
#if NGPRT_FINE_PAIR & 1
        if constexpr (F16) {
            fine_rows_paired(table, b[0], hy, hz, mask, fraw[l]);
            continue;
        }
#endif
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint32_t row = (uint32_t(b[0] + (k & 1)) ^ hy[(k >> 1) & 1] ^ hz[k >> 2]) & mask;
            NG_BOUNDS(row < sc.fine_len[l]);
            if constexpr (F16) {
                const uint4 v = ldg_fine(table + row);
                fraw[l][k][0] = v.x; fraw[l][k][1] = v.y; fraw[l][k][2] = v.z; fraw[l][k][3] = v.w;
            } else {
                ldg256(table + size_t(row) * 2, fraw[l][k]);
            }
        }
    }
    // ---- coarse interpolation (baking.hpp:72-78) ----
    float dec[W];
    {
        float w[8];
        corner_weights(cf, w);
#pragma unroll
        for (int i = 0; i < W; ++i) dec[i] = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int i = 0; i < W / 2; ++i) {
                const float2 v = F16 ? __half22float2(*reinterpret_cast<const __half2*>(&craw[k][i]))
                                     : make_float2(__uint_as_float(craw[k][2 * i]),
                                                   __uint_as_float(craw[k][2 * i + 1]));
                if (FC && F16 && NGPRT_FHFMA && !exact_channel(2 * i) && !exact_channel(2 * i + 1))
                    fhfma_pair(dec[2 * i], dec[2 * i + 1], craw[k][i], weight_f16(w[k]));
                else if (FC && !exact_channel(2 * i) && !exact_channel(2 * i + 1))
                    mac2(true, dec[2 * i], dec[2 * i + 1], w[k], v.x, v.y);
                else  // an exact channel's partner is exact too (one packed pair)
                    mac2x(dec[2 * i], dec[2 * i + 1], w[k], w[k], v.x, v.y);
            }
    }
    // ---- attention (split_decoder_output, model.hpp:18-21) ----
    const int mode = sc.fusion;
    const bool variant = mode == NGPRT_FUSION_SEPARATE_ATT_V || mode == NGPRT_FUSION_SHARED_ATT_V;
    if (variant) {
#pragma unroll
        for (int j = 0; j < 2 * L; ++j) scr[j * kBlock] = dec[8 + j];
        const int jstep = mode == NGPRT_FUSION_SHARED_ATT_V ? 2 : 1;
#pragma unroll 1
        for (int j = 0; j < 2 * L; j += 2 * jstep) {
            const int j2 = j + jstep;
            const bool two = j2 < 2 * L;
            const float y0 = activate_sigmoid(scr[j * kBlock], tab);
            float y1;
            if (FC && jstep == 1) {  // a beta logit: colour only, tensor mode -> fast sigmoid
                const float v = two ? scr[j2 * kBlock] : 0.0f;
                y1 = __fdividef(1.0f, 1.0f + __expf(-v));
            } else {
                y1 = activate_sigmoid(two ? scr[j2 * kBlock] : 0.0f, tab);
            }
            scr[j * kBlock] = y0;
            if (two) scr[j2 * kBlock] = y1;
        }
    }
    auto weights = [&](int l, float& wo, float& wb) {
        if (variant) {
            wo = scr[2 * l * kBlock];
            wb = mode == NGPRT_FUSION_SEPARATE_ATT_V ? scr[(2 * l + 1) * kBlock] : wo;
        } else if (mode == NGPRT_FUSION_SUM) {
            wo = wb = 1.0f;
        } else {
            wo = sc.att_w[2 * l];
            wb = mode == NGPRT_FUSION_SHARED_ATT_INV ? wo : sc.att_w[2 * l + 1];
        }
    };
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = dec[i];
    // ---- prefetched fine levels: interpolate (hash_grid.hpp:98-103) and fuse in order ----
#pragma unroll
    for (int l = 0; l < P; ++l) {
        float w[8];
        corner_weights(ff[l], w);
        float fine[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) fine[c] = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 v = F16 ? __half22float2(*reinterpret_cast<const __half2*>(&fraw[l][k][i]))
                                     : make_float2(__uint_as_float(fraw[l][k][2 * i]),
                                                   __uint_as_float(fraw[l][k][2 * i + 1]));
                if (FC && F16 && NGPRT_FHFMA && i != 0)
                    fhfma_pair(fine[2 * i], fine[2 * i + 1], fraw[l][k][i], weight_f16(w[k]));
                else if (FC && i != 0)
                    mac2(true, fine[2 * i], fine[2 * i + 1], w[k], v.x, v.y);
                else
                    mac2x(fine[2 * i], fine[2 * i + 1], w[k], w[k], v.x, v.y);
            }
        }
        if (keep_level > 0 && l + 1 != keep_level) {
#pragma unroll
            for (int c = 1; c < 8; ++c) fine[c] = 0.0f;
        }
        float wo, wb;
        weights(l, wo, wb);
        mac2x(out[0], out[1], wo, wb, fine[0], fine[1]);
#pragma unroll
        for (int c = 2; c < 8; c += 2) mac2(FC, out[c], out[c + 1], wb, fine[c], fine[c + 1]);
    }
    // ---- levels P..P+A-1 from shared memory ----
    if constexpr (A > 0) asm volatile("cp.async.wait_group 0;" ::: "memory");
#pragma unroll
    for (int j = 0; j < A; ++j) {
        const int l = P + j;
        float w[8];
        corner_weights(fa[j], w);
        float fine[8];
#pragma unroll
        for (int c = 0; c < 8; ++c) fine[c] = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const uint4 r = stage[(j * 8 + k) * kBlock];
            const __half2* h = reinterpret_cast<const __half2*>(&r);
#pragma unroll
            for (int i = 0; i < 4; ++i) {
                const float2 v = __half22float2(h[i]);
                if (FC && NGPRT_FHFMA && i != 0)
                    fhfma_pair(fine[2 * i], fine[2 * i + 1], (&r.x)[i], weight_f16(w[k]));
                else if (FC && i != 0)
                    mac2(true, fine[2 * i], fine[2 * i + 1], w[k], v.x, v.y);
                else
                    mac2x(fine[2 * i], fine[2 * i + 1], w[k], w[k], v.x, v.y);
            }
        }
        if (keep_level > 0 && l + 1 != keep_level) {
#pragma unroll
            for (int c = 1; c < 8; ++c) fine[c] = 0.0f;
        }
        float wo, wb;
        weights(l, wo, wb);
        mac2x(out[0], out[1], wo, wb, fine[0], fine[1]);
#pragma unroll
        for (int c = 2; c < 8; c += 2) mac2(FC, out[c], out[c + 1], wb, fine[c], fine[c + 1]);
    }
    // ---- remaining levels one round trip each ----
#pragma unroll 1
    for (int l = P + A; l < L; ++l) {
        float fine[8];
        fine_level<F16, FC>(sc, l, x, fine);
        if (keep_level > 0 && l + 1 != keep_level) {
#pragma unroll
            for (int c = 1; c < 8; ++c) fine[c] = 0.0f;
        }
        float wo, wb;
        weights(l, wo, wb);
        mac2x(out[0], out[1], wo, wb, fine[0], fine[1]);
#pragma unroll
        for (int c = 2; c < 8; c += 2) mac2(FC, out[c], out[c + 1], wb, fine[c], fine[c + 1]);
    }
}

// NGPRT_LANE_SMEM: a lane's parked sample position and colour accumulators
// (C_d, F) live in its shared-memory scratch column instead of registers (they
// are touched once per sample), which frees ~10 registers for the decode.
#ifndef NGPRT_LANE_SMEM
#define NGPRT_LANE_SMEM 1
#endif
constexpr bool kLaneSmem = NGPRT_LANE_SMEM != 0;
constexpr int kLaneRows = kLaneSmem ? 10 : 0;  // xc[3], cd[3], fs[4]
// Scratch-column row of lane field j (0..9) after `base` attention rows.
__device__ __forceinline__ float& lane_row(float* scr, int base, int j) { return scr[(base + j) * kBlock]; }

// voxel_exit_step's finiteness test (1: one per-ray flag for a zero or subnormal
// direction component, set in start_ray, plus the selected minimum; 0: every
// approximate ratio tested at every exit step)
#ifndef NGPRT_EXIT_FLAG
#define NGPRT_EXIT_FLAG 1
#endif
// Lane::out_idx bit 31 is that flag; pixel indices of one launch stay below 2^31
// (ngprt_render splits larger camera batches).
constexpr uint32_t kIdxMask = NGPRT_EXIT_FLAG ? 0x7fffffffu : 0xffffffffu;
// NGPRT_STREAM_HINTS (experiment): 1 = evict-first stores of the per-ray
// accumulators, 2 = evict-first loads of the K0 ray records.
#ifndef NGPRT_STREAM_HINTS
#define NGPRT_STREAM_HINTS 0
#endif
// NGPRT_TILE_STRIP (experiment): ray-tile order, see start_ray (0: row-major)
#ifndef NGPRT_TILE_STRIP
#define NGPRT_TILE_STRIP 0
#endif
// NGPRT_TWO_RAYS (experiment, march_kernel): two rays per lane; 2 also switches
// rays inside a step burst.
#ifndef NGPRT_TWO_RAYS
#define NGPRT_TWO_RAYS 0
#endif
// Per-lane ray state.
// NGPRT_PROBE_REUSE: a lane keeps the last probe code and its level-1 voxel and
// skips the load when the next marching point is in the same voxel (experiment).
#ifndef NGPRT_PROBE_REUSE
#define NGPRT_PROBE_REUSE 0
#endif
struct Lane {
    Ray ray;
    float t, t1;
    float xc[3];  // clamped sample position of a parked (pending) lane
    float cd[3], fs[4], T;
    uint32_t n_march, n_occ, n_occ_acc, n_dist;
    uint32_t out_idx;
#if NGPRT_PROBE_REUSE
    uint32_t last_pidx, last_code;  // probe code of the last marching point's level-1 voxel
#endif
    bool has_ray, pending;
};

// Compact sharded index -> (camera, window pixel); false for a padding slot
// (ngprt_render_opts.shard_*: local tile j is global tile rank + j * world).
__device__ __forceinline__ bool shard_pixel(const MarchParams& p, uint32_t idx, uint32_t& cam,
                                            uint32_t& px, uint32_t& py) {
    const uint32_t t2 = p.shard_tile * p.shard_tile, per_cam = p.shard_local * t2;
    cam = idx / per_cam;
    const uint32_t r = idx - cam * per_cam, j = r / t2, l = r - j * t2;
    const uint32_t T = p.shard_rank + j * p.shard_world;
    if (T >= p.shard_tiles) return false;
    px = (T % p.shard_tiles_x) * p.shard_tile + l % p.shard_tile;
    py = (T / p.shard_tiles_x) * p.shard_tile + l / p.shard_tile;
    return px < p.w && py < p.h;
}

__device__ __forceinline__ void write_result(const MarchParams& p, const Lane& s, bool valid,
                                             float* scr, int lb) {
    RayAcc r;
    if constexpr (kLaneSmem) {
        r.a = make_float4(lane_row(scr, lb, 3), lane_row(scr, lb, 4), lane_row(scr, lb, 5), s.T);
        r.b = make_float4(lane_row(scr, lb, 6), lane_row(scr, lb, 7), lane_row(scr, lb, 8),
                          lane_row(scr, lb, 9));
    } else {
        r.a = make_float4(s.cd[0], s.cd[1], s.cd[2], s.T);
        r.b = make_float4(s.fs[0], s.fs[1], s.fs[2], s.fs[3]);
    }
    r.c = make_float4(valid ? s.ray.d[0] : 0.f, valid ? s.ray.d[1] : 0.f,
                      valid ? s.ray.d[2] : 0.f, valid ? 1.f : 0.f);
    const uint32_t idx = s.out_idx & kIdxMask;
    NG_BOUNDS(idx < p.n_slots);
#if NGPRT_STREAM_HINTS & 1
    // the 48 B per-ray accumulator is read once, by K2: evict-first in L2 so it
    // does not push the gathered rows out
    __stcs(&p.acc[idx].a, r.a);
    __stcs(&p.acc[idx].b, r.b);
    __stcs(&p.acc[idx].c, r.c);
#else
    p.acc[idx] = r;
#endif
    if (p.stats) {
        ngprt_ray_stats st;
        st.marching = s.n_march;
        st.occupied = s.n_occ;
        st.occ_acc = s.n_occ_acc;
        st.dist_acc = s.n_dist;
        p.stats[idx] = st;
    }
}

// Start the ray of slot `slot` (0..31) of ray tile `tile` from the K0 ray
// buffer. Rays K0 already finished (missed the ROI) leave the lane idle.
__device__ __forceinline__ void start_ray(const MarchParams& p, uint32_t tile, uint32_t slot,
                                          Lane& s, float* scr, int lb) {
    const uint32_t cam = tile / p.tiles_per_cam, tt = tile % p.tiles_per_cam;
    s.has_ray = false;
    if (p.shard_world) {
        // sharded: ray tile tt = (local shard tile j, ray tile inside it); K0 has
        // already finished the padding pixels
        const uint32_t j = tt / p.shard_rt_per_tile, sub = tt % p.shard_rt_per_tile;
        const uint32_t lx = (sub % p.shard_rt_x) * kRayTileW + (slot % kRayTileW),
                       ly = (sub / p.shard_rt_x) * kRayTileH + (slot / kRayTileW);
        const uint32_t T = p.shard_rank + j * p.shard_world;
        if (T >= p.shard_tiles) return;
        const uint32_t px = (T % p.shard_tiles_x) * p.shard_tile + lx,
                       py = (T / p.shard_tiles_x) * p.shard_tile + ly;
        if (px >= p.w || py >= p.h) return;
        s.out_idx = ((cam * p.shard_local + j) * p.shard_tile + ly) * p.shard_tile + lx;
    } else {
#if NGPRT_TILE_STRIP
        // experiment: tiles column-major inside strips of NGPRT_TILE_STRIP tile rows,
        // so the tiles in flight cover a compact 2D region instead of a row band
        const uint32_t tiles_y = p.tiles_per_cam / p.tiles_x;
        const uint32_t strip = tt / (NGPRT_TILE_STRIP * p.tiles_x);
        const uint32_t r = tt - strip * NGPRT_TILE_STRIP * p.tiles_x;
        const uint32_t hs = min(uint32_t(NGPRT_TILE_STRIP), tiles_y - strip * NGPRT_TILE_STRIP);
        const uint32_t tx = r / hs, ty = strip * NGPRT_TILE_STRIP + r % hs;
        const uint32_t px = tx * kRayTileW + (slot % kRayTileW), py = ty * kRayTileH + (slot / kRayTileW);
#else
        const uint32_t px = (tt % p.tiles_x) * kRayTileW + (slot % kRayTileW),
                       py = (tt / p.tiles_x) * kRayTileH + (slot / kRayTileW);
#endif
        if (px >= p.w || py >= p.h) return;
        s.out_idx = (cam * p.h + py) * p.w + px;
    }
    NG_BOUNDS(s.out_idx < p.n_slots);
#if NGPRT_STREAM_HINTS & 2
    const float4 a = __ldcs(p.rays + 2 * size_t(s.out_idx));  // read once: evict-first
    const float4 b = __ldcs(p.rays + 2 * size_t(s.out_idx) + 1);
#else
    const float4 a = __ldg(p.rays + 2 * size_t(s.out_idx));
    const float4 b = __ldg(p.rays + 2 * size_t(s.out_idx) + 1);
#endif
    if (!(b.w >= 0.0f)) return;  // K0 wrote the result (generate_rays/clip_to_roi miss)
    s.ray.o[0] = a.x; s.ray.o[1] = a.y; s.ray.o[2] = a.z;
    s.ray.d[0] = b.x; s.ray.d[1] = b.y; s.ray.d[2] = b.z;
    s.t = a.w;
    s.t1 = b.w;
#if NGPRT_EXIT_FLAG
    // a zero or subnormal direction component sends every voxel_exit_step of
    // this ray to the exact all-axes path (flag in the pixel index's top bit)
    if (!(fabsf(b.x) >= 1.17549435e-38f && fabsf(b.y) >= 1.17549435e-38f &&
          fabsf(b.z) >= 1.17549435e-38f))
        s.out_idx |= ~kIdxMask;
#endif
    if constexpr (kLaneSmem) {
#pragma unroll
        for (int j = 3; j < 10; ++j) lane_row(scr, lb, j) = 0.f;
    } else {
        s.cd[0] = s.cd[1] = s.cd[2] = 0.f;
        s.fs[0] = s.fs[1] = s.fs[2] = s.fs[3] = 0.f;
    }
    s.T = 1.0f;
    s.n_march = s.n_occ = s.n_occ_acc = s.n_dist = 0;
#if NGPRT_PROBE_REUSE
    s.last_pidx = 0xffffffffu;
#endif
    s.pending = false;
    s.has_ray = true;
}

// Probe-code layout: x-major (default) or 4x4x4 bricks of level-1 voxels
// (128 B = one L1 line). Bricks measured neutral on B200, and x-major costs
// fewer index instructions per marching point.
#ifndef NGPRT_PROBE_BRICK
#define NGPRT_PROBE_BRICK 0
#endif
__device__ __forceinline__ uint32_t probe_index(uint32_t x, uint32_t y, uint32_t z, uint32_t r1) {
#if NGPRT_PROBE_BRICK
    const uint32_t rb = r1 >> 2;
    return (((x >> 2) + rb * ((y >> 2) + rb * (z >> 2))) << 6) | ((z & 3u) << 4) | ((y & 3u) << 2) | (x & 3u);
#else
    return x + r1 * (y + r1 * z);
#endif
}

// voxel_exit_step selection form (1: sign-bit bound offset and a two-level
// compare-and-select of the smallest ratio; 0: the earlier axis-index form)
#ifndef NGPRT_EXIT_SEL
#define NGPRT_EXIT_SEL 1
#endif
// Park-time L1 prefetch (NGPRT_PARK_PREFETCH bits: 1 coarse rows, 2 fine level 0,
// 4 fine level 1): a lane that reaches an occupied point requests its sample's
// rows into L1 with register-free prefetches, so the warp's later decode (when
// enough lanes have parked) hits L1 instead of waiting on L2.
#ifndef NGPRT_PARK_PREFETCH
#define NGPRT_PARK_PREFETCH 0
#endif
__device__ __forceinline__ void prefetch_l1(const void* p) {
    asm volatile("prefetch.global.L1 [%0];" ::"l"(p));
}
__device__ __forceinline__ void park_prefetch(const DevScene& sc, const float x[3]) {
#if NGPRT_PARK_PREFETCH
    if (!sc.fast_decode) return;
    const bool f16 = sc.storage == NGPRT_STORAGE_F16;
    if (NGPRT_PARK_PREFETCH & 1) {
        int cb[3];
        float cf[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) stencil_axis(x[a], sc.coarse_h, sc.L_C, cb[a], cf[a]);
        const uint32_t r1 = uint32_t(sc.L_C) + 1;
        const uint32_t key0 = uint32_t(cb[0]) + r1 * (uint32_t(cb[1]) + r1 * uint32_t(cb[2]));
        const char* base = static_cast<const char*>(sc.coarse);
        const size_t row_bytes = f16 ? 32 : 64;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            prefetch_l1(base + size_t(key0 + (k & 1) + ((k >> 1) & 1) * r1 + (k >> 2) * r1 * r1) * row_bytes);
    }
#pragma unroll
    for (int l = 0; l < 2; ++l) {
        if (!((NGPRT_PARK_PREFETCH >> (1 + l)) & 1) || l >= sc.L) continue;
        int b[3];
        float f[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) stencil_axis(x[a], sc.fine_h[l], sc.fine_res[l], b[a], f[a]);
        const uint32_t mask = sc.fine_mask[l];
        const uint32_t hy[2] = {uint32_t(b[1]) * 2654435761u, uint32_t(b[1] + 1) * 2654435761u};
        const uint32_t hz[2] = {uint32_t(b[2]) * 805459861u, uint32_t(b[2] + 1) * 805459861u};
        const char* table = static_cast<const char*>(sc.fine[l]);
        const size_t row_bytes = f16 ? 16 : 32;
#pragma unroll
        for (int k = 0; k < 8; ++k)
            prefetch_l1(table + size_t((uint32_t(b[0] + (k & 1)) ^ hy[(k >> 1) & 1] ^ hz[k >> 2]) & mask) * row_bytes);
    }
#else
    (void)sc;
    (void)x;
#endif
}

// One marching point (march, occupancy.hpp:310-324): probe (:218-231) via the
// per-level-1 probe code; occupied -> park for decode; empty -> next_step (:261-276).
// Returns false when the ray left the clip interval.
template <bool STATS>
__device__ __forceinline__ bool march_point(const DevScene& sc, const MarchParams& p, Lane& s,
                                            float* scr, int lb) {
    if (!(s.t < s.t1)) return false;
    float xu[3], xc[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        xu[a] = s.ray.o[a] + s.ray.d[a] * s.t;  // Ray::at (volume.hpp:19)
        xc[a] = fminf(fmaxf(xu[a], -1.0f), 1.0f);  // == clamp (common.hpp:94-97) for non-NaN
    }
    if constexpr (STATS) ++s.n_march;
    const int r0 = sc.occ_res[0], r1 = sc.occ_res[1];
    int i0[3];
#pragma unroll
    for (int a = 0; a < 3; ++a) i0[a] = voxel_1d_clamped(xc[a], sc.occ_h0, r0);
    // level-k voxel = level-0 voxel >> k (exact: r_k = r0 / 2^k)
    const uint32_t pidx = probe_index(uint32_t(i0[0] >> 1), uint32_t(i0[1] >> 1), uint32_t(i0[2] >> 1), uint32_t(r1));
    NG_BOUNDS(pidx < uint32_t(r1) * uint32_t(r1) * uint32_t(r1));
#if NGPRT_PROBE_REUSE
    // consecutive marching points inside one level-1 voxel share its probe code
    uint32_t code;
    if (pidx == s.last_pidx) {
        code = s.last_code;
    } else {
        code = ldg_probe(sc.probe + pidx);
        s.last_pidx = pidx;
        s.last_code = code;
    }
#else
    const uint32_t code = ldg_probe(sc.probe + pidx);
#endif
    // occupancy_probe counters: e + 1 levels read (5 when level 0 decides).
    // Written branch-free so every empty point reaches next_step on one path.
    if constexpr (STATS) s.n_occ_acc += ((code >> 8) & 7u) + 1u;
    // level-0 bit from the code's child byte (no second dependent load), gated
    // by the code's e == 4 flag
    const uint32_t child = uint32_t(i0[0] & 1) | (uint32_t(i0[1] & 1) << 1) | (uint32_t(i0[2] & 1) << 2);
    if ((code >> child) & (code >> 15) & 1u) {
        if constexpr (STATS) ++s.n_occ;
        s.pending = true;
        park_prefetch(sc, xc);
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            if constexpr (kLaneSmem) lane_row(scr, lb, a) = xc[a];
            else s.xc[a] = xc[a];
        }
        return true;
    }
    const int exit_k = int(code >> 11) & 7;  // e == 4 ? 0 : 4 - e
    // next_step (occupancy.hpp:261-276) on the unclamped point ray.at(t). Its
    // voxel_of clamps the index to [0, res-1], so the unclamped point's voxel is
    // the clamped point's: (x+1)*h < 0 <=> x < -1 and (x+1)*h >= res <=> x >= 1.
    const int* iu = i0;
    // res(exit level) < dist_res as a per-scene bit mask over the levels (no
    // per-lane indexed constant load: divergent exit levels would serialise it)
    uint32_t g = 0;
    const bool consult = p.use_grid && ((code >> 14) & 1u);
    if (consult) {
        if constexpr (STATS) ++s.n_dist;
        if (sc.dist_is_l1) {
            g = code & 0xffu;  // the probe code's own level-1 voxel (iu >> 1 == pidx's voxel)
        } else {
            const int gr = sc.dist_res;
            const int vx = voxel_1d_clamped(xc[0], sc.dist_h, gr),
                      vy = voxel_1d_clamped(xc[1], sc.dist_h, gr),
                      vz = voxel_1d_clamped(xc[2], sc.dist_h, gr);
            const size_t di = size_t(vx) + size_t(gr) * (size_t(vy) + size_t(gr) * vz);
            NG_BOUNDS(di < size_t(gr) * gr * gr);
            g = __ldg(sc.dist + di);
        }
    }
    float step;
    if (g > 0 && !p.max_step_rule) {
        // Eq. 9: a positive distance value replaces s_occ, which has no other use
        // and no side effect, so voxel_exit_step is skipped (same t sequence).
        step = sc.dist_vox * float(g);
    } else {
        // voxel_exit_step (occupancy.hpp:238-255): t_exit = min over axes of the
        // IEEE quotient (bound - o) / d. RN division is monotonic, so the min is the
        // quotient of the axis with the smallest exact ratio: an approximate ratio
        // (MUFU.RCP, a few ulp) picks it and one exact division evaluates it. Axes
        // within 2^-16 relative of the approximate minimum (near-ties, or anything
        // non-finite) are all evaluated exactly; the result is the reference's.
        constexpr float kBig = 3.402823466e38f;
        float num[3], q[3];
        bool finite = true;
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            const float d = s.ray.d[a];
            const int v = iu[a] >> exit_k;
            float bound;
            if (sc.occ_pow2) {
                // lo = -1 + 2v/res and hi = lo + 2/res are exact for a power-of-two res
                // (multiples of 2/res in [-1, 1]), so bound = -1 + (v + [d > 0]) * (2/res)
                // is one exactly-rounded FMA with the same value
                // 2/r_k = (2/r0) * 2^k: exponent arithmetic on the (normal) power of two
                const float two_over_res =
                    __int_as_float(__float_as_int(sc.lvl_two_over_res[0]) + (exit_k << 23));
#if NGPRT_EXIT_SEL
                // v + [d > 0] from the sign bit; a zero d (either sign) only reaches the
                // exact path below, which skips that axis, so its bound is never used
                bound = __fmaf_rn(float(v + 1 - int(__float_as_uint(d) >> 31)), two_over_res, -1.0f);
#else
                bound = __fmaf_rn(float(v + (d > 0.0f ? 1 : 0)), two_over_res, -1.0f);
#endif
            } else {
                const float lo = -1.0f + (2.0f * float(v)) / float(sc.occ_res[exit_k]);
                bound = d > 0.0f ? lo + sc.lvl_two_over_res[exit_k] : lo;
            }
            num[a] = bound - s.ray.o[a];
            float rd;
            asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(rd) : "f"(d));
            // d == 0: rcp.approx gives inf, so q is inf or NaN and the axis goes to the
            // exact path below, which skips it as the reference does
            q[a] = num[a] * rd;
#if !NGPRT_EXIT_FLAG
            finite = finite && fabsf(q[a]) < 3.0e38f;
#endif
        }
        // smallest approximate ratio, its axis, and the second smallest
#if NGPRT_EXIT_SEL
        // two compare-and-select levels carry the numerator and direction of the
        // smaller ratio along (no axis index). Only used when every q is finite, where
        // the comparisons agree with fminf / fmaxf.
        const bool p01 = q[0] <= q[1];
        const float m01 = p01 ? q[0] : q[1], x01 = p01 ? q[1] : q[0];
        const float n01 = p01 ? num[0] : num[1], d01 = p01 ? s.ray.d[0] : s.ray.d[1];
        const bool p2 = m01 <= q[2];
        const float qmin = p2 ? m01 : q[2], q2nd = p2 ? fminf(x01, q[2]) : m01;
#if NGPRT_EXIT_FLAG
        // every |d| >= FLT_MIN: each reciprocal is finite and nonzero and no q is NaN;
        // an overflowed q (|d| near FLT_MIN) is +-inf: -inf is caught here, +inf
        // only stands for a true ratio beyond FLT_MAX, which is never the minimum
        finite = !(s.out_idx & ~kIdxMask) && fabsf(qmin) < 3.0e38f;
#endif
        float t_exit = kBig;
        const bool tie = !finite || !(q2nd > qmin + (fabsf(qmin) * 1.52587890625e-5f + 1e-30f));
        if (!tie) {
            // finite ratios: some d != 0, so the division is the reference's minimum
            t_exit = (p2 ? n01 : num[2]) / (p2 ? d01 : s.ray.d[2]);
        } else {
#else
        const float m01 = fminf(q[0], q[1]), x01 = fmaxf(q[0], q[1]);
        const float qmin = fminf(m01, q[2]), q2nd = fminf(x01, fmaxf(m01, q[2]));
        const int amin = (q[0] <= q[1] && q[0] <= q[2]) ? 0 : (q[1] <= q[2] ? 1 : 2);
        float t_exit = kBig;
        const bool tie = !finite || !(q2nd > qmin + (fabsf(qmin) * 1.52587890625e-5f + 1e-30f));
        if (!tie) {
            if (qmin < kBig) {  // else every d == 0: t_exit stays max (the reference's start)
                const float dsel = amin == 0 ? s.ray.d[0] : (amin == 1 ? s.ray.d[1] : s.ray.d[2]);
                const float nsel = amin == 0 ? num[0] : (amin == 1 ? num[1] : num[2]);
                t_exit = nsel / dsel;
            }
        } else {
#endif  // near-tie or non-finite: every axis exactly, as the reference
#pragma unroll
            for (int a = 0; a < 3; ++a) {
                const float d = s.ray.d[a];
                if (d == 0.0f) continue;
                const float tc = num[a] / d;
                t_exit = (tc < t_exit) ? tc : t_exit;
            }
        }
        float sz = t_exit - s.t;
        if (!(sz > 0.0f)) sz = 0.0f;
        const float s_occ = sz + 1e-6f;
        step = s_occ;
        if (g > 0) {  // max_step_rule
            const float s_dist = sc.dist_vox * float(g);
            step = (s_dist < s_occ) ? s_occ : s_dist;
        }
    }
    s.t += step;
    return true;
}

// STATS = false (no per-ray counters requested): the counter updates are compiled out.
template <int L, bool F16, bool MLPF, bool FC, bool STATS>
__global__ void __launch_bounds__(kBlock, kMinBlocks<L, F16>) march_kernel(const DevScene sc,
                                                                   const MarchParams p) {
    __shared__ unsigned long long tab[32];
#ifndef NGPRT_SCRATCH_ROWS
#define NGPRT_SCRATCH_ROWS (2 * L)
#endif
    // 2L attention logits per thread (8L fine features in MLP fusion), then the
    // lane-state rows.
    constexpr int kAttRows = MLPF ? 8 * L : NGPRT_SCRATCH_ROWS;
    // NGPRT_TWO_RAYS: a second ray per lane (its lane rows, then its register
    // fields: o, d, t, t1, T, out_idx, 4 counters)
    constexpr int kAltRows = NGPRT_TWO_RAYS ? kLaneRows + 14 : 0;
    __shared__ float scratch[kBlock * (kAttRows + kLaneRows + kAltRows)];
    constexpr int lb = kAttRows;  // first lane-state row
    constexpr int kStageLv = (F16 && !MLPF) ? kFineA<L> : 0;
    __shared__ uint4 fstage[kStageLv > 0 ? kStageLv * 8 * kBlock : 1];  // cp.async fine rows
    load_exp_table(tab);
    __syncthreads();
    float* scr = scratch + threadIdx.x;  // element j at scr[j * kBlock]: conflict-free banks
    uint4* stage = fstage + (kStageLv > 0 ? threadIdx.x : 0);
    const uint32_t lane = threadIdx.x & 31u;
    const unsigned lt_mask = (1u << lane) - 1u;
    const uint32_t total_tiles = p.tiles_per_cam * uint32_t(p.n_cams);
    const float step = p.step;

    uint32_t tile = 0, tile_next_slot = 32;  // warp-uniform tile cursor
    bool fetch_done = false;                 // warp-uniform
    Lane s;
    s.has_ray = false;
    s.pending = false;

#if NGPRT_TWO_RAYS
    // Two rays per lane (experiment): the ray in registers is the current one;
    // the other's register fields sit in the lane's scratch rows at altb and
    // its lane rows at lb + kLaneRows * (1 - cur). A lane whose current ray is
    // parked steps its other ray, and a decode takes whichever ray is parked,
    // so fewer lanes idle in either phase. Each ray still marches, decodes and
    // composites in its own order, so results and counters are unchanged.
    constexpr int altb = lb + 2 * kLaneRows;
    int cur = 0;
    bool alt_has = false, alt_pending = false;
    auto swap_slot = [&]() {
        auto sw = [&](float& f, int j) {
            const float t = lane_row(scr, altb, j);
            lane_row(scr, altb, j) = f;
            f = t;
        };
        auto swu = [&](uint32_t& u, int j) {
            float f = __uint_as_float(u);
            sw(f, j);
            u = __float_as_uint(f);
        };
#pragma unroll
        for (int a = 0; a < 3; ++a) {
            sw(s.ray.o[a], a);
            sw(s.ray.d[a], 3 + a);
        }
        sw(s.t, 6);
        sw(s.t1, 7);
        sw(s.T, 8);
        swu(s.out_idx, 9);
        if constexpr (STATS) {
            swu(s.n_march, 10);
            swu(s.n_occ, 11);
            swu(s.n_occ_acc, 12);
            swu(s.n_dist, 13);
        }
        const bool h = s.has_ray, q = s.pending;
        s.has_ray = alt_has;
        s.pending = alt_pending;
        alt_has = h;
        alt_pending = q;
        cur ^= 1;
    };
    auto refill = [&]() {  // the current slot of every lane without a ray
        unsigned need = __ballot_sync(kFull, !s.has_ray);
        while (need && !fetch_done) {
            if (tile_next_slot == 32) {
                uint32_t nt = 0;
                if (lane == 0) nt = atomicAdd(p.work, 1u);
                nt = __shfl_sync(kFull, nt, 0);
                if (nt >= total_tiles) {
                    fetch_done = true;
                    break;
                }
                tile = nt;
                tile_next_slot = 0;
            }
            const uint32_t avail = 32u - tile_next_slot;
            const uint32_t take = min(uint32_t(__popc(need)), avail);
            const uint32_t rank = __popc(need & lt_mask);
            if (((need >> lane) & 1u) && rank < take)
                start_ray(p, tile, tile_next_slot + rank, s, scr, lb + cur * kLaneRows);
            tile_next_slot += take;
            need = __ballot_sync(kFull, !s.has_ray);
        }
    };
    while (true) {
        if (!s.has_ray && alt_has) swap_slot();
        refill();
        if (!fetch_done) {
            const bool want = s.has_ray && !alt_has;
            if (__ballot_sync(kFull, want)) {
                if (want) swap_slot();
                refill();
            }
        }
        const unsigned active = __ballot_sync(kFull, s.has_ray || alt_has);
        if (!active) {
            if (fetch_done) break;
            continue;
        }
        const bool cur_parked = s.has_ray && s.pending, alt_parked = alt_has && alt_pending;
        const bool cur_step = s.has_ray && !s.pending, alt_step = alt_has && !alt_pending;
        const unsigned parked = __ballot_sync(kFull, cur_parked || alt_parked);
        const unsigned stepping = __ballot_sync(kFull, cur_step || alt_step);
        if (parked && (__popc(parked) >= p.decode_min || stepping == 0)) {
            if (!cur_parked && alt_parked) swap_slot();
            if (s.has_ray && s.pending) {
                const int lbc = lb + cur * kLaneRows;
                float f[8];
                float xq[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) xq[a] = lane_row(scr, lbc, a);
                if constexpr (!MLPF) {
                    if (sc.fast_decode)
                        decode_point_fast<L, FC, F16>(sc, xq, p.keep_level, tab, scr, stage, f);
                    else
                        decode_point<L, F16, MLPF>(sc, xq, p.keep_level, tab, scr, f);
                } else {
                    decode_point<L, F16, MLPF>(sc, xq, p.keep_level, tab, scr, f);
                }
                const float sigma = activate_density(f[0], tab);
                const float a = alpha_from_sigma(sigma, step, tab);
                const float w = a * s.T;
                float c[7];
#pragma unroll
                for (int j = 0; j < 7; ++j) c[j] = lane_row(scr, lbc, 3 + j);
                c[0] = mac(FC, c[0], w, f[1]);
                mac2(FC, c[1], c[2], w, f[2], f[3]);
                mac2(FC, c[3], c[4], w, f[4], f[5]);
                mac2(FC, c[5], c[6], w, f[6], f[7]);
#pragma unroll
                for (int j = 0; j < 7; ++j) lane_row(scr, lbc, 3 + j) = c[j];
                s.T = s.T * (1.0f - a);
                s.pending = false;
                if (p.early_stop && s.T < float(2e-3)) {  // kEarlyStopTransmittance
                    write_result(p, s, true, scr, lbc);
                    s.has_ray = false;
                } else {
                    s.t += step;
                }
            }
        } else {
            if (!cur_step && alt_step) swap_slot();
            if (s.has_ray && !s.pending) {
#pragma unroll 1
                for (int it = 0; it < p.step_burst; ++it) {
                    const int lbc = lb + cur * kLaneRows;
                    if (!march_point<STATS>(sc, p, s, scr, lbc)) {
                        write_result(p, s, true, scr, lbc);
                        s.has_ray = false;
                        break;
                    }
                    if (s.pending) {
                        if (NGPRT_TWO_RAYS >= 2 && alt_has && !alt_pending) {
                            swap_slot();  // keep stepping with the other ray
                            continue;
                        }
                        break;
                    }
                }
            }
        }
    }
    return;
#endif
    while (true) {
        // ---- refill idle lanes from the warp's tile; fetch tiles as needed ----
        unsigned need = __ballot_sync(kFull, !s.has_ray);
        while (need && !fetch_done) {
            if (tile_next_slot == 32) {
                uint32_t nt = 0;
                if (lane == 0) nt = atomicAdd(p.work, 1u);
                nt = __shfl_sync(kFull, nt, 0);
                if (nt >= total_tiles) {
                    fetch_done = true;
                    break;
                }
                tile = nt;
                tile_next_slot = 0;
            }
            const uint32_t avail = 32u - tile_next_slot;
            const uint32_t take = min(uint32_t(__popc(need)), avail);
            const uint32_t rank = __popc(need & lt_mask);
            if (((need >> lane) & 1u) && rank < take) start_ray(p, tile, tile_next_slot + rank, s, scr, lb);
            tile_next_slot += take;
            need = __ballot_sync(kFull, !s.has_ray);
        }
        const unsigned active = __ballot_sync(kFull, s.has_ray);
        if (!active) {
            if (fetch_done) break;
            continue;
        }
        const unsigned parked = __ballot_sync(kFull, s.has_ray && s.pending);
        const unsigned stepping = active & ~parked;
        if (parked && (__popc(parked) >= p.decode_min || stepping == 0)) {
            // ---- decode phase: emit(t) of the canonical render_ray ----
            if (s.has_ray && s.pending) {
                float f[8];
                float xq[3];
#pragma unroll
                for (int a = 0; a < 3; ++a) xq[a] = kLaneSmem ? lane_row(scr, lb, a) : s.xc[a];
                if constexpr (!MLPF) {
                    if (sc.fast_decode)
                        decode_point_fast<L, FC, F16>(sc, xq, p.keep_level, tab, scr, stage, f);
                    else
                        decode_point<L, F16, MLPF>(sc, xq, p.keep_level, tab, scr, f);
                } else {
                    decode_point<L, F16, MLPF>(sc, xq, p.keep_level, tab, scr, f);
                }
                // composite, volume.hpp:61-70
                const float sigma = activate_density(f[0], tab);
                const float a = alpha_from_sigma(sigma, step, tab);
                const float w = a * s.T;
                if constexpr (kLaneSmem) {
                    float c[7];
#pragma unroll
                    for (int j = 0; j < 7; ++j) c[j] = lane_row(scr, lb, 3 + j);
                    c[0] = mac(FC, c[0], w, f[1]);
                    mac2(FC, c[1], c[2], w, f[2], f[3]);
                    mac2(FC, c[3], c[4], w, f[4], f[5]);
                    mac2(FC, c[5], c[6], w, f[6], f[7]);
#pragma unroll
                    for (int j = 0; j < 7; ++j) lane_row(scr, lb, 3 + j) = c[j];
                } else {
                    s.cd[0] = mac(FC, s.cd[0], w, f[1]);
                    mac2(FC, s.cd[1], s.cd[2], w, f[2], f[3]);
                    mac2(FC, s.fs[0], s.fs[1], w, f[4], f[5]);
                    mac2(FC, s.fs[2], s.fs[3], w, f[6], f[7]);
                }
                s.T = s.T * (1.0f - a);
                s.pending = false;
                if (p.early_stop && s.T < float(2e-3)) {  // kEarlyStopTransmittance
                    write_result(p, s, true, scr, lb);
                    s.has_ray = false;
                } else {
                    s.t += step;
                }
            }
        } else if (s.has_ray && !s.pending) {
            // ---- step phase: cheap empty-space marching ----
#pragma unroll 1
            for (int it = 0; it < p.step_burst; ++it) {
                if (!march_point<STATS>(sc, p, s, scr, lb)) {
                    write_result(p, s, true, scr, lb);
                    s.has_ray = false;
                    break;
                }
                if (s.pending) break;
            }
        }
    }
}

// K0: ray generation for every pixel of the window (generate_rays, scene.hpp:211-228,
// then clip_to_roi<float>, occupancy.hpp:308). Rays that miss are finished here
// (black, zero counters); the others are queued for K1 as (o, t0), (d, t1).
__global__ void __launch_bounds__(256) raygen_kernel(const MarchParams p) {
    uint32_t px, py, idx;
    int cam;
    if (p.shard_world) {
        // compact sharded index space (one thread per slot, padding included:
        // pixels past the window and a rank's missing last tile come out black)
        idx = blockIdx.x * 256 + threadIdx.x;
        if (idx >= uint32_t(p.n_cams) * p.shard_local * p.shard_tile * p.shard_tile) return;
        uint32_t c;
        const bool in = shard_pixel(p, idx, c, px, py);
        cam = int(c);
        if (!in) {
            const_cast<float4*>(p.rays)[2 * size_t(idx) + 1] = make_float4(0.f, 0.f, 0.f, -1.0f);
            RayAcc a;
            a.a = make_float4(0.f, 0.f, 0.f, 1.0f);
            a.b = make_float4(0.f, 0.f, 0.f, 0.f);
            a.c = make_float4(0.f, 0.f, 0.f, 0.f);
            p.acc[idx] = a;
            if (p.stats) p.stats[idx] = ngprt_ray_stats{0u, 0u, 0u, 0u};
            return;
        }
    } else {
        px = blockIdx.x * 32 + (threadIdx.x & 31);
        py = blockIdx.y * 8 + (threadIdx.x >> 5);
        cam = blockIdx.z;
        if (px >= p.w || py >= p.h) return;
        idx = (uint32_t(cam) * p.h + py) * p.w + px;
    }
    NG_BOUNDS(idx < p.n_slots);
    Ray r;
    const bool valid = generate_ray(p.cams[cam], double(p.x0 + px) + 0.5, double(p.y0 + py) + 0.5, r);
    float t0 = 0.f, t1 = -1.0f;
    const bool march = valid && clip_f(r, t0, t1);
    float4* out = const_cast<float4*>(p.rays) + 2 * size_t(idx);
    if (march) {
        out[0] = make_float4(r.o[0], r.o[1], r.o[2], t0);
        out[1] = make_float4(r.d[0], r.d[1], r.d[2], t1);
        return;
    }
    out[1] = make_float4(0.f, 0.f, 0.f, -1.0f);
    RayAcc a;
    a.a = make_float4(0.f, 0.f, 0.f, 1.0f);
    a.b = make_float4(0.f, 0.f, 0.f, 0.f);
    a.c = make_float4(valid ? r.d[0] : 0.f, valid ? r.d[1] : 0.f, valid ? r.d[2] : 0.f,
                      valid ? 1.f : 0.f);
    p.acc[idx] = a;
    if (p.stats) p.stats[idx] = ngprt_ray_stats{0u, 0u, 0u, 0u};
}

template <int L, bool F16, bool MLPF, bool FC = false, bool STATS = true>
int ctas_per_sm_t() {
    int n = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&n, march_kernel<L, F16, MLPF, FC, STATS>, kBlock, 0);
    return n > 0 ? n : 1;
}

template <int L, bool F16, bool MLPF, bool FC = false, bool STATS = true>
void launch_t(const DevScene& sc, const MarchParams& p, cudaStream_t st, cudaEvent_t between) {
    static PerDeviceInt grid_of;
    const int grid = grid_of.get([](int dev) {
        int sms = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        // NGPRT_K1_CARVEOUT=<percent>: shared-memory carveout hint for K1 (tuning only;
        // the driver's default, a 102 KB shared / 154 KB L1 split at 6 CTAs per SM, is
        // as fast as the 64 KB split, and a smaller L1 is much slower: DESIGN.md §5)
        if (const char* cv = getenv("NGPRT_K1_CARVEOUT"))
            cudaFuncSetAttribute(march_kernel<L, F16, MLPF, FC, STATS>,
                                 cudaFuncAttributePreferredSharedMemoryCarveout, atoi(cv));
        return sms * ctas_per_sm_t<L, F16, MLPF, FC, STATS>();
    });
    if (p.shard_world) {
        const uint32_t n = uint32_t(p.n_cams) * p.shard_local * p.shard_tile * p.shard_tile;
        raygen_kernel<<<(n + 255) / 256, 256, 0, st>>>(p);
    } else {
        raygen_kernel<<<dim3((p.w + 31) / 32, (p.h + 7) / 8, p.n_cams), 256, 0, st>>>(p);
    }
    if (between) cudaEventRecord(between, st);
    const uint32_t tiles = p.tiles_per_cam * uint32_t(p.n_cams);
    const uint32_t need = (tiles + 3) / 4;  // 4 warps per CTA
    march_kernel<L, F16, MLPF, FC, STATS><<<std::min<uint32_t>(grid, need), kBlock, 0, st>>>(sc, p);
}

template <int L>
void launch_l(const DevScene& sc, const MarchParams& p, cudaStream_t st, cudaEvent_t ev) {
    const bool f16 = sc.storage == NGPRT_STORAGE_F16, mlp = sc.fusion == NGPRT_FUSION_MLP;
    if (mlp) {
        f16 ? launch_t<L, true, true>(sc, p, st, ev) : launch_t<L, false, true>(sc, p, st, ev);
    } else {
        // FC (tensor-MLP mode colour FMA) needs the fast decode; STATS = false when
        // no per-ray counters are requested
        const bool fc = sc.fast_decode && p.fast_color;
        if (f16)
            fc ? (p.stats ? launch_t<L, true, false, true>(sc, p, st, ev)
                          : launch_t<L, true, false, true, false>(sc, p, st, ev))
               : (p.stats ? launch_t<L, true, false>(sc, p, st, ev)
                          : launch_t<L, true, false, false, false>(sc, p, st, ev));
        else
            fc ? (p.stats ? launch_t<L, false, false, true>(sc, p, st, ev)
                          : launch_t<L, false, false, true, false>(sc, p, st, ev))
               : (p.stats ? launch_t<L, false, false>(sc, p, st, ev)
                          : launch_t<L, false, false, false, false>(sc, p, st, ev));
    }
}

// Probe codes (see DevScene::probe).
__global__ void probe_code_kernel(const DevScene sc, uint16_t* __restrict__ out) {
    const int r1 = sc.occ_res[1];
    const size_t n = size_t(r1) * r1 * r1;
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const int x = int(i % r1), y = int((i / r1) % r1), z = int(i / (size_t(r1) * r1));
        int e = 0;
#pragma unroll
        for (int k = 4; k >= 1; --k) {
            const int r = sc.occ_res[k], sh = k - 1;
            const size_t b = size_t(x >> sh) + size_t(r) * (size_t(y >> sh) + size_t(r) * size_t(z >> sh));
            if (!((sc.occ[k][b >> 5] >> (b & 31)) & 1u)) break;
            ++e;
        }
        // Payload byte: the pyramid is an OR-reduction, so a level-1 voxel with
        // e == 4 is occupied (its distance value is 0) and one with e < 4 has 8
        // empty children. The byte therefore carries the 8 level-0 child bits
        // (bit c = child (c&1, c>>1&1, c>>2)) when e == 4, else the distance value.
        uint32_t payload;
        if (e == 4) {
            payload = 0;
            const int r0 = sc.occ_res[0];
#pragma unroll
            for (int c = 0; c < 8; ++c) {
                const size_t b = size_t(2 * x + (c & 1)) +
                                 size_t(r0) * (size_t(2 * y + ((c >> 1) & 1)) + size_t(r0) * size_t(2 * z + (c >> 2)));
                payload |= ((sc.occ[0][b >> 5] >> (b & 31)) & 1u) << c;
            }
        } else {
            payload = (sc.dist && sc.dist_is_l1) ? sc.dist[i] : 0u;
        }
        // decoded fields for the marcher: exit level, whether next_step consults
        // the distance grid at that level, and the e == 4 flag
        const uint32_t exit_k = e == 4 ? 0u : uint32_t(4 - e);
        const uint32_t consult = (sc.consult_mask >> exit_k) & 1u;
        out[probe_index(uint32_t(x), uint32_t(y), uint32_t(z), uint32_t(r1))] =
            uint16_t((uint32_t(e) << 8) | payload | (exit_k << 11) | (consult << 14) |
                     (uint32_t(e == 4) << 15));
    }
}

}  // namespace

void launch_march(const DevScene& sc, const MarchParams& p, cudaStream_t st, cudaEvent_t between) {
    switch (sc.L) {
        case 1: launch_l<1>(sc, p, st, between); break;
        case 2: launch_l<2>(sc, p, st, between); break;
        case 3: launch_l<3>(sc, p, st, between); break;
        default: launch_l<4>(sc, p, st, between); break;
    }
}

int march_ctas_per_sm(const DevScene& sc) {
    const bool f16 = sc.storage == NGPRT_STORAGE_F16;
    switch (sc.L) {
        case 1: return f16 ? ctas_per_sm_t<1, true, false>() : ctas_per_sm_t<1, false, false>();
        case 2: return f16 ? ctas_per_sm_t<2, true, false>() : ctas_per_sm_t<2, false, false>();
        case 3: return f16 ? ctas_per_sm_t<3, true, false>() : ctas_per_sm_t<3, false, false>();
        default: return f16 ? ctas_per_sm_t<4, true, false>() : ctas_per_sm_t<4, false, false>();
    }
}

void launch_probe_codes(const DevScene& sc, uint16_t* out, cudaStream_t st) {
    probe_code_kernel<<<148 * 8, 256, 0, st>>>(sc, out);
}

// ---------------------------------------------------------------------------
// Test hooks
// ---------------------------------------------------------------------------
namespace {
__global__ void expf_kernel(const float* x, float* y, size_t n) {
    __shared__ unsigned long long tab[32];
    load_exp_table(tab);
    __syncthreads();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        y[i] = glibc_expf(x[i], tab);
}
__global__ void expf_range_kernel(uint32_t first, size_t n, uint32_t* y) {
    __shared__ unsigned long long tab[32];
    load_exp_table(tab);
    __syncthreads();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        y[i] = __float_as_uint(glibc_expf(__uint_as_float(first + uint32_t(i)), tab));
}
// The marcher K1 runs (march_point, same code path and flags), one thread per
// given ray, with emit(t) always continuing: records every empty-skip segment
// (t, t + s) and every occupied sample t, as the reference's march() does with
// its skip_segments vector (occupancy.hpp:302-326), plus the MarchCounters.
__global__ void __launch_bounds__(kBlock) march_segments_kernel(
    const DevScene sc, const MarchParams p, const float* __restrict__ rays8, int n, int max_seg,
    float* __restrict__ seg, int* __restrict__ nseg, float* __restrict__ samples,
    int* __restrict__ nsmp, uint32_t* __restrict__ counters) {
    __shared__ float scratch[kBlock * (kLaneRows > 0 ? kLaneRows : 1)];
    float* scr = scratch + threadIdx.x;
    const int i = blockIdx.x * kBlock + threadIdx.x;
    if (i >= n) return;
    Ray r;
    for (int a = 0; a < 3; ++a) {
        r.o[a] = rays8[8 * i + a];
        r.d[a] = rays8[8 * i + 3 + a];
    }
    r.tn = rays8[8 * i + 6];
    r.tf = rays8[8 * i + 7];
    Lane s;
    s.ray = r;
    s.out_idx = 0;
#if NGPRT_EXIT_FLAG
    if (!(fabsf(r.d[0]) >= 1.17549435e-38f && fabsf(r.d[1]) >= 1.17549435e-38f &&
          fabsf(r.d[2]) >= 1.17549435e-38f))
        s.out_idx |= ~kIdxMask;
#endif
    s.n_march = s.n_occ = s.n_occ_acc = s.n_dist = 0;
#if NGPRT_PROBE_REUSE
    s.last_pidx = 0xffffffffu;
#endif
    s.pending = false;
    int ns = 0, nt = 0;
    float t0, t1;
    if (clip_f(r, t0, t1)) {  // march(): clip_to_roi<float>, occupancy.hpp:308
        s.t = t0;
        s.t1 = t1;
        while (true) {
            const float tb = s.t;
            if (!march_point<true>(sc, p, s, scr, 0)) break;
            if (s.pending) {
                if (nt < max_seg) samples[size_t(i) * max_seg + nt] = tb;
                ++nt;
                s.pending = false;
                s.t += p.step;
            } else {
                if (ns < max_seg) {
                    seg[(size_t(i) * max_seg + ns) * 2] = tb;
                    seg[(size_t(i) * max_seg + ns) * 2 + 1] = s.t;
                }
                ++ns;
            }
        }
    }
    nseg[i] = ns;
    nsmp[i] = nt;
    counters[4 * i] = s.n_march;
    counters[4 * i + 1] = s.n_occ;
    counters[4 * i + 2] = s.n_occ_acc;
    counters[4 * i + 3] = s.n_dist;
}

__global__ void hash_kernel(DevScene sc, const int32_t* c, size_t n, unsigned long long* out) {
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x)
        out[i] = fine_index(sc, 0, c[3 * i], c[3 * i + 1], c[3 * i + 2]);
}
}  // namespace

void launch_test_expf(const float* x, float* y, size_t n, cudaStream_t st) {
    expf_kernel<<<148 * 8, 256, 0, st>>>(x, y, n);
}
void launch_test_expf_range(uint32_t first, size_t n, uint32_t* y, cudaStream_t st) {
    expf_range_kernel<<<148 * 16, 256, 0, st>>>(first, n, y);
}
void launch_test_march_segments(const DevScene& sc, float step, int use_grid, int max_step_rule,
                                const float* rays8, int n, int max_seg, float* seg, int* nseg,
                                float* samples, int* nsmp, uint32_t* counters, cudaStream_t st) {
    MarchParams p{};
    p.step = step;
    p.use_grid = use_grid;
    p.max_step_rule = max_step_rule;
    march_segments_kernel<<<(n + kBlock - 1) / kBlock, kBlock, 0, st>>>(sc, p, rays8, n, max_seg, seg,
                                                                      nseg, samples, nsmp, counters);
}
void launch_test_hash(const DevScene& sc0, const int32_t* corners, size_t n, int res,
                      unsigned long long len, int mode, uint32_t mask, unsigned long long* out,
                      cudaStream_t st) {
    DevScene sc = sc0;
    sc.fine_res[0] = res;
    sc.fine_len[0] = len;
    sc.fine_mode[0] = mode;
    sc.fine_mask[0] = mask;
    hash_kernel<<<148 * 4, 256, 0, st>>>(sc, corners, n, out);
}

}  // namespace ngprt_dev
