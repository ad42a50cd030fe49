// device_common.cuh — device-side building blocks shared by the render kernels.
//
// Parity contract: every translation unit that includes
// this header is compiled with -fmad=false, so plain `a * b + c` is two IEEE
// roundings exactly like the reference built for x86-64 (no FMA contraction).
// Where the reference itself fuses (glibc's expf, see below) we call __fma_rn.
#pragma once

#include <cuda_fp16.h>
#include <stdint.h>
#include <stdio.h>  // device printf of the NGPRT_DEBUG_BOUNDS checks

#include "ngprt_cuda.h"

namespace ngprt_dev {

// ---------------------------------------------------------------------------
// glibc 2.39 expf (sysdeps/ieee754/flt-32/e_expf.c, the FMA ifunc variant that
// x86-64 hosts with FMA+AVX2 select). The reference calls it through
// std::exp(float) in activate_density (nn.hpp:82), activate_sigmoid (nn.hpp:93)
// and alpha_from_sigma (volume.hpp:32). It is not correctly rounded, so CUDA's
// expf or (float)exp(double) would not reproduce the reference bit-for-bit.
// Constants were read from the host libm's __exp2f_data and the port is checked
// exhaustively against the host glibc (tests/test_expf.py).
// tab[i] = asuint64(2^(i/32)) - (i << 47)
// ---------------------------------------------------------------------------
__device__ __constant__ static const unsigned long long kExp2fTab[32] = {
    0x3ff0000000000000ull, 0x3fefd9b0d3158574ull, 0x3fefb5586cf9890full, 0x3fef9301d0125b51ull,
    0x3fef72b83c7d517bull, 0x3fef54873168b9aaull, 0x3fef387a6e756238ull, 0x3fef1e9df51fdee1ull,
    0x3fef06fe0a31b715ull, 0x3feef1a7373aa9cbull, 0x3feedea64c123422ull, 0x3feece086061892dull,
    0x3feebfdad5362a27ull, 0x3feeb42b569d4f82ull, 0x3feeab07dd485429ull, 0x3feea47eb03a5585ull,
    0x3feea09e667f3bcdull, 0x3fee9f75e8ec5f74ull, 0x3feea11473eb0187ull, 0x3feea589994cce13ull,
    0x3feeace5422aa0dbull, 0x3feeb737b0cdc5e5ull, 0x3feec49182a3f090ull, 0x3feed503b23e255dull,
    0x3feee89f995ad3adull, 0x3feeff76f2fb5e47ull, 0x3fef199bdd85529cull, 0x3fef3720dcef9069ull,
    0x3fef5818dcfba487ull, 0x3fef7c97337b9b5full, 0x3fefa4afa2a490daull, 0x3fefd0765b6e4540ull};

// The table lives in shared memory inside the kernels (divergent indices would
// serialise the constant cache); this overload takes it explicitly.
__device__ __forceinline__ float glibc_expf(float x, const unsigned long long* __restrict__ tab) {
    const double kInvLn2N = 0x1.71547652b82fep+5;  // 32/ln2
    const double kShift = 0x1.8p+52;
    const double kC0 = 0x1.c6af84b912394p-20, kC1 = 0x1.ebfce50fac4f3p-13,
                 kC2 = 0x1.62e42ff0c52d6p-6;
    const uint32_t ux = __float_as_uint(x);
    const uint32_t abstop = (ux >> 20) & 0x7ffu;
    if (abstop >= 0x42bu) {                     // |x| >= 88 or nan
        if (ux == 0xff800000u) return 0.0f;     // -inf
        if (abstop >= 0x7f8u) return x + x;     // inf / nan
        if (x > 0x1.62e42ep6f) return __int_as_float(0x7f800000);  // __math_oflowf
        if (x < -0x1.9fe368p6f) return 0.0f;    // __math_uflowf
    }
    const double xd = double(x);
    double kd = __fma_rn(kInvLn2N, xd, kShift);
    const unsigned long long ki = (unsigned long long)__double_as_longlong(kd);
    kd = __dsub_rn(kd, kShift);
    const double r = __fma_rn(kInvLn2N, xd, -kd);
    const unsigned long long t = tab[ki & 31ull] + (ki << 47);
    const double s = __longlong_as_double((long long)t);
    const double z = __fma_rn(kC0, r, kC1);
    const double r2 = __dmul_rn(r, r);
    double y = __fma_rn(kC2, r, 1.0);
    y = __fma_rn(z, r2, y);
    y = __dmul_rn(y, s);
    return __double2float_rn(y);
}

__device__ __forceinline__ void load_exp_table(unsigned long long* smem_tab) {
    for (int i = threadIdx.x; i < 32; i += blockDim.x) smem_tab[i] = kExp2fTab[i];
}

// activate_density nn.hpp:80-83, activate_sigmoid nn.hpp:91-94, alpha_from_sigma volume.hpp:30-33
__device__ __forceinline__ float clamp_ref(float v, float lo, float hi) {
    return v < lo ? lo : (v > hi ? hi : v);
}
__device__ __forceinline__ float activate_density(float pre, const unsigned long long* tab) {
    return glibc_expf(clamp_ref(pre, -15.0f, 15.0f), tab);
}
__device__ __forceinline__ float activate_sigmoid(float pre, const unsigned long long* tab) {
    return 1.0f / (1.0f + glibc_expf(-pre, tab));
}
__device__ __forceinline__ float alpha_from_sigma(float sigma, float delta,
                                                  const unsigned long long* tab) {
    return 1.0f - glibc_expf(-sigma * delta, tab);
}

// sh_encode, nn.hpp:107-132 (16 outputs, same per-term operation order)
__device__ __forceinline__ void sh_encode(float x, float y, float z, float* out) {
    const float xx = x * x, yy = y * y, zz = z * z;
    out[0] = 0.28209479177387814f;
    out[1] = 0.4886025119029199f * y;
    out[2] = 0.4886025119029199f * z;
    out[3] = 0.4886025119029199f * x;
    out[4] = 1.0925484305920792f * x * y;
    out[5] = 1.0925484305920792f * y * z;
    out[6] = 0.31539156525252005f * (3.0f * zz - 1.0f);
    out[7] = 1.0925484305920792f * x * z;
    out[8] = 0.5462742152960396f * (xx - yy);
    out[9] = 0.5900435899266435f * y * (3.0f * xx - yy);
    out[10] = 2.890611442640554f * x * y * z;
    out[11] = 0.4570457994644658f * y * (5.0f * zz - 1.0f);
    out[12] = 0.3731763325901154f * z * (5.0f * zz - 3.0f);
    out[13] = 0.4570457994644658f * x * (5.0f * zz - 1.0f);
    out[14] = 1.445305721320277f * z * (xx - yy);
    out[15] = 0.5900435899266435f * x * (xx - 3.0f * yy);
}

// ---------------------------------------------------------------------------
// Scene as seen by the kernels (built by ngprt_scene_create).
// ---------------------------------------------------------------------------
// Device-side bounds assertions on every gather and per-ray store
// (NGPRT_DEBUG_BOUNDS=1 build variant, tools/build_variant.py; compiled out
// otherwise). They stand in for compute-sanitizer, which this GPU pool does not
// allow: tests/test_gpu_bounds.py renders the parity cases with the variant.
#ifndef NGPRT_DEBUG_BOUNDS
#define NGPRT_DEBUG_BOUNDS 0
#endif
#if NGPRT_DEBUG_BOUNDS
#define NG_BOUNDS(cond)                                                                 \
    do {                                                                                  \
        if (!(cond)) {                                                                    \
            printf("ngprt bounds check failed: %s (%s:%d)\n", #cond, __FILE__, __LINE__); \
            __trap();                                                                     \
        }                                                                                 \
    } while (0)
#else
#define NG_BOUNDS(cond) \
    do {                \
    } while (0)
#endif

struct DevScene {
    int L;
    int L_C;
    int fusion;           // ngprt_fusion_tag
    int storage;          // NGPRT_STORAGE_F32 / F16
    int fine_res[NGPRT_MAX_FINE_LEVELS];
    unsigned long long fine_len[NGPRT_MAX_FINE_LEVELS];
    uint32_t fine_mask[NGPRT_MAX_FINE_LEVELS];  // len-1 when len is a power of two <= 2^32
    int fine_mode[NGPRT_MAX_FINE_LEVELS];       // 0 direct, 1 hashed pow2, 2 hashed generic
    const void* coarse;   // dense (L_C+1)^3 rows x 16 elements (absent corners = zero rows)
    // NGPRT_COARSE_CELLS (experiment): per coarse cell, its 8 corner rows' W fp16
    // values back to back (16 W bytes per cell, L_C^3 cells), or null
    const void* coarse_cells;
    const void* fine[NGPRT_MAX_FINE_LEVELS];    // table_len x 8 elements
    float att_w[2 * NGPRT_MAX_FINE_LEVELS];     // post-sigmoid global weights (Inv modes)
    int occ_res[NGPRT_PYRAMID_LEVELS];
    const uint32_t* occ[NGPRT_PYRAMID_LEVELS];  // u64 words viewed as little-endian u32
    int dist_res;
    const uint8_t* dist;
    const float* psi;     // packed f32 weights: W0 (64x23) b0 W1 (64x64) b1 W2 (3x64) b2
    const float* fmlp;    // MLP fusion {8L,64,8}: W0 (64x8L) b0 (64) W1 (8x64) b1 (8), or null

    // ---- derived constants (ngprt_scene_create); each equals the float the
    // reference computes at that point, so using them is bit-exact ----
    float occ_h0;                                   // float(r0)/2.0f (to_grid_coord scale)
    float lvl_two_over_res[NGPRT_PYRAMID_LEVELS];   // 2.0f/float(r_k)  (voxel_exit_step hi)
    float lvl_inv_res[NGPRT_PYRAMID_LEVELS];        // 1/r_k, exact when r_k is a power of two
    int occ_pow2;                                   // every r_k is a power of two
    // Probe code per level-1 voxel (r1^3 u16): bits 8..10 = e, the number of
    // pyramid levels 4..1 whose bit is set before the first clear one (e = 4:
    // all set, level 0 decides); bits 0..7 = the 8 level-0 child bits when
    // e == 4, else the distance value G (when dist_res == r1); bits 11..13 = the
    // exit level (e == 4 ? 0 : 4 - e), bit 14 = consult_mask at that level, bit 15
    // = (e == 4). One load answers occupancy_probe and the distance read of a
    // marching point.
    const uint16_t* probe;
    int dist_is_l1;                                 // dist_res == r1
    uint32_t consult_mask;                          // bit k: dist grid exists and r_k < dist_res
    float dist_h;                                   // float(dist_res)/2.0f
    float dist_vox;                                 // float(2.0/dist_res) (DistanceGrid::voxel_size)
    float coarse_h;                                 // float(L_C)/2.0f
    float fine_h[NGPRT_MAX_FINE_LEVELS];            // float(fine_res[l])/2.0f
    int coarse_u32;                                 // (L_C+1)^3 < 2^32: 32-bit corner keys
    int fast_decode;                                // coarse_u32 and every level pow2-hashed
};

constexpr int kPsiW0 = 0, kPsiB0 = 64 * 23, kPsiW1 = kPsiB0 + 64, kPsiB1 = kPsiW1 + 64 * 64,
              kPsiW2 = kPsiB1 + 64, kPsiB2 = kPsiW2 + 3 * 64, kPsiTotal = kPsiB2 + 3;

// Per-ray record written by the marcher for the deferred MLP (48 B).
struct RayAcc {
    float4 a;  // c_d.xyz, final_t
    float4 b;  // F[0..3]
    float4 c;  // dir.xyz, valid (1 = ray generated)
};

}  // namespace ngprt_dev
