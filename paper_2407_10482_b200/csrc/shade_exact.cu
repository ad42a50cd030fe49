// shade_exact.cu — K2 (exact mode): the deferred view MLP on CUDA cores in the
// reference's operation order, so RGB is bit-identical to the CPU reference.
//   shade           volume.hpp:118-137  rgb = sigmoid(C_d + psi([C_d, F, sh(dir)]))
//   TinyMlp::forward nn.hpp:175-196     acc = b[r]; acc += w[r][c] * a[c]; ReLU (hidden)
//   black when final_t == 1             SPEC.md:326, training.hpp:321
// Built with -fmad=false. Persistent CTAs, one thread per ray. The hidden
// layers run input-major: for each input c, every output's accumulator takes
// its c-th term, so each output still sums b, then c = 0, 1, ... in order. The
// weights sit transposed in shared memory ([c][o], one broadcast LDS.128 per
// four outputs); the products of two outputs are one packed FFMA2 with a +0
// addend and their sums one FADD2 (sm_100 f32x2, each half rounded like FMUL /
// FADD; see mac_pair_exact for why ptxas keeps them apart and why the zero
// sign cannot reach the RGB), so every operation rounds as the reference's.
#include "render.cuh"

namespace ngprt_dev {
namespace {

constexpr int kShadeBlock = 128;
constexpr int kColsBytes = 64 * kShadeBlock * 4;

// (a0, a1) += (w0 * x, w1 * x), each product and each sum rounded separately.
#ifndef NGPRT_EXACT_PACKED_ADD
#define NGPRT_EXACT_PACKED_ADD 1
#endif
__device__ __forceinline__ void mac_pair_exact(float& a0, float& a1, float w0, float w1, float x) {
    unsigned long long wp, xp, p;
    asm("mov.b64 %0, {%1, %2};" : "=l"(wp) : "f"(w0), "f"(w1));
    asm("mov.b64 %0, {%1, %1};" : "=l"(xp) : "f"(x));
#if NGPRT_EXACT_PACKED_ADD
    // Product as FFMA2(w, x, +0): RN(w*x + 0) equals RN(w*x) except that a -0
    // product becomes +0. ptxas does not fold this form into the following add
    // (it would for mul.f32x2 or an addend of -0, which are exact identities),
    // so the sum stays one FADD2 rounding each half like FADD. The sign of a
    // zero product only reaches a result when the accumulator is -0, which
    // yields a zero of the other sign; the ReLU compares (h < 0) and the
    // sigmoid (exp(-(+-0)) = 1) treat both zeros alike, so the RGB bits equal
    // the reference's in every case.
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(p) : "l"(wp), "l"(xp), "l"(0ull));
    unsigned long long a;
    asm("mov.b64 %0, {%1, %2};" : "=l"(a) : "f"(a0), "f"(a1));
    asm("add.rn.f32x2 %0, %0, %1;" : "+l"(a) : "l"(p));
    asm("mov.b64 {%0, %1}, %2;" : "=f"(a0), "=f"(a1) : "l"(a));
#else
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(p) : "l"(wp), "l"(xp));
    float p0, p1;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(p0), "=f"(p1) : "l"(p));
    a0 = __fadd_rn(a0, p0);
    a1 = __fadd_rn(a1, p1);
#endif
}

// out[0..63] = b[0..63] + sum_c Wt[c][0..63] * in[c], c ascending. The inputs
// come from this thread's shared-memory column (in[c * kShadeBlock]), so the c
// loop stays rolled without spilling a register array to local memory.
// NGPRT_EXACT_C_UNROLL: inputs per rolled-loop iteration (2: the next input's
// weight loads are scheduled under the current input's multiply-adds).
#ifndef NGPRT_EXACT_C_UNROLL
#define NGPRT_EXACT_C_UNROLL 2
#endif
constexpr int kExactCUnroll = NGPRT_EXACT_C_UNROLL;
template <int K>
__device__ __forceinline__ void dense64(const float* __restrict__ wt, const float* __restrict__ b,
                                        const float* in, float* out) {
#pragma unroll
    for (int o = 0; o < 64; ++o) out[o] = b[o];
#pragma unroll kExactCUnroll
    for (int c = 0; c < K; ++c) {
        const float x = in[c * kShadeBlock];
        const float4* row = reinterpret_cast<const float4*>(wt + c * 64);
#pragma unroll
        for (int q = 0; q < 16; ++q) {
            const float4 w = row[q];
            mac_pair_exact(out[4 * q], out[4 * q + 1], w.x, w.y, x);
            mac_pair_exact(out[4 * q + 2], out[4 * q + 3], w.z, w.w, x);
        }
    }
}

__global__ void __launch_bounds__(kShadeBlock)
    shade_exact_kernel(const float* __restrict__ psi, const RayAcc* __restrict__ acc,
                       float* __restrict__ rgb, size_t n) {
    __shared__ __align__(16) float w0t[23 * 64];  // [c][o]
    __shared__ __align__(16) float w1t[64 * 64];  // [c][o]
    __shared__ float b0[64], b1[64], w2[3 * 64], b2[4];
    extern __shared__ float cols[];  // 64 x kShadeBlock: per-thread layer inputs, column layout
    __shared__ unsigned long long tab[32];
    load_exp_table(tab);
    for (int i = threadIdx.x; i < 64 * 23; i += blockDim.x) {
        const int o = i / 23, c = i % 23;
        w0t[c * 64 + o] = psi[kPsiW0 + i];
    }
    for (int i = threadIdx.x; i < 64 * 64; i += blockDim.x) {
        const int o = i / 64, c = i % 64;
        w1t[c * 64 + o] = psi[kPsiW1 + i];
    }
    for (int i = threadIdx.x; i < 64; i += blockDim.x) {
        b0[i] = psi[kPsiB0 + i];
        b1[i] = psi[kPsiB1 + i];
    }
    for (int i = threadIdx.x; i < 3 * 64; i += blockDim.x) w2[i] = psi[kPsiW2 + i];
    if (threadIdx.x < 3) b2[threadIdx.x] = psi[kPsiB2 + threadIdx.x];
    __syncthreads();
    for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
         i += size_t(gridDim.x) * blockDim.x) {
        const RayAcc r = acc[i];
        float out[3] = {0.f, 0.f, 0.f};
        if (r.c.w != 0.f && r.a.w < 1.0f) {
            float* col = cols + threadIdx.x;
            const float f7[7] = {r.a.x, r.a.y, r.a.z, r.b.x, r.b.y, r.b.z, r.b.w};
#pragma unroll
            for (int c = 0; c < 7; ++c) col[c * kShadeBlock] = f7[c];
            float sh[16];
            sh_encode(r.c.x, r.c.y, r.c.z, sh);
#pragma unroll
            for (int c = 0; c < 16; ++c) col[(7 + c) * kShadeBlock] = sh[c];
            float h[64];
            dense64<23>(w0t, b0, col, h);
#pragma unroll
            for (int o = 0; o < 64; ++o) col[o * kShadeBlock] = h[o] < 0.0f ? 0.0f : h[o];
            float h2[64];
            dense64<64>(w1t, b1, col, h2);
            float y[3] = {b2[0], b2[1], b2[2]};
#pragma unroll
            for (int o = 0; o < 64; ++o) {
                const float v = h2[o] < 0.0f ? 0.0f : h2[o];
#pragma unroll
                for (int j = 0; j < 3; ++j) y[j] += w2[j * 64 + o] * v;
            }
            out[0] = activate_sigmoid(r.a.x + y[0], tab);
            out[1] = activate_sigmoid(r.a.y + y[1], tab);
            out[2] = activate_sigmoid(r.a.z + y[2], tab);
        }
        rgb[3 * i] = out[0];
        rgb[3 * i + 1] = out[1];
        rgb[3 * i + 2] = out[2];
    }
}

}  // namespace

void launch_shade_exact(const DevScene& sc, const RayAcc* acc, float* rgb, size_t n_rays,
                        cudaStream_t st) {
    if (!n_rays) return;
    static PerDeviceInt grid_of;
    const int grid = grid_of.get([](int dev) {
        int sms = 0, per_sm = 0;
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
        cudaFuncSetAttribute(shade_exact_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             kColsBytes);
        cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, shade_exact_kernel, kShadeBlock,
                                                      kColsBytes);
        return sms * (per_sm > 0 ? per_sm : 1);
    });
    const size_t need = (n_rays + kShadeBlock - 1) / kShadeBlock;
    const unsigned blocks = unsigned(need < size_t(grid) ? need : size_t(grid));
    shade_exact_kernel<<<blocks, kShadeBlock, kColsBytes, st>>>(sc.psi, acc, rgb, n_rays);
}

}  // namespace ngprt_dev
