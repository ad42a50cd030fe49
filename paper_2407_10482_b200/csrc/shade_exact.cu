// shade_exact.cu — K2 (exact mode): the deferred view MLP on CUDA cores in the
// reference's operation order, so RGB is bit-identical to the CPU reference.
//   shade           volume.hpp:118-137  rgb = sigmoid(C_d + psi([C_d, F, sh(dir)]))
//   TinyMlp::forward nn.hpp:175-196     acc = b[r]; acc += w[r][c] * a[c]; ReLU (hidden)
//   black when final_t == 1             SPEC.md:326, training.hpp:321
// Built with -fmad=false. One thread per ray; weights broadcast from shared memory.
#include "render.cuh"

namespace ngprt_dev {
namespace {

constexpr int kShadeBlock = 128;

__global__ void __launch_bounds__(kShadeBlock)
    shade_exact_kernel(const float* __restrict__ psi, const RayAcc* __restrict__ acc,
                       float* __restrict__ rgb, size_t n) {
    __shared__ float w[kPsiTotal];
    __shared__ unsigned long long tab[32];
    load_exp_table(tab);
    for (int i = threadIdx.x; i < kPsiTotal; i += blockDim.x) w[i] = psi[i];
    __syncthreads();
    const size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x;
    if (i >= n) return;
    const RayAcc r = acc[i];
    float out[3] = {0.f, 0.f, 0.f};
    if (r.c.w != 0.f && r.a.w < 1.0f) {
        float in[23];
        in[0] = r.a.x; in[1] = r.a.y; in[2] = r.a.z;
        in[3] = r.b.x; in[4] = r.b.y; in[5] = r.b.z; in[6] = r.b.w;
        sh_encode(r.c.x, r.c.y, r.c.z, in + 7);
        float h1[64];
#pragma unroll 4
        for (int o = 0; o < 64; ++o) {
            float a = w[kPsiB0 + o];
            const float* wr = w + kPsiW0 + o * 23;
#pragma unroll
            for (int c = 0; c < 23; ++c) a += wr[c] * in[c];
            h1[o] = a < 0.0f ? 0.0f : a;
        }
        // Layer 2 row by row; layer 3 accumulates in the same c-order as the
        // reference's inner loop, so h2 never needs to be materialised.
        float y[3] = {w[kPsiB2], w[kPsiB2 + 1], w[kPsiB2 + 2]};
        for (int o = 0; o < 64; ++o) {
            float a = w[kPsiB1 + o];
            const float* wr = w + kPsiW1 + o * 64;
#pragma unroll
            for (int c = 0; c < 64; ++c) a += wr[c] * h1[c];
            const float h2 = a < 0.0f ? 0.0f : a;
#pragma unroll
            for (int j = 0; j < 3; ++j) y[j] += w[kPsiW2 + j * 64 + o] * h2;
        }
        out[0] = activate_sigmoid(r.a.x + y[0], tab);
        out[1] = activate_sigmoid(r.a.y + y[1], tab);
        out[2] = activate_sigmoid(r.a.z + y[2], tab);
    }
    rgb[3 * i] = out[0];
    rgb[3 * i + 1] = out[1];
    rgb[3 * i + 2] = out[2];
}

}  // namespace

void launch_shade_exact(const DevScene& sc, const RayAcc* acc, float* rgb, size_t n_rays,
                        cudaStream_t st) {
    if (!n_rays) return;
    const unsigned blocks = unsigned((n_rays + kShadeBlock - 1) / kShadeBlock);
    shade_exact_kernel<<<blocks, kShadeBlock, 0, st>>>(sc.psi, acc, rgb, n_rays);
}

}  // namespace ngprt_dev
