// measure_peaks.cu — the bandwidth ceilings SURVEY.md §8(d) asks K1 to be
// reported against, measured on this B200 (MEASURED_PEAKS.json holds only the
// HBM copy bandwidth and the bf16 tensor throughput):
//   l2_read      streaming 16-B loads over a 64 MiB buffer (L2-resident)
//   l2_gather32  random 32-B sectors from a 64 MiB table (the fine tables' size)
//   l2_gather16  random 16-B rows from a 64 MiB table (one fp16 fine row)
//   hbm_gather32 random 32-B sectors from a 4 GiB table (the coarse grid's size)
//   hbm_read     streaming 16-B loads over 4 GiB
// Each kernel is timed with CUDA events after a warm-up, best of 5. Bytes are
// the useful bytes requested (32 or 16 per gather). Prints one JSON object.
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o measure_peaks measure_peaks.cu
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>

__device__ __forceinline__ uint32_t mix(uint32_t x) {  // cheap per-thread hash
    x ^= x >> 16;
    x *= 0x7feb352du;
    x ^= x >> 15;
    x *= 0x846ca68bu;
    x ^= x >> 16;
    return x;
}

__global__ void stream_read(const uint4* __restrict__ p, size_t n, size_t iters, uint4* sink) {
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (size_t it = 0; it < iters; ++it)
        for (size_t i = blockIdx.x * size_t(blockDim.x) + threadIdx.x; i < n;
             i += size_t(gridDim.x) * blockDim.x) {
            const uint4 v = __ldg(p + i);
            acc.x ^= v.x;
            acc.y ^= v.y;
            acc.z ^= v.z;
            acc.w ^= v.w;
        }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) *sink = acc;
}

// ROWB-byte random rows; every thread issues `per_thread` independent gathers
// (8 in flight at a time, like K1's eight corner rows).
template <int ROWB>
__global__ void gather(const uint4* __restrict__ p, uint32_t rows_mask, uint32_t per_thread,
                       uint4* sink) {
    const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
    uint32_t h = mix(tid * 0x9e3779b9u + 1u);
    uint4 acc = make_uint4(0, 0, 0, 0);
    for (uint32_t i = 0; i < per_thread; i += 8) {
        uint4 v[8][ROWB / 16];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            h = mix(h + uint32_t(k));
            const uint4* row = p + size_t(h & rows_mask) * (ROWB / 16);
#pragma unroll
            for (int q = 0; q < ROWB / 16; ++q) v[k][q] = __ldg(row + q);
        }
#pragma unroll
        for (int k = 0; k < 8; ++k)
#pragma unroll
            for (int q = 0; q < ROWB / 16; ++q) {
                acc.x ^= v[k][q].x;
                acc.y ^= v[k][q].y;
                acc.z ^= v[k][q].z;
                acc.w ^= v[k][q].w;
            }
    }
    if ((acc.x ^ acc.y ^ acc.z ^ acc.w) == 0x12345678u) *sink = acc;
}

template <class F>
static float best_ms(F&& launch) {
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    launch();
    cudaDeviceSynchronize();
    float best = 1e30f;
    for (int r = 0; r < 5; ++r) {
        cudaEventRecord(a);
        launch();
        cudaEventRecord(b);
        cudaEventSynchronize(b);
        float ms = 0.f;
        cudaEventElapsedTime(&ms, a, b);
        best = ms < best ? ms : best;
    }
    cudaEventDestroy(a);
    cudaEventDestroy(b);
    return best;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t small = size_t(64) << 20, big = size_t(4) << 30;
    uint4 *s = nullptr, *g = nullptr, *sink = nullptr;
    if (cudaMalloc(&s, small) != cudaSuccess || cudaMalloc(&g, big) != cudaSuccess ||
        cudaMalloc(&sink, 64) != cudaSuccess) {
        std::printf("{\"error\": \"cudaMalloc failed\"}\n");
        return 1;
    }
    cudaMemset(s, 1, small);
    cudaMemset(g, 2, big);
    const dim3 grid(sms * 8), block(256);
    const size_t threads = size_t(grid.x) * block.x;

    const size_t n_small = small / 16, iters = 20;
    const float l2_ms = best_ms([&] { stream_read<<<grid, block>>>(s, n_small, iters, sink); });
    const double l2_read = double(small) * iters / (l2_ms * 1e-3) / 1e9;

    const float hbm_ms = best_ms([&] { stream_read<<<grid, block>>>(g, big / 16, 1, sink); });
    const double hbm_read = double(big) / (hbm_ms * 1e-3) / 1e9;

    const uint32_t per = 256;
    const float g32s_ms = best_ms([&] { gather<32><<<grid, block>>>(s, uint32_t(small / 32 - 1), per, sink); });
    const double l2_g32 = double(threads) * per * 32 / (g32s_ms * 1e-3) / 1e9;
    const float g16s_ms = best_ms([&] { gather<16><<<grid, block>>>(s, uint32_t(small / 16 - 1), per, sink); });
    const double l2_g16 = double(threads) * per * 16 / (g16s_ms * 1e-3) / 1e9;
    const float g32b_ms = best_ms([&] { gather<32><<<grid, block>>>(g, uint32_t(big / 32 - 1), per, sink); });
    const double hbm_g32 = double(threads) * per * 32 / (g32b_ms * 1e-3) / 1e9;

    const cudaError_t e = cudaGetLastError();
    std::printf("{\"l2_read_gbs\": %.1f, \"l2_gather32_gbs\": %.1f, \"l2_gather16_gbs\": %.1f, "
                "\"hbm_gather32_gbs\": %.1f, \"hbm_read_gbs\": %.1f, \"sms\": %d, \"cuda\": \"%s\", "
                "\"method\": \"best of 5 CUDA-event timings; 64 MiB (L2-resident) and 4 GiB tables; "
                "random rows from a per-thread hash, 8 gathers in flight per thread; useful bytes only\"}\n",
                l2_read, l2_g32, l2_g16, hbm_g32, hbm_read, sms, cudaGetErrorString(e));
    return e == cudaSuccess ? 0 : 1;
}
