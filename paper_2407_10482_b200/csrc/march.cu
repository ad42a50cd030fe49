// march.cu — K1: ray generation, empty-space-skipping march, per-sample gather
// of baked coarse rows and fine hash features, attention fusion and
// front-to-back compositing with early stop. One thread per ray, 16x8 pixel
// tiles per 128-thread CTA.
//
// Built with -fmad=false: every float/double expression below rounds exactly
// where the reference's does. Reference citations are
// relative to /root/reference/proj/include/ngprt/.
#include "render.cuh"

namespace ngprt_dev {
namespace {

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
#pragma unroll
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
#pragma unroll
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

// to_grid_coord hash_grid.hpp:23-26; voxel_of occupancy.hpp:94-102
__device__ __forceinline__ float grid_coord(float x, int res) {
    return (x - (-1.0f)) * (float(res) / 2.0f);
}
__device__ __forceinline__ int voxel_1d(float x, int res) {
    int i = int(floorf(grid_coord(x, res)));
    return i < 0 ? 0 : (i > res - 1 ? res - 1 : i);
}

__device__ __forceinline__ bool occ_bit(const uint32_t* __restrict__ g, int res, int x, int y,
                                        int z) {
    const unsigned long long i =
        (unsigned long long)x + (unsigned long long)res * ((unsigned long long)y +
                                                           (unsigned long long)res * z);
    return (__ldg(g + (i >> 5)) >> (uint32_t(i) & 31u)) & 1u;
}

// voxel_exit_step, occupancy.hpp:238-255 (x = ray.at(t), not clamped)
__device__ __forceinline__ float voxel_exit_step(const Ray& r, float t, int res) {
    float t_exit = 3.402823466e38f;
#pragma unroll
    for (int a = 0; a < 3; ++a) {
        const float d = r.d[a];
        if (d == 0.0f) continue;
        const float xa = r.o[a] + d * t;
        const int v = voxel_1d(xa, res);
        const float lo = -1.0f + 2.0f * float(v) / float(res);
        const float hi = lo + 2.0f / float(res);
        const float bound = d > 0.0f ? hi : lo;
        const float tc = (bound - r.o[a]) / d;
        t_exit = (tc < t_exit) ? tc : t_exit;
    }
    float s = t_exit - t;
    if (!(s > 0.0f)) s = 0.0f;
    return s + 1e-6f;
}

// Stencil along one axis: base index and fractional offset (hash_grid.hpp:38-46).
__device__ __forceinline__ void stencil_axis(float x, int res, int& base, float& frac) {
    const float u = grid_coord(x, res);
    int i = int(floorf(u));
    i = i < res - 1 ? i : res - 1;
    i = i > 0 ? i : 0;
    base = i;
    frac = u - float(i);
}

// Row loads: N leading elements of a row, converted to f32 (exact).
template <int N, bool F16>
__device__ __forceinline__ void load_coarse_row(const void* __restrict__ base,
                                                unsigned long long row, float* out) {
    if constexpr (F16) {
        const uint4* p = reinterpret_cast<const uint4*>(base) + row * 2;
        const uint4 a = __ldg(p);
        const __half2* ha = reinterpret_cast<const __half2*>(&a);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(ha[i]);
            out[2 * i] = f.x;
            out[2 * i + 1] = f.y;
        }
        if constexpr (N > 8) {
            const uint4 b = __ldg(p + 1);
            const __half2* hb = reinterpret_cast<const __half2*>(&b);
#pragma unroll
            for (int i = 0; i < (N - 8) / 2; ++i) {
                const float2 f = __half22float2(hb[i]);
                out[8 + 2 * i] = f.x;
                out[9 + 2 * i] = f.y;
            }
        }
    } else {
        const float4* p = reinterpret_cast<const float4*>(base) + row * 4;
#pragma unroll
        for (int q = 0; q < (N + 3) / 4; ++q) {
            const float4 v = __ldg(p + q);
            out[4 * q] = v.x;
            if (4 * q + 1 < N) out[4 * q + 1] = v.y;
            if (4 * q + 2 < N) out[4 * q + 2] = v.z;
            if (4 * q + 3 < N) out[4 * q + 3] = v.w;
        }
    }
}

template <bool F16>
__device__ __forceinline__ void load_fine_row(const void* __restrict__ base,
                                              unsigned long long row, float* out) {
    if constexpr (F16) {
        const uint4 a = __ldg(reinterpret_cast<const uint4*>(base) + row);
        const __half2* h = reinterpret_cast<const __half2*>(&a);
#pragma unroll
        for (int i = 0; i < 4; ++i) {
            const float2 f = __half22float2(h[i]);
            out[2 * i] = f.x;
            out[2 * i + 1] = f.y;
        }
    } else {
        const float4* p = reinterpret_cast<const float4*>(base) + row * 2;
        const float4 a = __ldg(p), b = __ldg(p + 1);
        out[0] = a.x; out[1] = a.y; out[2] = a.z; out[3] = a.w;
        out[4] = b.x; out[5] = b.y; out[6] = b.z; out[7] = b.w;
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

// decode_point_baked (baking.hpp:68-91) + split_decoder_output (model.hpp:13-22)
// + level_masked_fine (fusion.hpp:198-209) + fuse (fusion.hpp:107-173).
template <int L, bool F16>
__device__ __forceinline__ void decode_point(const DevScene& sc, const float x[3], int keep_level,
                                             const unsigned long long* tab, float out[8]) {
    constexpr int W = 8 + 2 * L;
    // coarse: stencil at L_C, 8 corner rows, interpolation in corner order
    // k = 0..7 from a zero start (baking.hpp:72-78; absent corners are zero rows)
    float dec[W];
    {
        int cb[3];
        float cf[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) stencil_axis(x[a], sc.L_C, cb[a], cf[a]);
        const unsigned long long r1 = (unsigned long long)sc.L_C + 1;
        float rows[8][W];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const unsigned long long key =
                (unsigned long long)(cb[0] + (k & 1)) +
                r1 * ((unsigned long long)(cb[1] + ((k >> 1) & 1)) +
                      r1 * (unsigned long long)(cb[2] + (k >> 2)));
            load_coarse_row<W, F16>(sc.coarse, key, rows[k]);
        }
#pragma unroll
        for (int i = 0; i < W; ++i) dec[i] = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            const float wx = dx ? cf[0] : 1.0f - cf[0];
            const float wy = dy ? cf[1] : 1.0f - cf[1];
            const float wz = dz ? cf[2] : 1.0f - cf[2];
            const float wk = wx * wy * wz;
#pragma unroll
            for (int i = 0; i < W; ++i) dec[i] += wk * rows[k][i];
        }
    }
    // fine levels: stencil, hash, 8 rows, interpolation (hash_grid.hpp:97-106)
    float fine[L][8];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        int b[3];
        float f[3];
#pragma unroll
        for (int a = 0; a < 3; ++a) stencil_axis(x[a], sc.fine_res[l], b[a], f[a]);
        float frow[8][8];
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            const unsigned long long idx = fine_index(sc, l, b[0] + dx, b[1] + dy, b[2] + dz);
            load_fine_row<F16>(sc.fine[l], idx, frow[k]);
        }
#pragma unroll
        for (int c = 0; c < 8; ++c) fine[l][c] = 0.0f;
#pragma unroll
        for (int k = 0; k < 8; ++k) {
            const int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
            const float wx = dx ? f[0] : 1.0f - f[0];
            const float wy = dy ? f[1] : 1.0f - f[1];
            const float wz = dz ? f[2] : 1.0f - f[2];
            const float wk = wx * wy * wz;
#pragma unroll
            for (int c = 0; c < 8; ++c) fine[l][c] += wk * frow[k][c];
        }
    }
    if (keep_level > 0) {
#pragma unroll
        for (int l = 0; l < L; ++l)
            if (l + 1 != keep_level)
#pragma unroll
                for (int c = 1; c < 8; ++c) fine[l][c] = 0.0f;
    }
    // effective weights (fusion.hpp:107-137) and the weighted fuse (:143-154)
    float wo[L], wb[L];
    const int mode = sc.fusion;
#pragma unroll
    for (int l = 0; l < L; ++l) {
        if (mode == NGPRT_FUSION_SEPARATE_ATT_V) {
            wo[l] = activate_sigmoid(dec[8 + 2 * l], tab);
            wb[l] = activate_sigmoid(dec[9 + 2 * l], tab);
        } else if (mode == NGPRT_FUSION_SHARED_ATT_V) {
            wo[l] = wb[l] = activate_sigmoid(dec[8 + 2 * l], tab);
        } else if (mode == NGPRT_FUSION_SUM) {
            wo[l] = wb[l] = 1.0f;
        } else if (mode == NGPRT_FUSION_SHARED_ATT_INV) {
            wo[l] = wb[l] = sc.att_w[2 * l];
        } else {
            wo[l] = sc.att_w[2 * l];
            wb[l] = sc.att_w[2 * l + 1];
        }
    }
#pragma unroll
    for (int i = 0; i < 8; ++i) out[i] = dec[i];
#pragma unroll
    for (int l = 0; l < L; ++l) {
        out[0] += wo[l] * fine[l][0];
#pragma unroll
        for (int c = 1; c < 8; ++c) out[c] += wb[l] * fine[l][c];
    }
}

template <int L, bool F16>
__global__ void __launch_bounds__(kBlock) march_kernel(const DevScene sc, const MarchParams p) {
    __shared__ unsigned long long tab[32];
    load_exp_table(tab);
    __syncthreads();

    const int cam_i = blockIdx.z;
    const uint32_t px = blockIdx.x * kTileW + (threadIdx.x % kTileW);
    const uint32_t py = blockIdx.y * kTileH + (threadIdx.x / kTileW);
    if (px >= p.w || py >= p.h) return;
    const CamParams& cam = p.cams[cam_i];
    const size_t out_idx = (size_t(cam_i) * p.h + py) * p.w + px;

    uint32_t n_march = 0, n_occ = 0, n_occ_acc = 0, n_dist_acc = 0;
    float cd[3] = {0.f, 0.f, 0.f}, fs[4] = {0.f, 0.f, 0.f, 0.f}, T = 1.0f;
    Ray ray;
    const bool valid =
        generate_ray(cam, double(p.x0 + px) + 0.5, double(p.y0 + py) + 0.5, ray);
    float t0, t1;
    if (valid && clip_f(ray, t0, t1)) {
        const float step = p.step;
        const bool use_grid = p.use_grid && sc.dist != nullptr;
        float t = t0;
        // march, occupancy.hpp:310-324
        while (t < t1) {
            float x[3];
#pragma unroll
            for (int a = 0; a < 3; ++a) x[a] = clamp_ref(ray.o[a] + ray.d[a] * t, -1.0f, 1.0f);
            ++n_march;
            // occupancy_probe (:218-231): the 5 bit reads are independent, so
            // issue them together; count only up to the first empty level.
            bool bits[NGPRT_PYRAMID_LEVELS];
#pragma unroll
            for (int k = NGPRT_PYRAMID_LEVELS - 1; k >= 0; --k) {
                const int res = sc.occ_res[k];
                bits[k] = occ_bit(sc.occ[k], res, voxel_1d(x[0], res), voxel_1d(x[1], res),
                                  voxel_1d(x[2], res));
            }
            int exit_res = 0;
#pragma unroll
            for (int k = NGPRT_PYRAMID_LEVELS - 1; k >= 0; --k) {
                if (exit_res) continue;
                ++n_occ_acc;
                if (!bits[k]) exit_res = sc.occ_res[k];
            }
            if (!exit_res) {
                ++n_occ;
                float f[8];
                decode_point<L, F16>(sc, x, p.keep_level, tab, f);
                // composite, volume.hpp:61-70
                const float sigma = activate_density(f[0], tab);
                const float a = alpha_from_sigma(sigma, step, tab);
                const float w = a * T;
#pragma unroll
                for (int c = 0; c < 3; ++c) cd[c] += w * f[1 + c];
#pragma unroll
                for (int c = 0; c < 4; ++c) fs[c] += w * f[4 + c];
                T = T * (1.0f - a);
                if (p.early_stop && T < float(2e-3)) break;  // kEarlyStopTransmittance
                t += step;
            } else {
                // next_step, occupancy.hpp:261-276
                const float s_occ = voxel_exit_step(ray, t, exit_res);
                float s = s_occ;
                if (use_grid && exit_res < sc.dist_res) {
                    const int gr = sc.dist_res;
                    const int vx = voxel_1d(ray.o[0] + ray.d[0] * t, gr);
                    const int vy = voxel_1d(ray.o[1] + ray.d[1] * t, gr);
                    const int vz = voxel_1d(ray.o[2] + ray.d[2] * t, gr);
                    ++n_dist_acc;
                    const uint8_t g = __ldg(sc.dist + (size_t(vx) +
                                                       size_t(gr) * (size_t(vy) + size_t(gr) * vz)));
                    if (g > 0) {
                        const float s_dist = float(2.0 / gr) * float(g);
                        s = p.max_step_rule ? ((s_dist < s_occ) ? s_occ : s_dist) : s_dist;
                    }
                }
                t += s;
            }
        }
    }
    RayAcc r;
    r.a = make_float4(cd[0], cd[1], cd[2], T);
    r.b = make_float4(fs[0], fs[1], fs[2], fs[3]);
    r.c = make_float4(valid ? ray.d[0] : 0.f, valid ? ray.d[1] : 0.f, valid ? ray.d[2] : 0.f,
                      valid ? 1.f : 0.f);
    p.acc[out_idx] = r;
    if (p.stats) {
        ngprt_ray_stats st;
        st.marching = n_march;
        st.occupied = n_occ;
        st.occ_acc = n_occ_acc;
        st.dist_acc = n_dist_acc;
        p.stats[out_idx] = st;
    }
}

template <int L, bool F16>
void launch_t(const DevScene& sc, const MarchParams& p, cudaStream_t st) {
    dim3 grid((p.w + kTileW - 1) / kTileW, (p.h + kTileH - 1) / kTileH, p.n_cams);
    march_kernel<L, F16><<<grid, kBlock, 0, st>>>(sc, p);
}

}  // namespace

void launch_march(const DevScene& sc, const MarchParams& p, cudaStream_t st) {
    const bool f16 = sc.storage == NGPRT_STORAGE_F16;
    switch (sc.L) {
        case 1: f16 ? launch_t<1, true>(sc, p, st) : launch_t<1, false>(sc, p, st); break;
        case 2: f16 ? launch_t<2, true>(sc, p, st) : launch_t<2, false>(sc, p, st); break;
        case 3: f16 ? launch_t<3, true>(sc, p, st) : launch_t<3, false>(sc, p, st); break;
        default: f16 ? launch_t<4, true>(sc, p, st) : launch_t<4, false>(sc, p, st); break;
    }
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
