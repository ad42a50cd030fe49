// ngprt_abi.cu — the extern "C" boundary (include/ngprt_cuda.h): scene upload
// and layout conversion, render dispatch, occupancy builders, error reporting.
// No exceptions cross this boundary; every failure returns a status and leaves
// a message for ngprt_last_error() (the reference throws, e.g. baking.hpp:396-405).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "render.cuh"

using namespace ngprt_dev;

namespace {

thread_local std::string g_err;

ngprt_status fail(ngprt_status s, const std::string& msg) {
    g_err = msg;
    return s;
}

#define NG_CUDA(call)                                                                   \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            return fail(e_ == cudaErrorMemoryAllocation ? NGPRT_ENOMEM : NGPRT_ECUDA,   \
                        std::string(#call) + ": " + cudaGetErrorString(e_));            \
        }                                                                               \
    } while (0)

bool fp16_exact(float v) {
    // f32 -> f16 (round to nearest even) -> f32 must be the identity.
    if (std::isnan(v)) return false;
    const float h = __half2float(__float2half_rn(v));
    return std::memcmp(&h, &v, 4) == 0;
}

float host_sigmoid(float x) { return 1.0f / (1.0f + std::exp(-x)); }  // nn.hpp:91-94 (glibc expf)

// Per-call scratch (renders, the distance transform) comes from the current
// device's stream-ordered pool; keep its memory mapped across synchronisations
// instead of trimming to zero (once per device).
void keep_pool_mapped() {
    static PerDeviceInt done;
    done.get([](int dev) {
        cudaMemPool_t pool;
        if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
            uint64_t keep = ~uint64_t(0);
            cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
        }
        return 1;
    });
}

}  // namespace

namespace ngprt_host {
void set_error(const std::string& msg) { g_err = msg; }  // used by the host-only units
}

struct ngprt_scene {
    int device = 0;
    DevScene ds{};
    std::vector<void*> allocs;
    void* psi_tc = nullptr;
    ShadeConsts shade_consts{};
    ngprt_scene_info info{};
    void* fine_block = nullptr;
    size_t fine_block_bytes = 0;
    // profiling events of the last profiled render: (before K1, after K1, after K2) per launch
    mutable std::mutex prof_mu;
    mutable std::vector<cudaEvent_t> prof_events;
    mutable int prof_launches = 0;
    // ngprt_render_host context: render + copy streams and device buffers, reused
    struct HostCtx {
        std::mutex mu;
        cudaStream_t render = nullptr, copy = nullptr;
        float* rgb = nullptr;
        size_t rgb_cap = 0;
        ngprt_ray_stats* stats = nullptr;
        size_t stats_cap = 0;
        std::vector<cudaEvent_t> band_done;
    };
    mutable HostCtx host;
    // ngprt_render_host_async: two frame slots (device outputs + completion
    // events), each with its own render stream (consecutive frames overlap: the
    // next frame's march starts in the SM slots the previous one's tail frees),
    // and one copy stream (frames reach the host in call order).
    struct AsyncCtx {
        std::mutex mu;
        cudaStream_t render[2] = {nullptr, nullptr}, copy = nullptr;
        struct Slot {
            float* rgb = nullptr;
            size_t rgb_cap = 0;
            ngprt_ray_stats* stats = nullptr;
            size_t stats_cap = 0;
            cudaEvent_t rendered = nullptr, copied = nullptr;
            bool busy = false;
        } slot[2];
        int next = 0;
    };
    mutable AsyncCtx async;

    ~ngprt_scene() {
        int prev = 0;
        cudaGetDevice(&prev);
        cudaSetDevice(device);
        if (host.render) cudaStreamSynchronize(host.render);
        if (host.copy) cudaStreamSynchronize(host.copy);
        for (cudaEvent_t e : host.band_done) cudaEventDestroy(e);
        if (host.render) cudaStreamDestroy(host.render);
        if (host.copy) cudaStreamDestroy(host.copy);
        if (host.rgb) cudaFree(host.rgb);
        if (host.stats) cudaFree(host.stats);
        for (cudaStream_t r : async.render)
            if (r) cudaStreamSynchronize(r);
        if (async.copy) cudaStreamSynchronize(async.copy);
        for (auto& sl : async.slot) {
            if (sl.rgb) cudaFree(sl.rgb);
            if (sl.stats) cudaFree(sl.stats);
            if (sl.rendered) cudaEventDestroy(sl.rendered);
            if (sl.copied) cudaEventDestroy(sl.copied);
        }
        for (cudaStream_t r : async.render)
            if (r) cudaStreamDestroy(r);
        if (async.copy) cudaStreamDestroy(async.copy);
        for (cudaEvent_t e : prof_events) cudaEventDestroy(e);
        // the fine tables' persisting L2 lines would otherwise outlive the scene
        // (normal-access writes cannot evict them)
        if (fine_block) cudaCtxResetPersistingL2Cache();
        for (void* p : allocs) cudaFree(p);
        cudaSetDevice(prev);
    }
    cudaEvent_t prof_event(size_t i) const {
        while (prof_events.size() <= i) {
            cudaEvent_t e;
            cudaEventCreate(&e);
            prof_events.push_back(e);
        }
        return prof_events[i];
    }
    template <class T>
    cudaError_t alloc(T** p, size_t bytes) {
        void* q = nullptr;
        cudaError_t e = cudaMalloc(&q, bytes ? bytes : 1);
        if (e == cudaSuccess) {
            allocs.push_back(q);
            info.device_bytes += bytes;
        }
        *p = static_cast<T*>(q);
        return e;
    }
};

extern "C" {

int ngprt_abi_version(void) { return NGPRT_ABI_VERSION; }

const char* ngprt_last_error(void) { return g_err.c_str(); }

ngprt_status ngprt_scene_create(const ngprt_scene_desc* d, int device, ngprt_scene** out) {
    const DeviceRestore keep;
    const NvtxRange range("ngprt_scene_create");
    if (!d || !out) return fail(NGPRT_EINVAL, "ngprt_scene_create: null argument");
    *out = nullptr;
    // --- validation (mirrors the reference's invariants) ---
    if (d->L < 1 || d->L > NGPRT_MAX_FINE_LEVELS)
        return fail(NGPRT_EINVAL, "L out of range (1..4; the reference accepts 2..4, baking.hpp:366)");
    if (d->L_C < 1) return fail(NGPRT_EINVAL, "L_C must be >= 1");
    if (d->fusion_tag > NGPRT_FUSION_MLP) return fail(NGPRT_EINVAL, "unknown fusion tag");
    if (d->fusion_tag == NGPRT_FUSION_MLP &&
        !(d->fusion_mlp_w[0] && d->fusion_mlp_w[1] && d->fusion_mlp_b[0] && d->fusion_mlp_b[1]))
        return fail(NGPRT_EINVAL, "fusion mode 'mlp' needs the {8L,64,8} fusion MLP (baking.hpp:482)");
    if ((d->fusion_tag == NGPRT_FUSION_SHARED_ATT_INV ||
         d->fusion_tag == NGPRT_FUSION_SEPARATE_ATT_INV) &&
        !d->att_globals)
        return fail(NGPRT_EINVAL, "invariant attention mode needs att_globals (baking.hpp:480)");
    if (d->occ_base_res < 16 || d->occ_base_res % 16)
        return fail(NGPRT_EINVAL, "occ_base_res must be a positive multiple of 16");
    if (d->occ_base_res > 1024) return fail(NGPRT_EUNSUPPORTED, "occ_base_res > 1024");
    if (!d->pyramid_words[0]) return fail(NGPRT_EINVAL, "pyramid level 0 is required");
    if (d->n_coarse && (!d->coarse_keys || !d->coarse_rows))
        return fail(NGPRT_EINVAL, "coarse keys/rows missing");
    for (int k = 0; k < 3; ++k)
        if (!d->psi_w[k] || !d->psi_b[k]) return fail(NGPRT_EINVAL, "psi weights missing");
    const int L = int(d->L);
    const int w = 8 + 2 * L;
    for (int l = 0; l < L; ++l) {
        if (!d->fine_tables[l] || d->fine_table_len[l] == 0)
            return fail(NGPRT_EINVAL, "fine table missing");
        if (d->fine_res[l] < 1) return fail(NGPRT_EINVAL, "fine resolution must be >= 1");
        if (!d->fine_hashed[l]) {
            const uint64_t r1 = uint64_t(d->fine_res[l]) + 1;
            if (r1 * r1 * r1 > d->fine_table_len[l])
                return fail(NGPRT_EINVAL, "direct-addressed fine level needs (res+1)^3 rows");
        }
    }
    const uint64_t r1c = uint64_t(d->L_C) + 1;
    const uint64_t n_corner = r1c * r1c * r1c;
    // Keys must be in range. A repeated key keeps its FIRST row, as the reference's
    // SparseCoarseGrid::add_row does (index.emplace ignores a second insert,
    // baking.hpp:33-38); later duplicates are dropped on the host so the device
    // scatter never writes one corner twice.
    std::vector<uint64_t> dedup_keys;
    std::vector<float> dedup_rows;
    const uint64_t* coarse_keys = d->coarse_keys;
    const float* coarse_rows = d->coarse_rows;
    uint64_t n_coarse = d->n_coarse;
    {
        std::vector<uint64_t> seen(d->n_coarse ? (n_corner + 63) / 64 : 0, 0);
        bool dup = false;
        for (uint64_t i = 0; i < d->n_coarse; ++i) {
            const uint64_t k = d->coarse_keys[i];
            if (k >= n_corner)
                return fail(NGPRT_EINVAL, "coarse key " + std::to_string(k) +
                                              " outside the (L_C+1)^3 corner grid");
            dup |= (seen[k >> 6] >> (k & 63)) & 1;
            seen[k >> 6] |= uint64_t(1) << (k & 63);
        }
        if (dup) {
            std::fill(seen.begin(), seen.end(), 0);
            for (uint64_t i = 0; i < d->n_coarse; ++i) {
                const uint64_t k = d->coarse_keys[i];
                if ((seen[k >> 6] >> (k & 63)) & 1) continue;
                seen[k >> 6] |= uint64_t(1) << (k & 63);
                dedup_keys.push_back(k);
                dedup_rows.insert(dedup_rows.end(), d->coarse_rows + i * w, d->coarse_rows + (i + 1) * w);
            }
            coarse_keys = dedup_keys.data();
            coarse_rows = dedup_rows.data();
            n_coarse = dedup_keys.size();
        }
    }
    if (d->dist_res) {
        bool ok = d->dist_values != nullptr;
        for (int k = 0; k < NGPRT_PYRAMID_LEVELS; ++k)
            ok |= (d->occ_base_res >> k) == d->dist_res;
        if (!ok) return fail(NGPRT_EINVAL, "dist_res matches no pyramid level and no values given");
    }

    int n_dev = 0;
    if (cudaGetDeviceCount(&n_dev) != cudaSuccess || n_dev == 0)
        return fail(NGPRT_ENODEV, "no CUDA device visible");
    if (device < 0 || device >= n_dev) return fail(NGPRT_EINVAL, "device index out of range");
    cudaDeviceProp prop;
    NG_CUDA(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10)
        return fail(NGPRT_ENODEV, std::string("this build targets sm_100a (B200); device is ") +
                                      prop.name);
    NG_CUDA(cudaSetDevice(device));
    keep_pool_mapped();

    // --- storage decision: fp16 only when lossless ---
    int storage = d->storage;
    if (const char* e = std::getenv("NGPRT_STORAGE"))  // tuning override: "f32" | "f16" | "auto"
        storage = std::strcmp(e, "f32") == 0 ? NGPRT_STORAGE_F32
                  : std::strcmp(e, "f16") == 0 ? NGPRT_STORAGE_F16 : storage;
    if (storage == NGPRT_STORAGE_AUTO) {
        bool exact = true;
        for (uint64_t i = 0; exact && i < n_coarse * uint64_t(w); ++i)
            exact = fp16_exact(coarse_rows[i]);
        for (int l = 0; exact && l < L; ++l)
            for (uint64_t i = 0; exact && i < d->fine_table_len[l] * 8; ++i)
                exact = fp16_exact(d->fine_tables[l][i]);
        storage = exact ? NGPRT_STORAGE_F16 : NGPRT_STORAGE_F32;
    }
    const bool f16 = storage == NGPRT_STORAGE_F16;
    const size_t esz = f16 ? 2 : 4;

    auto* s = new ngprt_scene;
    s->device = device;
    s->info.device = device;
    DevScene& ds = s->ds;
    ds.L = L;
    ds.L_C = int(d->L_C);
    ds.fusion = d->fusion_tag;
    ds.storage = storage;
    s->info.storage = uint8_t(storage);
    s->info.coarse_row_stride = 16;
    cudaStream_t st;
    if (cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking) != cudaSuccess) {
        delete s;
        return fail(NGPRT_ECUDA, "cudaStreamCreate failed");
    }
    auto cleanup = [&](ngprt_status status) {
        cudaStreamSynchronize(st);
        cudaStreamDestroy(st);
        if (status != NGPRT_OK) delete s;
        return status;
    };
#define NG_TRY(call)                                                                    \
    do {                                                                                \
        cudaError_t e_ = (call);                                                        \
        if (e_ != cudaSuccess) {                                                        \
            g_err = std::string(#call) + ": " + cudaGetErrorString(e_);                 \
            return cleanup(e_ == cudaErrorMemoryAllocation ? NGPRT_ENOMEM : NGPRT_ECUDA); \
        }                                                                               \
    } while (0)

    // --- coarse rows: dense (L_C+1)^3 x 16 grid; absent corners are zero rows ---
    {
        const size_t bytes = size_t(n_corner) * 16 * esz;
        void* dense;
        NG_TRY(s->alloc(&dense, bytes));
        NG_TRY(cudaMemsetAsync(dense, 0, bytes, st));
        s->info.coarse_bytes = bytes;
        if (n_coarse) {
            unsigned long long* dkeys;
            float* drows;
            NG_TRY(cudaMallocAsync(&dkeys, n_coarse * 8, st));
            NG_TRY(cudaMallocAsync(&drows, n_coarse * w * 4, st));
            NG_TRY(cudaMemcpyAsync(dkeys, coarse_keys, n_coarse * 8, cudaMemcpyHostToDevice, st));
            NG_TRY(cudaMemcpyAsync(drows, coarse_rows, n_coarse * w * 4, cudaMemcpyHostToDevice, st));
            launch_scatter_coarse(dkeys, drows, n_coarse, w, dense, f16, st);
            NG_TRY(cudaGetLastError());
            NG_TRY(cudaFreeAsync(dkeys, st));
            NG_TRY(cudaFreeAsync(drows, st));
        }
        ds.coarse = dense;
#ifdef NGPRT_COARSE_CELLS
        ds.coarse_cells = nullptr;
        if (f16 && (w % 2) == 0) {
            const size_t cb = size_t(d->L_C) * d->L_C * d->L_C * 16 * w;
            void* cells;
            NG_TRY(s->alloc(&cells, cb));
            launch_coarse_cells(dense, int(d->L_C), int(w), cells, st);
            NG_TRY(cudaGetLastError());
            ds.coarse_cells = cells;
        }
#endif
    }
    // --- fine tables: one contiguous block (one L2 access-policy window) ---
    {
        size_t total = 0;
        size_t offs[NGPRT_MAX_FINE_LEVELS];
        for (int l = 0; l < L; ++l) {
            offs[l] = total;
            total += size_t(d->fine_table_len[l]) * 8 * esz;
            total = (total + 255) & ~size_t(255);
        }
        char* block;
        NG_TRY(s->alloc(&block, total));
        s->fine_block = block;
        s->fine_block_bytes = total;
        s->info.fine_bytes = total;
        for (int l = 0; l < L; ++l) {
            const size_t n = size_t(d->fine_table_len[l]) * 8;
            float* tmp;
            NG_TRY(cudaMallocAsync(&tmp, n * 4, st));
            NG_TRY(cudaMemcpyAsync(tmp, d->fine_tables[l], n * 4, cudaMemcpyHostToDevice, st));
            launch_convert_fine(tmp, block + offs[l], n, f16, st);
            NG_TRY(cudaGetLastError());
            NG_TRY(cudaFreeAsync(tmp, st));
            ds.fine[l] = block + offs[l];
            ds.fine_res[l] = int(d->fine_res[l]);
            ds.fine_len[l] = d->fine_table_len[l];
            const uint64_t len = d->fine_table_len[l];
            if (!d->fine_hashed[l]) {
                ds.fine_mode[l] = 0;
            } else if ((len & (len - 1)) == 0 && len <= (uint64_t(1) << 32)) {
                ds.fine_mode[l] = 1;
                ds.fine_mask[l] = uint32_t(len - 1);
            } else {
                ds.fine_mode[l] = 2;
            }
        }
    }
    // --- occupancy pyramid (K3 for missing levels) ---
    {
        int res = int(d->occ_base_res);
        for (int k = 0; k < NGPRT_PYRAMID_LEVELS; ++k) {
            const int r = res >> k;
            const size_t words = (size_t(r) * r * r + 63) / 64;
            uint64_t* g;
            NG_TRY(s->alloc(&g, words * 8));
            s->info.pyramid_bytes += words * 8;
            if (k == 0 || d->pyramid_words[k]) {
                NG_TRY(cudaMemcpyAsync(g, d->pyramid_words[k], words * 8, cudaMemcpyHostToDevice, st));
            } else {
                NG_TRY(cudaMemsetAsync(g, 0, words * 8, st));
                launch_pyramid_level(ds.occ[k - 1], r * 2, reinterpret_cast<uint32_t*>(g), st);
                NG_TRY(cudaGetLastError());
            }
            ds.occ[k] = reinterpret_cast<const uint32_t*>(g);
            ds.occ_res[k] = r;
            s->info.dev_pyramid[k] = g;
        }
    }
    // --- distance grid (K4 when not supplied) ---
    if (d->dist_res) {
        const size_t r = d->dist_res, n = r * r * r;
        uint8_t* g;
        NG_TRY(s->alloc(&g, n));
        s->info.dist_bytes = n;
        if (d->dist_values) {
            NG_TRY(cudaMemcpyAsync(g, d->dist_values, n, cudaMemcpyHostToDevice, st));
        } else {
            int k = 0;
            while (ds.occ_res[k] != int(r)) ++k;
            uint16_t *a, *b;
            NG_TRY(cudaMallocAsync(&a, n * 2 + kDistScratchPad, st));
            NG_TRY(cudaMallocAsync(&b, n * 2, st));
            launch_distance_grid(ds.occ[k], int(r), a, b, g, st);
            NG_TRY(cudaGetLastError());
            NG_TRY(cudaFreeAsync(a, st));
            NG_TRY(cudaFreeAsync(b, st));
        }
        ds.dist = g;
        ds.dist_res = int(r);
        s->info.dev_dist = g;
    } else {
        ds.dist = nullptr;
        ds.dist_res = 0;
    }
    // --- derived constants: each is the float the reference computes in place ---
    {
        const int r0 = ds.occ_res[0];
        ds.occ_h0 = float(r0) / 2.0f;                     // to_grid_coord, hash_grid.hpp:23-26
        for (int k = 0; k < NGPRT_PYRAMID_LEVELS; ++k) {
            ds.lvl_two_over_res[k] = 2.0f / float(ds.occ_res[k]);  // occupancy.hpp:247
            ds.lvl_inv_res[k] = 1.0f / float(ds.occ_res[k]);
        }
        ds.occ_pow2 = (r0 & (r0 - 1)) == 0;
        ds.dist_is_l1 = ds.dist_res != 0 && ds.dist_res == ds.occ_res[1];
        // next_step consults the grid iff res(exit level) < dist_res (occupancy.hpp:267)
        ds.consult_mask = 0;
        for (int k = 0; k < NGPRT_PYRAMID_LEVELS; ++k)
            if (ds.dist && ds.occ_res[k] < ds.dist_res) ds.consult_mask |= 1u << k;
        ds.dist_h = ds.dist_res ? float(ds.dist_res) / 2.0f : 0.f;
        ds.dist_vox = ds.dist_res ? float(2.0 / ds.dist_res) : 0.f;  // DistanceGrid::voxel_size
        ds.coarse_h = float(ds.L_C) / 2.0f;
        for (int l = 0; l < L; ++l) ds.fine_h[l] = float(ds.fine_res[l]) / 2.0f;
        ds.coarse_u32 = n_corner < (uint64_t(1) << 32);
        ds.fast_decode = ds.coarse_u32;
        for (int l = 0; l < L; ++l) ds.fast_decode &= ds.fine_mode[l] == 1;
        if (const char* e = std::getenv("NGPRT_FAST_DECODE")) ds.fast_decode &= std::atoi(e) != 0;
        const size_t r1 = size_t(ds.occ_res[1]);
        uint16_t* probe;
        NG_TRY(s->alloc(&probe, r1 * r1 * r1 * 2));
        ds.probe = probe;
        launch_probe_codes(ds, probe, st);
        NG_TRY(cudaGetLastError());
    }
    // --- psi (packed f32 for the exact path; tcgen05 operand image for the tensor path) ---
    {
        std::vector<float> packed(kPsiTotal);
        std::memcpy(packed.data() + kPsiW0, d->psi_w[0], 64 * 23 * 4);
        std::memcpy(packed.data() + kPsiB0, d->psi_b[0], 64 * 4);
        std::memcpy(packed.data() + kPsiW1, d->psi_w[1], 64 * 64 * 4);
        std::memcpy(packed.data() + kPsiB1, d->psi_b[1], 64 * 4);
        std::memcpy(packed.data() + kPsiW2, d->psi_w[2], 3 * 64 * 4);
        std::memcpy(packed.data() + kPsiB2, d->psi_b[2], 3 * 4);
        float* g;
        NG_TRY(s->alloc(&g, kPsiTotal * 4));
        NG_TRY(cudaMemcpyAsync(g, packed.data(), kPsiTotal * 4, cudaMemcpyHostToDevice, st));
        NG_TRY(cudaStreamSynchronize(st));  // `packed` is pageable and local
        ds.psi = g;
        std::vector<unsigned char> tc(psi_tc_bytes());
        pack_psi_tc(packed.data(), tc.data());
        shade_consts_from_psi(packed.data(), &s->shade_consts);
        NG_TRY(s->alloc(&s->psi_tc, tc.size()));
        NG_TRY(cudaMemcpyAsync(s->psi_tc, tc.data(), tc.size(), cudaMemcpyHostToDevice, st));
        NG_TRY(cudaStreamSynchronize(st));
    }
    // --- MLP-fusion ablation weights {8L,64,8}, packed f32 (fusion.hpp:91,162-171) ---
    ds.fmlp = nullptr;
    if (d->fusion_tag == NGPRT_FUSION_MLP) {
        const size_t in = size_t(8) * L;
        std::vector<float> packed(64 * in + 64 + 8 * 64 + 8);
        std::memcpy(packed.data(), d->fusion_mlp_w[0], 64 * in * 4);
        std::memcpy(packed.data() + 64 * in, d->fusion_mlp_b[0], 64 * 4);
        std::memcpy(packed.data() + 64 * in + 64, d->fusion_mlp_w[1], 8 * 64 * 4);
        std::memcpy(packed.data() + 64 * in + 64 + 8 * 64, d->fusion_mlp_b[1], 8 * 4);
        float* g;
        NG_TRY(s->alloc(&g, packed.size() * 4));
        NG_TRY(cudaMemcpyAsync(g, packed.data(), packed.size() * 4, cudaMemcpyHostToDevice, st));
        NG_TRY(cudaStreamSynchronize(st));
        ds.fmlp = g;
    }
    // --- invariant attention weights: activate_sigmoid(global_pre) (fusion.hpp:123-132) ---
    if (d->fusion_tag == NGPRT_FUSION_SHARED_ATT_INV || d->fusion_tag == NGPRT_FUSION_SEPARATE_ATT_INV)
        for (int i = 0; i < 2 * L; ++i) ds.att_w[i] = host_sigmoid(d->att_globals[i]);
    NG_TRY(cudaStreamSynchronize(st));
#undef NG_TRY
    cleanup(NGPRT_OK);
    *out = s;
    return NGPRT_OK;
}

void ngprt_scene_destroy(ngprt_scene* s) { delete s; }

ngprt_status ngprt_scene_info_get(const ngprt_scene* s, ngprt_scene_info* info) {
    if (!s || !info) return fail(NGPRT_EINVAL, "null argument");
    *info = s->info;
    return NGPRT_OK;
}

namespace {

// Keep the fine hash tables (random 16 B gathers, the L2-hot working set)
// resident: an access-policy window over the contiguous fine block, backed by
// a persisting L2 set-aside sized to it (north_star: "L2-resident through an
// access-policy window").
void set_l2_window(const ngprt_scene* s, cudaStream_t st, cudaStreamAttrValue* saved) {
    cudaStreamGetAttribute(st, cudaStreamAttributeAccessPolicyWindow, saved);
    // tuning hooks: NGPRT_L2_WINDOW=0 renders without the window, =2 applies it
    // whatever the table size, NGPRT_L2_HIT_RATIO
    // scales the persisting fraction of it
    static const int window_on = [] {
        const char* e = std::getenv("NGPRT_L2_WINDOW");
        return e ? std::atoi(e) : 1;
    }();
    static const float ratio_scale = [] {
        const char* e = std::getenv("NGPRT_L2_HIT_RATIO");
        return e ? float(std::atof(e)) : 1.0f;
    }();
    if (!window_on) return;
    int max_win = 0, max_persist = 0;
    cudaDeviceGetAttribute(&max_win, cudaDevAttrMaxAccessPolicyWindowSize, s->device);
    cudaDeviceGetAttribute(&max_persist, cudaDevAttrMaxPersistingL2CacheSize, s->device);
    if (max_win <= 0 || max_persist <= 0 || !s->fine_block) return;
    // Persist the fine tables only while they fit in half of the persisting
    // set-aside (41 MB on B200): above that the persisting lines cost the coarse
    // rows more hits than they save (measured: c1's 32 MB block
    // 0.233 -> 0.229 ms with the window; c3's 64 MB 3.36 -> 3.41 ms, c2's 128 MB
    // 0.238 -> 0.247 ms), and LRU keeps the hot fine rows resident by itself.
    if (window_on == 1 && s->fine_block_bytes > size_t(max_persist) / 2) return;
    const size_t win = std::min<size_t>(s->fine_block_bytes, size_t(max_win));
    size_t cur = 0;
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    const size_t want = std::min<size_t>(win, size_t(max_persist));
    if (cur < want) cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, want);
    cudaDeviceGetLimit(&cur, cudaLimitPersistingL2CacheSize);
    cudaStreamAttrValue v{};
    v.accessPolicyWindow.base_ptr = s->fine_block;
    v.accessPolicyWindow.num_bytes = win;
    v.accessPolicyWindow.hitRatio = std::min(1.0f, ratio_scale * float(double(cur) / double(win)));
    v.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    v.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &v);
}

// Interleaved-tile sharding geometry of one call (ngprt_render_opts.shard_*).
struct Shard {
    uint32_t world = 0, rank = 0, tile = 0, tiles_x = 0, tiles = 0, local = 0;
    size_t pixels = 0;  // per camera, compact
};

uint32_t shard_tile_or_default(uint32_t t) { return t ? t : 32u; }

ngprt_status shard_of(const ngprt_render_opts* o, uint32_t W, uint32_t H, Shard* sh) {
    *sh = Shard{};
    if (o->shard_world == 0) return NGPRT_OK;  // unsharded
    const uint32_t tile = shard_tile_or_default(o->shard_tile);
    if (tile % 8 || tile > 1024)
        return fail(NGPRT_EINVAL, "shard_tile must be a multiple of 8 and <= 1024");
    if (o->shard_rank >= o->shard_world) return fail(NGPRT_EINVAL, "shard_rank >= shard_world");
    sh->world = o->shard_world;
    sh->rank = o->shard_rank;
    sh->tile = tile;
    sh->tiles_x = (W + tile - 1) / tile;
    sh->tiles = sh->tiles_x * ((H + tile - 1) / tile);
    sh->local = (sh->tiles + sh->world - 1) / sh->world;
    sh->pixels = size_t(sh->local) * tile * tile;
    return NGPRT_OK;
}

// Output pixels per camera of a call (compact when sharded).
size_t out_pixels_per_cam(const ngprt_render_opts* o, uint32_t W, uint32_t H) {
    if (o->shard_world == 0) return size_t(W) * H;
    const uint64_t t = shard_tile_or_default(o->shard_tile);
    const uint64_t n = ((W + t - 1) / t) * ((H + t - 1) / t);
    return size_t((n + o->shard_world - 1) / o->shard_world * t * t);
}

ngprt_status render_impl(const ngprt_scene* s, const ngprt_camera* cams, int n_cams,
                         const ngprt_render_opts* o, float* rgb, ngprt_ray_stats* stats,
                         cudaStream_t st) {
    const NvtxRange range(o && o->shard_world ? "ngprt_render (shard)" : "ngprt_render");
    if (!s || !cams || !o || !rgb) return fail(NGPRT_EINVAL, "ngprt_render: null argument");
    if (n_cams <= 0) return fail(NGPRT_EINVAL, "ngprt_render: n_cams must be > 0");
    if (o->keep_level < 0 || o->keep_level > s->ds.L)
        return fail(NGPRT_EINVAL, "level_masked_fine: keep_level out of range (fusion.hpp:201-202)");
    if (o->mlp_mode != NGPRT_MLP_EXACT && o->mlp_mode != NGPRT_MLP_TENSOR)
        return fail(NGPRT_EINVAL, "unknown mlp_mode");
    const bool window = o->w && o->h;
    const uint32_t W = window ? o->w : cams[0].width, H = window ? o->h : cams[0].height;
    for (int c = 0; c < n_cams; ++c) {
        const ngprt_camera& cam = cams[c];
        if (!window && (cam.width != W || cam.height != H))
            return fail(NGPRT_EINVAL, "all cameras of one call must share width/height");
        if (uint64_t(o->x0) + W > cam.width || uint64_t(o->y0) + H > cam.height)
            return fail(NGPRT_EINVAL, "generate_rays: pixel out of bounds (scene.hpp:214-215)");
        if (!(cam.fx != 0.0) || !(cam.fy != 0.0)) return fail(NGPRT_EINVAL, "zero focal length");
    }
    if (W == 0 || H == 0) return NGPRT_OK;
    Shard sh;
    if (const ngprt_status e = shard_of(o, W, H, &sh)) return e;
    NG_CUDA(cudaSetDevice(s->device));
    const size_t per_cam = sh.world ? sh.pixels : size_t(W) * H;
    // K0/K1 index the pixels of one launch in 31 bits (K1 keeps a per-ray flag in bit 31)
    if (per_cam >= (size_t(1) << 31)) return fail(NGPRT_EINVAL, "frame too large (>= 2^31 pixels)");
    const int cams_per_launch =
        int(std::min<size_t>(kMaxCamsPerLaunch, ((size_t(1) << 31) - 1) / per_cam));
    RayAcc* acc = nullptr;
    const int chunk = std::min(n_cams, cams_per_launch);
    const size_t acc_bytes = per_cam * chunk * sizeof(RayAcc);
    const size_t ray_bytes = per_cam * chunk * 2 * sizeof(float4);
    NG_CUDA(cudaMallocAsync(&acc, acc_bytes + ray_bytes + 256, st));
    const float4* rays = reinterpret_cast<const float4*>(reinterpret_cast<char*>(acc) + acc_bytes);
    unsigned int* work =
        reinterpret_cast<unsigned int*>(reinterpret_cast<char*>(acc) + acc_bytes + ray_bytes);
    cudaStreamAttrValue saved{};
    set_l2_window(s, st, &saved);
    MarchParams p{};
    p.x0 = o->x0;
    p.y0 = o->y0;
    p.w = W;
    p.h = H;
    p.step = o->step > 0 ? o->step : float(2.0 * std::sqrt(3.0) / 512.0);  // kBaseStep config.hpp:11
    p.use_grid = o->use_dist_grid;
    p.max_step_rule = o->max_step_rule;
    p.early_stop = o->early_stop;
    p.keep_level = o->keep_level;
    p.acc = acc;
    p.work = work;
    p.rays = rays;
    {
        // K1 scheduling policy; NGPRT_DECODE_MIN / NGPRT_STEP_BURST override for tuning
        static const int dmin = [] {
            const char* e = std::getenv("NGPRT_DECODE_MIN");
            return e ? std::max(1, std::min(32, std::atoi(e))) : 4;
        }();
        static const int burst = [] {
            const char* e = std::getenv("NGPRT_STEP_BURST");
            return e ? std::max(1, std::min(64, std::atoi(e))) : 6;
        }();
        p.decode_min = dmin;
        p.step_burst = burst;
        // Tensor-MLP mode tolerates 1e-3 on RGB: K1 then accumulates the colour
        // channels with FMA (density / attention / transmittance stay exact, so
        // the per-ray counters do too). NGPRT_FAST_COLOR=0 keeps them exact.
        static const int fast_color = [] {
            const char* e = std::getenv("NGPRT_FAST_COLOR");
            return e ? (std::atoi(e) != 0) : 1;
        }();
        p.fast_color = (o->mlp_mode == NGPRT_MLP_TENSOR) && fast_color;
    }
    p.tiles_x = (W + kRayTileW - 1) / kRayTileW;
    p.tiles_per_cam = p.tiles_x * ((H + kRayTileH - 1) / kRayTileH);
    if (sh.world) {
        p.shard_world = sh.world;
        p.shard_rank = sh.rank;
        p.shard_tile = sh.tile;
        p.shard_tiles_x = sh.tiles_x;
        p.shard_tiles = sh.tiles;
        p.shard_local = sh.local;
        p.shard_rt_x = sh.tile / kRayTileW;
        p.shard_rt_per_tile = p.shard_rt_x * (sh.tile / kRayTileH);
        p.tiles_per_cam = sh.local * p.shard_rt_per_tile;
    }
    std::unique_lock<std::mutex> prof_lock(s->prof_mu, std::defer_lock);
    if (o->profile) {
        prof_lock.lock();
        s->prof_launches = 0;
    }
    for (int c0 = 0; c0 < n_cams; c0 += cams_per_launch) {
        const int nc = std::min(cams_per_launch, n_cams - c0);
        p.n_cams = nc;
        p.n_slots = uint32_t(per_cam * nc);
        for (int i = 0; i < nc; ++i) {
            const ngprt_camera& cam = cams[c0 + i];
            CamParams& cp = p.cams[i];
            for (int k = 0; k < 12; ++k) cp.m[k] = cam.c2w[k];
            cp.fx = cam.fx;
            cp.fy = cam.fy;
            cp.cx = cam.cx;
            cp.cy = cam.cy;
            cp.width = cam.width;
            cp.height = cam.height;
        }
        p.stats = stats ? stats + size_t(c0) * per_cam : nullptr;
        const int li = s->prof_launches;
        NG_CUDA(cudaMemsetAsync(work, 0, sizeof(unsigned int), st));
        if (o->profile) cudaEventRecord(s->prof_event(4 * li), st);
        launch_march(s->ds, p, st, o->profile ? s->prof_event(4 * li + 1) : nullptr);
        if (o->profile) cudaEventRecord(s->prof_event(4 * li + 2), st);
        float* out = rgb + size_t(c0) * per_cam * 3;
        if (o->mlp_mode == NGPRT_MLP_EXACT)
            launch_shade_exact(s->ds, acc, out, per_cam * nc, st);
        else
            launch_shade_tensor(s->ds, s->psi_tc, s->shade_consts, acc, out, per_cam * nc, st);
        if (o->profile) {
            cudaEventRecord(s->prof_event(4 * li + 3), st);
            s->prof_launches = li + 1;
        }
    }
    cudaStreamSetAttribute(st, cudaStreamAttributeAccessPolicyWindow, &saved);
    NG_CUDA(cudaGetLastError());
    NG_CUDA(cudaFreeAsync(acc, st));
    return NGPRT_OK;
}

}  // namespace

ngprt_status ngprt_render(const ngprt_scene* s, const ngprt_camera* cams, int n_cams,
                          const ngprt_render_opts* o, float* rgb_dev, ngprt_ray_stats* stats_dev,
                          void* stream) {
    const DeviceRestore keep;
    return render_impl(s, cams, n_cams, o, rgb_dev, stats_dev, static_cast<cudaStream_t>(stream));
}

ngprt_status ngprt_render_host(const ngprt_scene* s, const ngprt_camera* cams, int n_cams,
                               const ngprt_render_opts* o, float* rgb_host,
                               ngprt_ray_stats* stats_host) {
    const DeviceRestore keep;
    if (!s || !cams || !o || !rgb_host) return fail(NGPRT_EINVAL, "ngprt_render_host: null argument");
    if (n_cams <= 0) return fail(NGPRT_EINVAL, "ngprt_render_host: n_cams must be > 0");
    NG_CUDA(cudaSetDevice(s->device));
    const bool window = o->w && o->h;
    const uint32_t W = window ? o->w : cams[0].width, H = window ? o->h : cams[0].height;
    for (int c = 1; c < n_cams; ++c)
        if (!window && (cams[c].width != W || cams[c].height != H))
            return fail(NGPRT_EINVAL, "all cameras of one call must share width/height");
    const size_t per_cam = out_pixels_per_cam(o, W, H), n = per_cam * size_t(n_cams);
    // One call at a time per scene through the cached stream pair and buffers.
    std::lock_guard<std::mutex> lock(s->host.mu);
    auto& hc = s->host;
    if (!hc.render) {
        NG_CUDA(cudaStreamCreateWithFlags(&hc.render, cudaStreamNonBlocking));
        NG_CUDA(cudaStreamCreateWithFlags(&hc.copy, cudaStreamNonBlocking));
    }
    if (hc.rgb_cap < n) {
        if (hc.rgb) cudaFree(hc.rgb);
        hc.rgb = nullptr;
        NG_CUDA(cudaMalloc(&hc.rgb, n * 12));
        hc.rgb_cap = n;
    }
    if (stats_host && hc.stats_cap < n) {
        if (hc.stats) cudaFree(hc.stats);
        hc.stats = nullptr;
        NG_CUDA(cudaMalloc(&hc.stats, n * sizeof(ngprt_ray_stats)));
        hc.stats_cap = n;
    }
    // Pinned (page-locked / registered) host output: the kernels write it directly
    // over the bus (zero-copy), so the transfer overlaps the deferred-MLP kernel
    // instead of following it. NGPRT_ZERO_COPY=0 disables.
    static const bool zc_enabled = [] {
        const char* e = std::getenv("NGPRT_ZERO_COPY");
        return !(e && std::atoi(e) == 0);
    }();
    auto pinned = [](const void* p) -> void* {
        cudaPointerAttributes a{};
        if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
            cudaGetLastError();
            return nullptr;
        }
        return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
    };
    float* rgb_zc = zc_enabled ? static_cast<float*>(pinned(rgb_host)) : nullptr;
    ngprt_ray_stats* stats_zc =
        (zc_enabled && stats_host) ? static_cast<ngprt_ray_stats*>(pinned(stats_host)) : nullptr;
    if (rgb_zc && (!stats_host || stats_zc)) {
        ngprt_status st = render_impl(s, cams, n_cams, o, rgb_zc, stats_zc, hc.render);
        const cudaError_t e = cudaStreamSynchronize(hc.render);
        if (st == NGPRT_OK && e != cudaSuccess)
            st = fail(NGPRT_ECUDA, std::string("ngprt_render_host: ") + cudaGetErrorString(e));
        return st;
    }
    // Otherwise render to device buffers and copy out; optional row bands let the
    // copy of band i (copy stream) overlap the render of band i+1. Measured on
    // B200 the per-band tails cost more than they hide, so one band is the
    // default; NGPRT_HOST_BANDS overrides.
    static const int band_override = [] {
        const char* e = std::getenv("NGPRT_HOST_BANDS");
        return e ? std::atoi(e) : 0;
    }();
    int nb = band_override > 0 ? band_override : 1;
    nb = std::max(1, std::min<int>(nb, int(H)));
    if (o->shard_world) nb = 1;  // a sharded call's compact output has no row bands
    while (hc.band_done.size() < size_t(n_cams) * nb) {
        cudaEvent_t e;
        NG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
        hc.band_done.push_back(e);
    }
    const uint32_t x0 = window ? o->x0 : 0, y0 = window ? o->y0 : 0;
    ngprt_status status = NGPRT_OK;
    for (int c = 0; c < n_cams && status == NGPRT_OK; ++c) {
        for (int b = 0; b < nb && status == NGPRT_OK; ++b) {
            const uint32_t r0 = uint32_t(size_t(H) * b / nb), r1 = uint32_t(size_t(H) * (b + 1) / nb);
            if (r1 <= r0) continue;
            ngprt_render_opts ob = *o;
            ob.x0 = x0;
            ob.y0 = y0 + r0;
            ob.w = W;
            ob.h = r1 - r0;
            const size_t off = size_t(c) * per_cam + size_t(r0) * W;
            const size_t cnt = nb == 1 ? per_cam : size_t(r1 - r0) * W;
            status = render_impl(s, cams + c, 1, &ob, hc.rgb + 3 * off,
                                 stats_host ? hc.stats + off : nullptr, hc.render);
            if (status != NGPRT_OK) break;
            cudaEvent_t ev = hc.band_done[size_t(c) * nb + b];
            cudaEventRecord(ev, hc.render);
            cudaStreamWaitEvent(hc.copy, ev, 0);
            cudaMemcpyAsync(rgb_host + 3 * off, hc.rgb + 3 * off, cnt * 12, cudaMemcpyDeviceToHost,
                            hc.copy);
            if (stats_host)
                cudaMemcpyAsync(stats_host + off, hc.stats + off, cnt * sizeof(ngprt_ray_stats),
                                cudaMemcpyDeviceToHost, hc.copy);
        }
    }
    const cudaError_t e1 = cudaStreamSynchronize(hc.render);
    const cudaError_t e2 = cudaStreamSynchronize(hc.copy);
    if (status == NGPRT_OK && (e1 != cudaSuccess || e2 != cudaSuccess))
        status = fail(NGPRT_ECUDA, std::string("ngprt_render_host: ") +
                                       cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    return status;
}

ngprt_status ngprt_render_host_async(const ngprt_scene* s, const ngprt_camera* cams, int n_cams,
                                     const ngprt_render_opts* o, float* rgb_host,
                                     ngprt_ray_stats* stats_host) {
    const DeviceRestore keep;
    if (!s || !cams || !o || !rgb_host)
        return fail(NGPRT_EINVAL, "ngprt_render_host_async: null argument");
    if (n_cams <= 0) return fail(NGPRT_EINVAL, "ngprt_render_host_async: n_cams must be > 0");
    NG_CUDA(cudaSetDevice(s->device));
    const bool window = o->w && o->h;
    const uint32_t W = window ? o->w : cams[0].width, H = window ? o->h : cams[0].height;
    const size_t n = out_pixels_per_cam(o, W, H) * size_t(n_cams);
    std::lock_guard<std::mutex> lock(s->async.mu);
    auto& ac = s->async;
    if (!ac.copy) {
        for (auto& r : ac.render) NG_CUDA(cudaStreamCreateWithFlags(&r, cudaStreamNonBlocking));
        NG_CUDA(cudaStreamCreateWithFlags(&ac.copy, cudaStreamNonBlocking));
        for (auto& sl : ac.slot) {
            NG_CUDA(cudaEventCreateWithFlags(&sl.rendered, cudaEventDisableTiming));
            NG_CUDA(cudaEventCreateWithFlags(&sl.copied, cudaEventDisableTiming));
        }
    }
    const int k = ac.next;
    auto& sl = ac.slot[k];
    ac.next ^= 1;
    if (sl.busy) {  // the frame two back still owns this slot's device buffers
        NG_CUDA(cudaEventSynchronize(sl.copied));
        sl.busy = false;
    }
    if (sl.rgb_cap < n) {
        if (sl.rgb) cudaFree(sl.rgb);
        sl.rgb = nullptr;
        NG_CUDA(cudaMalloc(&sl.rgb, n * 12));
        sl.rgb_cap = n;
    }
    if (stats_host && sl.stats_cap < n) {
        if (sl.stats) cudaFree(sl.stats);
        sl.stats = nullptr;
        NG_CUDA(cudaMalloc(&sl.stats, n * sizeof(ngprt_ray_stats)));
        sl.stats_cap = n;
    }
    const ngprt_status st = render_impl(s, cams, n_cams, o, sl.rgb, stats_host ? sl.stats : nullptr,
                                        ac.render[k]);
    if (st != NGPRT_OK) return st;
    NG_CUDA(cudaEventRecord(sl.rendered, ac.render[k]));
    NG_CUDA(cudaStreamWaitEvent(ac.copy, sl.rendered, 0));
    NG_CUDA(cudaMemcpyAsync(rgb_host, sl.rgb, n * 12, cudaMemcpyDeviceToHost, ac.copy));
    if (stats_host)
        NG_CUDA(cudaMemcpyAsync(stats_host, sl.stats, n * sizeof(ngprt_ray_stats),
                                cudaMemcpyDeviceToHost, ac.copy));
    NG_CUDA(cudaEventRecord(sl.copied, ac.copy));
    sl.busy = true;
    return NGPRT_OK;
}

ngprt_status ngprt_render_host_wait(const ngprt_scene* s) {
    const DeviceRestore keep;
    if (!s) return fail(NGPRT_EINVAL, "ngprt_render_host_wait: null scene");
    std::lock_guard<std::mutex> lock(s->async.mu);
    auto& ac = s->async;
    if (!ac.copy) return NGPRT_OK;
    NG_CUDA(cudaSetDevice(s->device));
    cudaError_t e1 = cudaStreamSynchronize(ac.render[0]);
    const cudaError_t e1b = cudaStreamSynchronize(ac.render[1]);
    if (e1 == cudaSuccess) e1 = e1b;
    const cudaError_t e2 = cudaStreamSynchronize(ac.copy);
    for (auto& sl : ac.slot) sl.busy = false;
    if (e1 != cudaSuccess || e2 != cudaSuccess)
        return fail(NGPRT_ECUDA, std::string("ngprt_render_host_wait: ") +
                                     cudaGetErrorString(e1 != cudaSuccess ? e1 : e2));
    return NGPRT_OK;
}

ngprt_status ngprt_render_timing3(const ngprt_scene* s, float* ms_raygen, float* ms_march,
                                  float* ms_shade, int* n_launches) {
    if (!s) return fail(NGPRT_EINVAL, "null scene");
    std::lock_guard<std::mutex> g(s->prof_mu);
    float t[3] = {0.f, 0.f, 0.f};
    for (int i = 0; i < s->prof_launches; ++i)
        for (int k = 0; k < 3; ++k) {
            float x = 0.f;
            NG_CUDA(cudaEventElapsedTime(&x, s->prof_events[4 * i + k], s->prof_events[4 * i + k + 1]));
            t[k] += x;
        }
    if (ms_raygen) *ms_raygen = t[0];
    if (ms_march) *ms_march = t[1];
    if (ms_shade) *ms_shade = t[2];
    if (n_launches) *n_launches = 3 * s->prof_launches;  // K0, K1, K2 per camera batch
    return NGPRT_OK;
}

ngprt_status ngprt_render_timing(const ngprt_scene* s, float* ms_march, float* ms_shade,
                                 int* n_launches) {
    return ngprt_render_timing3(s, nullptr, ms_march, ms_shade, n_launches);
}

ngprt_status ngprt_build_pyramid(const uint64_t* base, uint32_t base_res,
                                 uint64_t* const levels[NGPRT_PYRAMID_LEVELS - 1], void* stream) {
    if (!base || !levels) return fail(NGPRT_EINVAL, "ngprt_build_pyramid: null argument");
    if (base_res < 16 || base_res % 16) return fail(NGPRT_EINVAL, "base_res must be a multiple of 16");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const uint32_t* src = reinterpret_cast<const uint32_t*>(base);
    for (int k = 1; k < NGPRT_PYRAMID_LEVELS; ++k) {
        const int r = int(base_res >> k);
        const size_t words = (size_t(r) * r * r + 63) / 64;
        NG_CUDA(cudaMemsetAsync(levels[k - 1], 0, words * 8, st));
        launch_pyramid_level(src, r * 2, reinterpret_cast<uint32_t*>(levels[k - 1]), st);
        src = reinterpret_cast<const uint32_t*>(levels[k - 1]);
    }
    NG_CUDA(cudaGetLastError());
    return NGPRT_OK;
}

ngprt_status ngprt_build_distance_grid(const uint64_t* occ, uint32_t res, uint8_t* out,
                                       void* stream) {
    if (!occ || !out || res == 0) return fail(NGPRT_EINVAL, "ngprt_build_distance_grid: bad argument");
    if (res > 32768) return fail(NGPRT_EINVAL, "resolution too large");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t n = size_t(res) * res * res;
    keep_pool_mapped();
    uint16_t *a, *b;
    NG_CUDA(cudaMallocAsync(&a, n * 2 + kDistScratchPad, st));
    NG_CUDA(cudaMallocAsync(&b, n * 2, st));
    launch_distance_grid(reinterpret_cast<const uint32_t*>(occ), int(res), a, b, out, st);
    NG_CUDA(cudaGetLastError());
    NG_CUDA(cudaFreeAsync(a, st));
    NG_CUDA(cudaFreeAsync(b, st));
    return NGPRT_OK;
}

ngprt_status ngprt_test_expf(const float* x, float* y, uint64_t n, void* stream) {
    launch_test_expf(x, y, n, static_cast<cudaStream_t>(stream));
    NG_CUDA(cudaGetLastError());
    return NGPRT_OK;
}

ngprt_status ngprt_test_expf_range(uint32_t first, uint64_t n, uint32_t* y, void* stream) {
    launch_test_expf_range(first, n, y, static_cast<cudaStream_t>(stream));
    NG_CUDA(cudaGetLastError());
    return NGPRT_OK;
}

ngprt_status ngprt_test_march_segments(const ngprt_scene* s, const float* rays8, int n_rays,
                                       float step, int use_grid, int max_step_rule, int max_seg,
                                       float* seg, int* n_seg, float* samples, int* n_samples,
                                       uint32_t* counters, void* stream) {
    if (!s || !rays8 || n_rays < 0 || max_seg < 0 || !seg || !n_seg || !samples || !n_samples ||
        !counters)
        return fail(NGPRT_EINVAL, "ngprt_test_march_segments: bad argument");
    if (n_rays == 0) return NGPRT_OK;
    NG_CUDA(cudaSetDevice(s->device));
    launch_test_march_segments(s->ds, step > 0 ? step : float(2.0 * std::sqrt(3.0) / 512.0),
                               use_grid, max_step_rule, rays8, n_rays, max_seg, seg, n_seg, samples,
                               n_samples, counters, static_cast<cudaStream_t>(stream));
    NG_CUDA(cudaGetLastError());
    return NGPRT_OK;
}

ngprt_status ngprt_test_hash_index(const int32_t* corners, uint64_t n, uint32_t res,
                                   uint64_t table_len, uint8_t hashed, uint64_t* out,
                                   void* stream) {
    DevScene sc{};
    int mode = 0;
    uint32_t mask = 0;
    if (hashed) {
        if ((table_len & (table_len - 1)) == 0 && table_len <= (uint64_t(1) << 32)) {
            mode = 1;
            mask = uint32_t(table_len - 1);
        } else {
            mode = 2;
        }
    }
    launch_test_hash(sc, corners, n, int(res), table_len, mode, mask,
                     reinterpret_cast<unsigned long long*>(out), static_cast<cudaStream_t>(stream));
    NG_CUDA(cudaGetLastError());
    return NGPRT_OK;
}

}  // extern "C"
