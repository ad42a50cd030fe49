/*
 * oracle/ngprt_oracle.c — TEST INFRASTRUCTURE ONLY. CPU restatement of the
 * reference's per-ray render path, used as the parity checker by tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline leg. Nothing in the
 * product (paper_2407_10482_b200/) links, imports or calls this file.
 *
 * Parity pinned: tests/test_oracle_golden.py checks it bit-for-bit against
 * fixtures produced by the reference itself (oracle/_ref, tests/golden/gen_golden.py).
 *
 * Every function cites the reference file:line it restates (paths relative to
 * /root/reference/proj/include/ngprt/). Arithmetic is IEEE binary32/binary64
 * in the reference's operation order; build with -ffp-contract=off.
 * expf is the host glibc expf, exactly what the reference calls (std::exp(float)).
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#include "../include/ngprt_cuda.h"

#ifdef _OPENMP
#include <omp.h>
#endif

#define ROI_LO (-1.0)
#define ROI_HI (1.0)
#define KEARLY 2e-3 /* kEarlyStopTransmittance, volume.hpp:36 */

/* ---- numerics (nn.hpp) ---- */
static float clampf_ref(float v, float lo, float hi) { return v < lo ? lo : (v > hi ? hi : v); } /* common.hpp:94-97 */
static int clampi_ref(int v, int lo, int hi) { return v < lo ? lo : (v > hi ? hi : v); }
float orc_activate_density(float pre) { return expf(clampf_ref(pre, -15.0f, 15.0f)); } /* nn.hpp:80-83 */
float orc_activate_sigmoid(float pre) { return 1.0f / (1.0f + expf(-pre)); }          /* nn.hpp:91-94 */
float orc_alpha(float sigma, float delta) { return 1.0f - expf(-sigma * delta); }     /* volume.hpp:30-33 */

/* sh_encode, nn.hpp:107-132 (degree 4, no Condon-Shortley) */
void orc_sh_encode(const float* d, float* out) {
    const float x = d[0], y = d[1], z = d[2];
    const float xx = x * x, yy = y * y, zz = z * z;
    out[0] = (float)0.28209479177387814;
    out[1] = (float)0.4886025119029199 * y;
    out[2] = (float)0.4886025119029199 * z;
    out[3] = (float)0.4886025119029199 * x;
    out[4] = (float)1.0925484305920792 * x * y;
    out[5] = (float)1.0925484305920792 * y * z;
    out[6] = (float)0.31539156525252005 * (3.0f * zz - 1.0f);
    out[7] = (float)1.0925484305920792 * x * z;
    out[8] = (float)0.5462742152960396 * (xx - yy);
    out[9] = (float)0.5900435899266435 * y * (3.0f * xx - yy);
    out[10] = (float)2.890611442640554 * x * y * z;
    out[11] = (float)0.4570457994644658 * y * (5.0f * zz - 1.0f);
    out[12] = (float)0.3731763325901154 * z * (5.0f * zz - 3.0f);
    out[13] = (float)0.4570457994644658 * x * (5.0f * zz - 1.0f);
    out[14] = (float)1.445305721320277 * z * (xx - yy);
    out[15] = (float)0.5900435899266435 * x * (xx - 3.0f * yy);
}

/* TinyMlp::forward, nn.hpp:175-196: acc = b[r]; acc += w[r][c]*a[c]; ReLU on hidden layers */
void orc_mlp_forward(int nl, const int* widths, const float* const* W, const float* const* B,
                     const float* in, float* out) {
    float buf[2][256];
    int wi = widths[0];
    memcpy(buf[0], in, sizeof(float) * wi);
    int cur = 0;
    for (int k = 0; k < nl; ++k) {
        const int wo = widths[k + 1];
        const float* a = buf[cur];
        float* o = buf[cur ^ 1];
        for (int r = 0; r < wo; ++r) {
            float acc = B[k][r];
            const float* wr = W[k] + (size_t)r * wi;
            for (int c = 0; c < wi; ++c) acc += wr[c] * a[c];
            o[r] = (k + 1 < nl && acc < 0.0f) ? 0.0f : acc;
        }
        cur ^= 1;
        wi = wo;
    }
    memcpy(out, buf[cur], sizeof(float) * wi);
}

/* ---- hash grid (hash_grid.hpp) ---- */
static float to_grid_coord(float x, int res) { return (x - (float)ROI_LO) * ((float)res / (float)2.0); } /* :23-26 */

/* stencil, hash_grid.hpp:33-56: corner k bit0->x bit1->y bit2->z, w = (wx*wy)*wz */
static void stencil(const float* x, int res, int32_t corners[8][3], float w[8]) {
    int32_t base[3];
    float frac[3];
    for (int a = 0; a < 3; ++a) {
        float u = to_grid_coord(x[a], res);
        int32_t i = (int32_t)floorf(u);
        if (i > res - 1) i = res - 1;
        if (i < 0) i = 0;
        base[a] = i;
        frac[a] = u - (float)i;
    }
    for (int k = 0; k < 8; ++k) {
        int dx = k & 1, dy = (k >> 1) & 1, dz = (k >> 2) & 1;
        corners[k][0] = base[0] + dx;
        corners[k][1] = base[1] + dy;
        corners[k][2] = base[2] + dz;
        float wx = dx ? frac[0] : 1.0f - frac[0];
        float wy = dy ? frac[1] : 1.0f - frac[1];
        float wz = dz ? frac[2] : 1.0f - frac[2];
        w[k] = wx * wy * wz;
    }
}

/* HashLevel::hash_index, hash_grid.hpp:83-94 (primes :8-10) */
uint64_t orc_hash_index(int res, uint64_t table_len, int hashed, int32_t x, int32_t y, int32_t z) {
    if (!hashed) {
        uint64_t r1 = (uint64_t)res + 1;
        return (uint64_t)x + r1 * ((uint64_t)y + r1 * (uint64_t)z);
    }
    uint64_t h = (uint64_t)x * 1ull ^ (uint64_t)y * 2654435761ull ^ (uint64_t)z * 805459861ull;
    return h % table_len;
}

/* ---- occupancy (occupancy.hpp) ---- */
static int bit_get(const uint64_t* words, int res, int x, int y, int z) { /* BitGrid::get :22-25 */
    size_t i = (size_t)x + (size_t)res * ((size_t)y + (size_t)res * (size_t)z);
    return (int)((words[i >> 6] >> (i & 63)) & 1u);
}
static void bit_set(uint64_t* words, int res, int x, int y, int z) {
    size_t i = (size_t)x + (size_t)res * ((size_t)y + (size_t)res * (size_t)z);
    words[i >> 6] |= (uint64_t)1 << (i & 63);
}
static size_t grid_words(int res) { return ((size_t)res * res * res + 63) / 64; }

/* BitGrid::downsampled2 (:40-51) applied 4 times = build_pyramid (:114-119) */
void orc_build_pyramid(const uint64_t* base, int res, uint64_t* out_levels /* levels 1..4 concatenated */) {
    const uint64_t* src = base;
    int r = res;
    uint64_t* dst = out_levels;
    for (int k = 1; k < NGPRT_PYRAMID_LEVELS; ++k) {
        int ro = r / 2;
        memset(dst, 0, grid_words(ro) * 8);
        for (int z = 0; z < ro; ++z)
            for (int y = 0; y < ro; ++y)
                for (int x = 0; x < ro; ++x) {
                    int v = 0;
                    for (int c = 0; c < 8 && !v; ++c)
                        v = bit_get(src, r, 2 * x + (c & 1), 2 * y + ((c >> 1) & 1), 2 * z + (c >> 2));
                    if (v) bit_set(dst, ro, x, y, z);
                }
        src = dst;
        dst += grid_words(ro);
        r = ro;
    }
}

/* build_distance_grid, occupancy.hpp:136-194: two-pass 26-neighbour unit chamfer
 * (exact Chebyshev), G = min(255, max(0, D-1)) */
void orc_build_distance_grid(const uint64_t* occ, int r, uint8_t* out) {
    const uint32_t inf = 0x3FFFFFFF;
    size_t n = (size_t)r * r * r;
    uint32_t* d = (uint32_t*)malloc(n * sizeof(uint32_t));
#define IDX(x, y, z) ((size_t)(x) + (size_t)r * ((size_t)(y) + (size_t)r * (size_t)(z)))
    for (int z = 0; z < r; ++z)
        for (int y = 0; y < r; ++y)
            for (int x = 0; x < r; ++x) d[IDX(x, y, z)] = bit_get(occ, r, x, y, z) ? 0 : inf;
    for (int z = 0; z < r; ++z)
        for (int y = 0; y < r; ++y)
            for (int x = 0; x < r; ++x) {
                uint32_t* cur = &d[IDX(x, y, z)];
                if (*cur == 0) continue;
                uint32_t best = *cur;
                for (int dz = -1; dz <= 0; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (dz == 0 && (dy > 0 || (dy == 0 && dx >= 0))) continue;
                            int nx = x + dx, ny = y + dy, nz = z + dz;
                            if (nx < 0 || ny < 0 || nz < 0 || nx >= r || ny >= r || nz >= r) continue;
                            uint32_t c = d[IDX(nx, ny, nz)] + 1;
                            if (c < best) best = c;
                        }
                *cur = best;
            }
    for (int z = r - 1; z >= 0; --z)
        for (int y = r - 1; y >= 0; --y)
            for (int x = r - 1; x >= 0; --x) {
                uint32_t* cur = &d[IDX(x, y, z)];
                if (*cur == 0) continue;
                uint32_t best = *cur;
                for (int dz = 0; dz <= 1; ++dz)
                    for (int dy = -1; dy <= 1; ++dy)
                        for (int dx = -1; dx <= 1; ++dx) {
                            if (dz == 0 && (dy < 0 || (dy == 0 && dx <= 0))) continue;
                            int nx = x + dx, ny = y + dy, nz = z + dz;
                            if (nx < 0 || ny < 0 || nz < 0 || nx >= r || ny >= r || nz >= r) continue;
                            uint32_t c = d[IDX(nx, ny, nz)] + 1;
                            if (c < best) best = c;
                        }
                *cur = best;
            }
#undef IDX
    for (size_t i = 0; i < n; ++i) {
        uint32_t v = d[i] == 0 ? 0 : d[i] - 1;
        out[i] = (uint8_t)(v < 255 ? v : 255);
    }
    free(d);
}

/* ---- scene ---- */
typedef struct orc_scene {
    ngprt_scene_desc d;
    int L, w;                 /* levels, coarse row width 8+2L */
    uint64_t* keys;           /* sorted coarse keys */
    float* rows;              /* rows in sorted-key order */
    int pyr_res[NGPRT_PYRAMID_LEVELS];
    uint64_t* pyr[NGPRT_PYRAMID_LEVELS];
    uint64_t* pyr_store;
    uint8_t* dist;            /* owned or borrowed */
    int dist_owned;
    float att_w[2 * NGPRT_MAX_FINE_LEVELS]; /* post-sigmoid global weights (Inv modes) */
    float zero_row[16];
} orc_scene;

static const orc_scene* g_sort_ctx;
static int cmp_idx(const void* a, const void* b) {
    uint64_t ka = g_sort_ctx->d.coarse_keys[*(const uint64_t*)a];
    uint64_t kb = g_sort_ctx->d.coarse_keys[*(const uint64_t*)b];
    return ka < kb ? -1 : (ka > kb ? 1 : 0);
}

orc_scene* orc_scene_create(const ngprt_scene_desc* d) {
    orc_scene* s = (orc_scene*)calloc(1, sizeof(orc_scene));
    s->d = *d;
    s->L = (int)d->L;
    s->w = 8 + 2 * s->L;
    /* SparseCoarseGrid (baking.hpp:11-50) as sorted keys + binary search */
    uint64_t n = d->n_coarse;
    uint64_t* perm = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    for (uint64_t i = 0; i < n; ++i) perm[i] = i;
    g_sort_ctx = s;
    qsort(perm, n, sizeof(uint64_t), cmp_idx);
    s->keys = (uint64_t*)malloc((n ? n : 1) * sizeof(uint64_t));
    s->rows = (float*)malloc((n ? n : 1) * s->w * sizeof(float));
    for (uint64_t i = 0; i < n; ++i) {
        s->keys[i] = d->coarse_keys[perm[i]];
        memcpy(s->rows + i * s->w, d->coarse_rows + perm[i] * s->w, s->w * sizeof(float));
    }
    free(perm);
    /* build_pyramid from level 0 (occupancy.hpp:114-119) */
    int r = (int)d->occ_base_res;
    size_t total = 0;
    for (int k = 1; k < NGPRT_PYRAMID_LEVELS; ++k) total += grid_words(r >> k);
    s->pyr_store = (uint64_t*)malloc(total * 8);
    orc_build_pyramid(d->pyramid_words[0], r, s->pyr_store);
    s->pyr[0] = (uint64_t*)d->pyramid_words[0];
    s->pyr_res[0] = r;
    uint64_t* p = s->pyr_store;
    for (int k = 1; k < NGPRT_PYRAMID_LEVELS; ++k) {
        s->pyr[k] = p;
        s->pyr_res[k] = r >> k;
        p += grid_words(r >> k);
    }
    if (d->dist_res) {
        if (d->dist_values) {
            s->dist = (uint8_t*)d->dist_values;
        } else {
            int k = 0;
            while (k < NGPRT_PYRAMID_LEVELS && s->pyr_res[k] != (int)d->dist_res) ++k;
            if (k == NGPRT_PYRAMID_LEVELS) { free(s); return NULL; }
            s->dist = (uint8_t*)malloc((size_t)d->dist_res * d->dist_res * d->dist_res);
            s->dist_owned = 1;
            orc_build_distance_grid(s->pyr[k], (int)d->dist_res, s->dist);
        }
    }
    /* FusionMode::effective_weights for the invariant modes (fusion.hpp:123-132) */
    if (d->fusion_tag == NGPRT_FUSION_SHARED_ATT_INV || d->fusion_tag == NGPRT_FUSION_SEPARATE_ATT_INV)
        for (int i = 0; i < 2 * s->L; ++i) s->att_w[i] = orc_activate_sigmoid(d->att_globals[i]);
    return s;
}

void orc_scene_destroy(orc_scene* s) {
    if (!s) return;
    free(s->keys);
    free(s->rows);
    free(s->pyr_store);
    if (s->dist_owned) free(s->dist);
    free(s);
}

const uint64_t* orc_scene_pyramid_level(const orc_scene* s, int k) { return s->pyr[k]; }
const uint8_t* orc_scene_dist(const orc_scene* s) { return s->dist; }

/* SparseCoarseGrid::row (baking.hpp:40-43): absent -> zero row */
static const float* coarse_row(const orc_scene* s, uint64_t key) {
    uint64_t lo = 0, hi = s->d.n_coarse;
    while (lo < hi) {
        uint64_t mid = (lo + hi) / 2;
        if (s->keys[mid] < key) lo = mid + 1; else hi = mid;
    }
    if (lo < s->d.n_coarse && s->keys[lo] == key) return s->rows + lo * s->w;
    return s->zero_row;
}

/* decode_point_baked_raw + [level_masked_fine] + fuse (baking.hpp:68-91,
 * model.hpp:13-22, fusion.hpp:107-173, :198-209) */
void orc_decode_point(const orc_scene* s, const float* x, int keep_level, float* out) {
    const int L = s->L, w = s->w;
    int32_t c[8][3];
    float wt[8];
    stencil(x, (int)s->d.L_C, c, wt);
    float dec[16] = {0};
    const uint64_t r1 = (uint64_t)s->d.L_C + 1;
    for (int k = 0; k < 8; ++k) {
        uint64_t key = (uint64_t)c[k][0] + r1 * ((uint64_t)c[k][1] + r1 * (uint64_t)c[k][2]); /* key_of :28-31 */
        const float* row = coarse_row(s, key);
        float wk = wt[k];
        for (int i = 0; i < w; ++i) dec[i] += wk * row[i];
    }
    float omega[4], beta[4];
    for (int l = 0; l < L; ++l) {
        omega[l] = orc_activate_sigmoid(dec[8 + 2 * l]);
        beta[l] = orc_activate_sigmoid(dec[8 + 2 * l + 1]);
    }
    float fine[4][8];
    for (int l = 0; l < L; ++l) {
        const int res = (int)s->d.fine_res[l];
        int32_t fc[8][3];
        float fw[8];
        stencil(x, res, fc, fw);
        for (int f = 0; f < 8; ++f) fine[l][f] = 0.0f;
        for (int k = 0; k < 8; ++k) {
            uint64_t idx = orc_hash_index(res, s->d.fine_table_len[l], s->d.fine_hashed[l], fc[k][0],
                                          fc[k][1], fc[k][2]);
            const float* row = s->d.fine_tables[l] + idx * 8;
            float wk = fw[k];
            for (int f = 0; f < 8; ++f) fine[l][f] += wk * row[f];
        }
    }
    if (keep_level > 0)
        for (int l = 0; l < L; ++l)
            if (l + 1 != keep_level)
                for (int ch = 1; ch < 8; ++ch) fine[l][ch] = 0.0f;
    if (s->d.fusion_tag == NGPRT_FUSION_MLP) { /* fuse, MLP ablation: fusion.hpp:162-171 */
        float in[32], hat[8];
        for (int l = 0; l < L; ++l)
            for (int ch = 0; ch < 8; ++ch) in[8 * l + ch] = fine[l][ch];
        const int widths[3] = {8 * L, 64, 8};
        orc_mlp_forward(2, widths, s->d.fusion_mlp_w, s->d.fusion_mlp_b, in, hat);
        for (int i = 0; i < 8; ++i) out[i] = dec[i] + hat[i];
        return;
    }
    float wo[4], wb[4];
    for (int l = 0; l < L; ++l) {
        switch (s->d.fusion_tag) {
            case NGPRT_FUSION_SUM: wo[l] = wb[l] = 1.0f; break;
            case NGPRT_FUSION_SHARED_ATT_V: wo[l] = wb[l] = omega[l]; break;
            case NGPRT_FUSION_SEPARATE_ATT_V: wo[l] = omega[l]; wb[l] = beta[l]; break;
            case NGPRT_FUSION_SHARED_ATT_INV: wo[l] = wb[l] = s->att_w[2 * l]; break;
            default: wo[l] = s->att_w[2 * l]; wb[l] = s->att_w[2 * l + 1]; break;
        }
    }
    for (int i = 0; i < 8; ++i) out[i] = dec[i];
    for (int l = 0; l < L; ++l) {
        out[0] += wo[l] * fine[l][0];
        for (int ch = 1; ch < 4; ++ch) out[ch] += wb[l] * fine[l][ch];
        for (int ch = 4; ch < 8; ++ch) out[ch] += wb[l] * fine[l][ch];
    }
}

/* clip_to_roi<float>, occupancy.hpp:279-297 */
static int clip_f(const float* o, const float* d, float tn, float tf, float* t0, float* t1) {
    *t0 = tn;
    *t1 = tf;
    for (int a = 0; a < 3; ++a) {
        if (d[a] == 0.0f) {
            if (o[a] < (float)ROI_LO || o[a] > (float)ROI_HI) return 0;
            continue;
        }
        float ta = ((float)ROI_LO - o[a]) / d[a];
        float tb = ((float)ROI_HI - o[a]) / d[a];
        if (ta > tb) { float tmp = ta; ta = tb; tb = tmp; }
        *t0 = (*t0 < ta) ? ta : *t0; /* std::max */
        *t1 = (tb < *t1) ? tb : *t1; /* std::min */
    }
    return *t0 < *t1;
}

/* generate_rays<float>, scene.hpp:211-228 (f64 then cast) */
int orc_generate_ray(const ngprt_camera* c, double u, double v, float* ray8) {
    const double* m = c->c2w;
    double dcx = (u - c->cx) / c->fx, dcy = (v - c->cy) / c->fy, dcz = 1.0;
    double wx = m[0] * dcx + m[1] * dcy + m[2] * dcz; /* c2w_rotate :203-206 */
    double wy = m[4] * dcx + m[5] * dcy + m[6] * dcz;
    double wz = m[8] * dcx + m[9] * dcy + m[10] * dcz;
    double n = sqrt(wx * wx + wy * wy + wz * wz); /* Vec3::normalized common.hpp:30-35 */
    wx = wx / n; wy = wy / n; wz = wz / n;
    double o[3] = {m[3], m[7], m[11]}, d[3] = {wx, wy, wz};
    double t0 = 0.0, t1 = 1e9;
    for (int a = 0; a < 3; ++a) { /* clip_to_roi<double> */
        if (d[a] == 0.0) {
            if (o[a] < ROI_LO || o[a] > ROI_HI) return 0;
            continue;
        }
        double ta = (ROI_LO - o[a]) / d[a], tb = (ROI_HI - o[a]) / d[a];
        if (ta > tb) { double tmp = ta; ta = tb; tb = tmp; }
        t0 = (t0 < ta) ? ta : t0;
        t1 = (tb < t1) ? tb : t1;
    }
    if (!(t0 < t1)) return 0;
    ray8[0] = (float)o[0]; ray8[1] = (float)o[1]; ray8[2] = (float)o[2];
    ray8[3] = (float)d[0]; ray8[4] = (float)d[1]; ray8[5] = (float)d[2];
    ray8[6] = (float)(t0 < 0.0 ? 0.0 : t0); /* std::max(t0, 0.0) */
    ray8[7] = (float)t1;
    return ray8[6] < ray8[7];
}

/* voxel_of, occupancy.hpp:94-102 */
static void voxel_of(const float* x, int res, int* v) {
    for (int a = 0; a < 3; ++a) v[a] = clampi_ref((int)floorf(to_grid_coord(x[a], res)), 0, res - 1);
}

/* voxel_exit_step, occupancy.hpp:238-255 (x = ray.at(t), unclamped) */
static float voxel_exit_step(const float* o, const float* d, float t, int res) {
    float x[3] = {o[0] + d[0] * t, o[1] + d[1] * t, o[2] + d[2] * t};
    int v[3];
    voxel_of(x, res, v);
    float t_exit = 3.40282347e38f;
    for (int a = 0; a < 3; ++a) {
        float da = d[a];
        if (da == 0.0f) continue;
        float lo = (float)ROI_LO + (float)2.0 * (float)v[a] / (float)res;
        float hi = lo + (float)2.0 / (float)res;
        float bound = da > 0.0f ? hi : lo;
        float tc = (bound - o[a]) / da;
        t_exit = (tc < t_exit) ? tc : t_exit;
    }
    float s = t_exit - t;
    if (!(s > 0.0f)) s = 0.0f;
    return s + (float)1e-6;
}

typedef struct { uint32_t marching, occupied, occ_acc, dist_acc; } orc_counters;

/* Canonical render_ray for one ray; returns shaded flag. */
static void render_ray(const orc_scene* s, const float* ray8, const ngprt_render_opts* o, float step,
                       float* rgb, orc_counters* mc) {
    const float* org = ray8;
    const float* dir = ray8 + 3;
    float t0, t1;
    float cd[3] = {0, 0, 0}, fs[4] = {0, 0, 0, 0}, T = 1.0f;
    int use_grid = o->use_dist_grid && s->dist != NULL;
    if (clip_f(org, dir, ray8[6], ray8[7], &t0, &t1)) {
        float t = t0;
        while (t < t1) { /* march, occupancy.hpp:310-324 */
            float x[3];
            for (int a = 0; a < 3; ++a) x[a] = clampf_ref(org[a] + dir[a] * t, -1.0f, 1.0f);
            mc->marching++;
            int exit_res = 0, occupied = 1;
            for (int k = NGPRT_PYRAMID_LEVELS - 1; k >= 0; --k) { /* occupancy_probe :218-231 */
                int v[3];
                voxel_of(x, s->pyr_res[k], v);
                mc->occ_acc++;
                if (!bit_get(s->pyr[k], s->pyr_res[k], v[0], v[1], v[2])) {
                    occupied = 0;
                    exit_res = s->pyr_res[k];
                    break;
                }
            }
            if (occupied) {
                mc->occupied++;
                float f[8];
                orc_decode_point(s, x, o->keep_level, f);
                /* composite, volume.hpp:61-70 */
                float sigma = orc_activate_density(f[0]);
                float a = orc_alpha(sigma, step);
                float w = a * T;
                for (int c = 0; c < 3; ++c) cd[c] += w * f[1 + c];
                for (int c = 0; c < 4; ++c) fs[c] += w * f[4 + c];
                T = T * (1.0f - a);
                if (o->early_stop && T < (float)KEARLY) break;
                t += step;
            } else { /* next_step, occupancy.hpp:261-276 */
                float s_occ = voxel_exit_step(org, dir, t, exit_res);
                float sstep = s_occ;
                if (use_grid && exit_res < (int)s->d.dist_res) {
                    float xu[3] = {org[0] + dir[0] * t, org[1] + dir[1] * t, org[2] + dir[2] * t};
                    int v[3];
                    const int gr = (int)s->d.dist_res;
                    voxel_of(xu, gr, v);
                    mc->dist_acc++;
                    uint8_t g = s->dist[(size_t)v[0] + (size_t)gr * ((size_t)v[1] + (size_t)gr * v[2])];
                    if (g > 0) {
                        float s_dist = (float)(2.0 / gr) * (float)g;
                        sstep = o->max_step_rule ? ((s_dist < s_occ) ? s_occ : s_dist) : s_dist;
                    }
                }
                t += sstep;
            }
        }
    }
    rgb[0] = rgb[1] = rgb[2] = 0.0f;
    if (T < 1.0f) { /* shade, volume.hpp:118-137 */
        float in[23];
        for (int c = 0; c < 3; ++c) in[c] = cd[c];
        for (int c = 0; c < 4; ++c) in[3 + c] = fs[c];
        orc_sh_encode(dir, in + 7);
        static const int widths[4] = {23, 64, 64, 3};
        float out[3];
        orc_mlp_forward(3, widths, s->d.psi_w, s->d.psi_b, in, out);
        for (int c = 0; c < 3; ++c) rgb[c] = orc_activate_sigmoid(cd[c] + out[c]);
    }
}

/* Render one camera window: rgb w*h*3, stats w*h*4 (nullable). */
int orc_render(const orc_scene* s, const ngprt_camera* cam, const ngprt_render_opts* o, float* rgb,
               uint32_t* stats, int nthreads) {
    const float step = o->step > 0 ? o->step : (float)(2.0 * sqrt(3.0) / 512.0); /* kBaseStep config.hpp:11 */
    const uint32_t W = (o->w && o->h) ? o->w : cam->width;
    const uint32_t H = (o->w && o->h) ? o->h : cam->height;
    (void)nthreads;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(dynamic, 1)
#endif
    for (int64_t py = 0; py < (int64_t)H; ++py) {
        for (uint32_t px = 0; px < W; ++px) {
            size_t pix = (size_t)py * W + px;
            float ray8[8];
            orc_counters mc = {0, 0, 0, 0};
            float* out = rgb + 3 * pix;
            out[0] = out[1] = out[2] = 0.0f;
            if (orc_generate_ray(cam, (double)(o->x0 + px) + 0.5, (double)(o->y0 + py) + 0.5, ray8))
                render_ray(s, ray8, o, step, out, &mc);
            if (stats) {
                stats[4 * pix + 0] = mc.marching;
                stats[4 * pix + 1] = mc.occupied;
                stats[4 * pix + 2] = mc.occ_acc;
                stats[4 * pix + 3] = mc.dist_acc;
            }
        }
    }
    return 0;
}

float orc_expf(float x) { return expf(x); }

/* expf over the consecutive bit patterns [first, first+n): out[i] = bits(expf(float(first+i))).
 * The exhaustive device-port check (tests/test_gpu_kernels.py) compares against this. */
void orc_expf_range(uint32_t first, uint64_t n, uint32_t* out, int nthreads) {
    (void)nthreads;
#ifdef _OPENMP
    if (nthreads > 0) omp_set_num_threads(nthreads);
#pragma omp parallel for schedule(static)
#endif
    for (int64_t i = 0; i < (int64_t)n; ++i) {
        uint32_t b = first + (uint32_t)i;
        float x, y;
        memcpy(&x, &b, 4);
        y = expf(x);
        memcpy(&out[i], &y, 4);
    }
}
