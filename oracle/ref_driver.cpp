// oracle/ref_driver.cpp — TEST INFRASTRUCTURE ONLY (never shipped, never measured as product).
//
// Compiles the UNMODIFIED reference headers in place (-I /root/reference/proj/include)
// into oracle/_ref/libngprt_ref.so and exposes, through extern "C", the reference's
// own functions on the render path plus the canonical render_ray composition.
// The reference implements no render function (SPEC.md:309-317 specifies it); the
// composition below is SURVEY.md §8(c) verbatim:
//   generate_rays (scene.hpp:211-228) -> march (occupancy.hpp:302-326) whose emit(t)
//   decodes (baking.hpp:84-91, + level_masked_fine fusion.hpp:198-209 when keep_level)
//   and tracks T like composite (volume.hpp:61-70) -> composite (volume.hpp:51-75)
//   -> shade (volume.hpp:118-137) iff final_t < 1 (training.hpp:321).
// Used by tests/golden/gen_golden.py to pin the C restatement (oracle/ngprt_oracle.c)
// and the synthetic-scene generator, and by bench.py --impl reference as the CPU
// baseline (OpenMP over rows; the scene is read-only).
#include "ngprt/baking.hpp"
#include "ngprt/config.hpp"
#include "ngprt/scene.hpp"

#include "../include/ngprt_cuda.h"

#include <omp.h>

using namespace ngprt;

namespace {

struct RefScene {
    BakedScene s;
    int dist_res = 0;
    bool has_dist = false;
};

thread_local std::string g_err;

BitGrid bitgrid_from_words(const uint64_t* w, int res) {
    BitGrid g(res);
    std::memcpy(g.words.data(), w, g.words.size() * sizeof(uint64_t));
    return g;
}

PosedDataset dataset_of(const ngprt_camera& c) {
    PosedDataset ds;
    ds.width = int(c.width);
    ds.height = int(c.height);
    ds.fx = c.fx;
    ds.fy = c.fy;
    ds.cx = c.cx;
    ds.cy = c.cy;
    Frame f;
    for (int i = 0; i < 16; ++i) f.c2w[i] = c.c2w[i];
    ds.frames.push_back(f);
    return ds;
}

} // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

void* ref_scene_create(const ngprt_scene_desc* d) {
    try {
        auto* r = new RefScene;
        BakedScene& s = r->s;
        const int L = int(d->L);
        s.cfg.corner_grid_res = int(d->L_C);
        s.cfg.fine_levels = L;
        s.cfg.fine_table_len = d->fine_table_len[0];
        s.tag = FusionTag(d->fusion_tag);
        s.coarse.init(int(d->L_C), L);
        const int w = 8 + 2 * L;
        for (uint64_t i = 0; i < d->n_coarse; ++i) {
            float* dst = s.coarse.add_row(d->coarse_keys[i]);
            std::memcpy(dst, d->coarse_rows + i * w, sizeof(float) * w);
        }
        s.fine.resize(L);
        for (int l = 0; l < L; ++l) {
            auto& lvl = s.fine[l];
            lvl.resolution = int(d->fine_res[l]);
            lvl.table_len = d->fine_table_len[l];
            lvl.feature_dim = kFineFeatureDim;
            lvl.addressing = d->fine_hashed[l] ? Addressing::Hashed : Addressing::Direct;
            lvl.entries.init("fine_l" + std::to_string(l + 1), lvl.table_len * kFineFeatureDim,
                             false);
            std::memcpy(lvl.entries.value.data(), d->fine_tables[l],
                        sizeof(float) * lvl.table_len * kFineFeatureDim);
        }
        Rng dummy(0);
        s.psi.init({kShadeInWidth, 64, 64, 3}, "psi", dummy, nullptr);
        for (int k = 0; k < 3; ++k) {
            std::memcpy(s.psi.weight[k].value.data(), d->psi_w[k],
                        sizeof(float) * s.psi.weight[k].value.size());
            std::memcpy(s.psi.bias[k].value.data(), d->psi_b[k],
                        sizeof(float) * s.psi.bias[k].value.size());
        }
        s.fusion.init(s.tag, L, dummy, nullptr);
        if (fusion_is_invariant(s.tag))
            for (int i = 0; i < 2 * L; ++i) s.fusion.global_pre.value[i] = d->att_globals[i];
        if (s.tag == FusionTag::Mlp)
            for (int k = 0; k < 2; ++k) {
                std::memcpy(s.fusion.mlp.weight[k].value.data(), d->fusion_mlp_w[k],
                            sizeof(float) * s.fusion.mlp.weight[k].value.size());
                std::memcpy(s.fusion.mlp.bias[k].value.data(), d->fusion_mlp_b[k],
                            sizeof(float) * s.fusion.mlp.bias[k].value.size());
            }
        // The reference's own pyramid and distance transform, from level 0 only.
        s.pyramid = build_pyramid(bitgrid_from_words(d->pyramid_words[0], int(d->occ_base_res)));
        if (d->dist_res) {
            r->has_dist = true;
            r->dist_res = int(d->dist_res);
            if (d->dist_values) {
                s.distance.resolution = int(d->dist_res);
                s.distance.voxel_size = Roi::extent / d->dist_res;
                s.distance.values.assign(d->dist_values,
                                         d->dist_values + size_t(d->dist_res) * d->dist_res *
                                                              d->dist_res);
            } else {
                int k = 0;
                while (k < kPyramidLevels && s.pyramid.levels[k].res != int(d->dist_res)) ++k;
                if (k == kPyramidLevels) throw std::invalid_argument("dist_res is no pyramid level");
                s.distance = build_distance_grid(s.pyramid.levels[k]);
            }
        }
        return r;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

void ref_scene_destroy(void* p) { delete static_cast<RefScene*>(p); }

// Canonical render_ray composition; fills rgb (w*h*3) and stats (w*h*4).
int ref_render(void* handle, const ngprt_camera* cam, const ngprt_render_opts* o, float* rgb,
               uint32_t* stats, int nthreads) {
    try {
        const RefScene& r = *static_cast<const RefScene*>(handle);
        const BakedScene& s = r.s;
        const PosedDataset ds = dataset_of(*cam);
        const float step = o->step > 0 ? o->step : float(kBaseStep);
        const DistanceGrid* grid = (o->use_dist_grid && r.has_dist) ? &s.distance : nullptr;
        const uint32_t x0 = o->x0, y0 = o->y0;
        const uint32_t W = (o->w && o->h) ? o->w : cam->width;
        const uint32_t H = (o->w && o->h) ? o->h : cam->height;
        const int L = s.cfg.fine_levels;
        if (nthreads > 0) omp_set_num_threads(nthreads);
        std::string err;
#pragma omp parallel for schedule(dynamic, 1)
        for (int64_t py = 0; py < int64_t(H); ++py) {
            std::vector<RaySample<float>> samples;
            for (uint32_t px = 0; px < W; ++px) {
                const size_t pix = size_t(py) * W + px;
                float* out = rgb + 3 * pix;
                out[0] = out[1] = out[2] = 0.f;
                MarchCounters mc;
                Ray<float> ray;
                try {
                    bool ok = generate_rays(ds, 0, double(x0 + px) + 0.5, double(y0 + py) + 0.5,
                                            ray);
                    if (ok) {
                        samples.clear();
                        float T = 1.f;
                        auto emit = [&](float t) {
                            Vec3f x = ray.at(t);
                            for (int a = 0; a < 3; ++a) x[a] = ngprt::clamp(x[a], -1.f, 1.f);
                            DeferredFeature<float> feat;
                            if (o->keep_level > 0) {
                                DeferredFeature<float> coarse;
                                AttentionParams<float> att;
                                std::array<DeferredFeature<float>, kMaxFineLevels> fine;
                                decode_point_baked_raw(s, x, coarse, att, fine);
                                auto masked = level_masked_fine(
                                    std::span<const DeferredFeature<float>>(fine.data(), L),
                                    o->keep_level);
                                feat = fuse(coarse,
                                            std::span<const DeferredFeature<float>>(masked), att,
                                            s.fusion);
                            } else {
                                feat = decode_point_baked(s, x);
                            }
                            samples.push_back({t, step, feat});
                            T = T * (1.f - alpha_from_sigma(activate_density(feat.sigma_pre()),
                                                            step));
                            return !(o->early_stop && T < float(kEarlyStopTransmittance));
                        };
                        mc = march(ray, s.pyramid, grid, step, o->max_step_rule != 0, emit);
                        auto acc = composite(std::span<const RaySample<float>>(samples),
                                             o->early_stop != 0);
                        if (acc.final_t < 1.f) {
                            Vec3f c = shade(acc, ray.dir, s.psi);
                            out[0] = c[0];
                            out[1] = c[1];
                            out[2] = c[2];
                        }
                    }
                } catch (const std::exception& e) {
#pragma omp critical
                    err = e.what();
                }
                if (stats) {
                    uint32_t* st = stats + 4 * pix;
                    st[0] = uint32_t(mc.marching_points);
                    st[1] = uint32_t(mc.occupied_points);
                    st[2] = uint32_t(mc.occ_grid_accesses);
                    st[3] = uint32_t(mc.dist_grid_accesses);
                }
            }
        }
        if (!err.empty()) {
            g_err = err;
            return 1;
        }
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// Pyramid levels 1..4 of the reference's build_pyramid, concatenated.
int ref_build_pyramid(const uint64_t* words, int res, uint64_t* out_levels) {
    auto p = build_pyramid(bitgrid_from_words(words, res));
    size_t off = 0;
    for (int k = 1; k < kPyramidLevels; ++k) {
        std::memcpy(out_levels + off, p.levels[k].words.data(),
                    p.levels[k].words.size() * sizeof(uint64_t));
        off += p.levels[k].words.size();
    }
    return 0;
}

int ref_build_distance_grid(const uint64_t* words, int res, uint8_t* out) {
    auto g = build_distance_grid(bitgrid_from_words(words, res));
    std::memcpy(out, g.values.data(), g.values.size());
    return 0;
}

uint64_t ref_hash_index(int res, uint64_t max_table_len, int x, int y, int z) {
    HashLevel<float> h;
    h.resolution = res;
    size_t corners = size_t(res + 1) * (res + 1) * (res + 1);
    h.addressing = corners <= max_table_len ? Addressing::Direct : Addressing::Hashed;
    h.table_len = corners <= max_table_len ? corners : max_table_len;
    return h.hash_index({x, y, z});
}

void ref_sh_encode(const float* dir, float* out16) {
    auto sh = sh_encode(Vec3f{dir[0], dir[1], dir[2]});
    for (int i = 0; i < kShDim; ++i) out16[i] = sh[i];
}

float ref_activate_density(float x) { return activate_density(x); }
float ref_activate_sigmoid(float x) { return activate_sigmoid(x); }
float ref_alpha(float sigma, float delta) { return alpha_from_sigma(sigma, delta); }
float ref_expf(float x) { return std::exp(x); }

// composite() over given (t, delta, feature) samples: out = [c_d(3), f(4), final_t, composited]
void ref_composite(int n, const float* t, const float* delta, const float* feat8, int early_stop,
                   float* out9) {
    std::vector<RaySample<float>> s(n);
    for (int i = 0; i < n; ++i) {
        s[i].t = t[i];
        s[i].delta = delta[i];
        for (int c = 0; c < 8; ++c) s[i].feature.v[c] = feat8[8 * i + c];
    }
    auto r = composite(std::span<const RaySample<float>>(s), early_stop != 0);
    for (int c = 0; c < 3; ++c) out9[c] = r.c_d[c];
    for (int c = 0; c < 4; ++c) out9[3 + c] = r.f[c];
    out9[7] = r.final_t;
    out9[8] = float(r.composited);
}

// decode_point_baked at a point (8 floats out).
int ref_decode_point(void* handle, const float* x3, int keep_level, float* out8) {
    try {
        const BakedScene& s = static_cast<const RefScene*>(handle)->s;
        Vec3f x{x3[0], x3[1], x3[2]};
        DeferredFeature<float> f;
        if (keep_level > 0) {
            DeferredFeature<float> coarse;
            AttentionParams<float> att;
            std::array<DeferredFeature<float>, kMaxFineLevels> fine;
            decode_point_baked_raw(s, x, coarse, att, fine);
            auto masked = level_masked_fine(
                std::span<const DeferredFeature<float>>(fine.data(), s.cfg.fine_levels),
                keep_level);
            f = fuse(coarse, std::span<const DeferredFeature<float>>(masked), att, s.fusion);
        } else {
            f = decode_point_baked(s, x);
        }
        for (int i = 0; i < 8; ++i) out8[i] = f.v[i];
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// shade() for given accumulations: acc = [c_d(3), f(4)], dir(3) -> rgb(3)
int ref_shade(void* handle, const float* acc7, const float* dir3, float* rgb3) {
    try {
        const BakedScene& s = static_cast<const RefScene*>(handle)->s;
        CompositeResult<float> a;
        for (int c = 0; c < 3; ++c) a.c_d[c] = acc7[c];
        for (int c = 0; c < 4; ++c) a.f[c] = acc7[3 + c];
        Vec3f rgb = shade(a, Vec3f{dir3[0], dir3[1], dir3[2]}, s.psi);
        for (int c = 0; c < 3; ++c) rgb3[c] = rgb[c];
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

// generate_rays for one pixel centre: returns ok, ray = [o(3), d(3), t_near, t_far]
int ref_generate_ray(const ngprt_camera* cam, double u, double v, float* ray8) {
    PosedDataset ds = dataset_of(*cam);
    Ray<float> r;
    bool ok = generate_rays(ds, 0, u, v, r);
    ray8[0] = r.origin.x; ray8[1] = r.origin.y; ray8[2] = r.origin.z;
    ray8[3] = r.dir.x; ray8[4] = r.dir.y; ray8[5] = r.dir.z;
    ray8[6] = r.t_near; ray8[7] = r.t_far;
    return ok ? 1 : 0;
}

// march() of one ray with a null emit-continue; records the empty-skip segments
// (t, t+s) for the SAFETY check against dda_oracle.
int ref_march_segments(void* handle, const float* ray8, float step, int use_grid,
                       int max_step_rule, uint32_t* counters4, float* seg, int max_seg,
                       float* samples_t, int max_samples, int* n_seg, int* n_samples) {
    const RefScene& r = *static_cast<const RefScene*>(handle);
    Ray<float> ray;
    ray.origin = {ray8[0], ray8[1], ray8[2]};
    ray.dir = {ray8[3], ray8[4], ray8[5]};
    ray.t_near = ray8[6];
    ray.t_far = ray8[7];
    std::vector<std::pair<float, float>> segs;
    std::vector<float> ts;
    auto mc = march(ray, r.s.pyramid, (use_grid && r.has_dist) ? &r.s.distance : nullptr, step,
                    max_step_rule != 0,
                    [&](float t) {
                        ts.push_back(t);
                        return true;
                    },
                    &segs);
    counters4[0] = uint32_t(mc.marching_points);
    counters4[1] = uint32_t(mc.occupied_points);
    counters4[2] = uint32_t(mc.occ_grid_accesses);
    counters4[3] = uint32_t(mc.dist_grid_accesses);
    *n_seg = int(segs.size());
    *n_samples = int(ts.size());
    for (int i = 0; i < int(segs.size()) && i < max_seg; ++i) {
        seg[2 * i] = segs[i].first;
        seg[2 * i + 1] = segs[i].second;
    }
    for (int i = 0; i < int(ts.size()) && i < max_samples; ++i) samples_t[i] = ts[i];
    return 0;
}

// dda_oracle (occupancy.hpp:366-417) over the level-0 grid: number of occupied
// voxels strictly inside (t0, t1) by more than eps (SPEC.md:414 boundary rule).
int ref_dda_hits(void* handle, const float* ray8, float t0, float t1, double eps) {
    const RefScene& r = *static_cast<const RefScene*>(handle);
    Ray<float> ray;
    ray.origin = {ray8[0], ray8[1], ray8[2]};
    ray.dir = {ray8[3], ray8[4], ray8[5]};
    ray.t_near = ray8[6];
    ray.t_far = ray8[7];
    auto hits = dda_oracle(ray, r.s.pyramid.levels[0], t0, t1);
    int n = 0;
    for (auto& h : hits)
        if (h.t_exit - h.t_entry > eps && h.t_exit > double(t0) + eps && h.t_entry < double(t1) - eps)
            ++n;
    return n;
}

// ---- pins for the synthetic-scene generator (paper_2407_10482_b200/csrc/synth.cpp) ----

// scene_occupancy(make_scene(name, seed), res) as packed words; returns box count or -1.
int ref_scene_occupancy(const char* name, uint64_t seed, int res, uint64_t* words) {
    try {
        auto sc = make_scene(name, seed);
        auto g = scene_occupancy(sc, res);
        std::memcpy(words, g.words.data(), g.words.size() * sizeof(uint64_t));
        return int(sc.boxes.size());
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

// the boxes of make_scene: lo(3) hi(3) sigma per box
int ref_scene_boxes(const char* name, uint64_t seed, double* out7, int max_boxes) {
    auto sc = make_scene(name, seed);
    int n = int(sc.boxes.size());
    for (int i = 0; i < n && i < max_boxes; ++i) {
        const auto& b = sc.boxes[i];
        double v[7] = {b.lo.x, b.lo.y, b.lo.z, b.hi.x, b.hi.y, b.hi.z, b.sigma};
        std::memcpy(out7 + 7 * i, v, sizeof v);
    }
    return n;
}

void ref_sphere_views(int n, double radius, double* out16n) {
    auto v = sphere_views(n, radius);
    for (int i = 0; i < n; ++i) std::memcpy(out16n + 16 * i, v[i].data(), 16 * sizeof(double));
}

// TinyMlp::init(widths, "psi", Rng(seed)) weights and biases, concatenated per layer.
void ref_tiny_mlp_init(const int* widths, int nw, uint64_t seed, float* w_out, float* b_out) {
    Rng rng(seed);
    TinyMlp<float> m;
    m.init(std::vector<int>(widths, widths + nw), "psi", rng, nullptr);
    size_t ow = 0, ob = 0;
    for (int k = 0; k < m.num_layers(); ++k) {
        std::memcpy(w_out + ow, m.weight[k].value.data(), m.weight[k].value.size() * sizeof(float));
        std::memcpy(b_out + ob, m.bias[k].value.data(), m.bias[k].value.size() * sizeof(float));
        ow += m.weight[k].value.size();
        ob += m.bias[k].value.size();
    }
}

// TinyMlp::forward (nn.hpp:175-196) on one input.
void ref_tiny_mlp_forward(const int* widths, int nw, const float* w, const float* b,
                          const float* in, float* out) {
    Rng rng(0);
    TinyMlp<float> m;
    m.init(std::vector<int>(widths, widths + nw), "m", rng, nullptr);
    size_t ow = 0, ob = 0;
    for (int k = 0; k < m.num_layers(); ++k) {
        std::memcpy(m.weight[k].value.data(), w + ow, m.weight[k].value.size() * sizeof(float));
        std::memcpy(m.bias[k].value.data(), b + ob, m.bias[k].value.size() * sizeof(float));
        ow += m.weight[k].value.size();
        ob += m.bias[k].value.size();
    }
    auto o = m.forward_alloc(std::span<const float>(in, size_t(widths[0])));
    std::memcpy(out, o.data(), o.size() * sizeof(float));
}

void ref_rng_uniform(uint64_t seed, double lo, double hi, uint64_t n, double* out) {
    Rng r(seed);
    for (uint64_t i = 0; i < n; ++i) out[i] = r.uniform(lo, hi);
}

uint32_t ref_crc32(const void* p, uint64_t n) { return crc32(p, n); }

// save_baked (baking.hpp:266-349) of a scene built by ref_scene_create.
int ref_save_baked(void* handle, const char* path) {
    try {
        save_baked(static_cast<RefScene*>(handle)->s, path);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

double ref_base_step() { return kBaseStep; }

// bake (baking.hpp:107-202) of the model a ngprt_model_desc describes, written
// with save_baked to `path`. The desc's arrays are copied into a reference
// NgpRtModel<float> (model.hpp:27-107) built by its own init.
int ref_bake(const ngprt_model_desc* md, const uint64_t* train_words, int train_res,
             const ngprt_bake_opts* o, const char* path) {
    try {
        EncodingConfig cfg;
        for (int k = 0; k < 6; ++k) cfg.coarse_resolutions[k] = int(md->coarse_res[k]);
        cfg.coarse_table_len = md->coarse_table_len;
        cfg.fine_levels = int(md->L);
        cfg.fine_table_len = md->fine_table_len[0];
        cfg.corner_grid_res = int(md->L_C);
        NgpRtModel<float> model;
        model.init(cfg, FusionTag(md->fusion_tag), 1);
        for (int k = 0; k < 6; ++k) {
            auto& v = model.encoding.coarse[k].entries.value;
            std::memcpy(v.data(), md->coarse_tables[k], v.size() * sizeof(float));
        }
        for (int k = 0; k < 2; ++k) {
            auto& w = model.aux.weight[k].value;
            auto& b = model.aux.bias[k].value;
            std::memcpy(w.data(), md->aux_w[k], w.size() * sizeof(float));
            std::memcpy(b.data(), md->aux_b[k], b.size() * sizeof(float));
        }
        for (int l = 0; l < int(md->L); ++l) {
            auto& lvl = model.encoding.fine[l];
            if (lvl.table_len != md->fine_table_len[l] || lvl.resolution != int(md->fine_res[l]))
                throw std::invalid_argument("ref_bake: fine level geometry differs from EncodingConfig");
            std::memcpy(lvl.entries.value.data(), md->fine_tables[l],
                        lvl.entries.value.size() * sizeof(float));
        }
        for (int k = 0; k < 3; ++k) {
            auto& w = model.psi.weight[k].value;
            auto& b = model.psi.bias[k].value;
            std::memcpy(w.data(), md->psi_w[k], w.size() * sizeof(float));
            std::memcpy(b.data(), md->psi_b[k], b.size() * sizeof(float));
        }
        if (fusion_is_invariant(model.fusion_tag))
            std::memcpy(model.fusion.global_pre.value.data(), md->att_globals,
                        model.fusion.global_pre.value.size() * sizeof(float));
        if (model.fusion_tag == FusionTag::Mlp)
            for (int k = 0; k < 2; ++k) {
                auto& w = model.fusion.mlp.weight[k].value;
                auto& b = model.fusion.mlp.bias[k].value;
                std::memcpy(w.data(), md->fusion_mlp_w[k], w.size() * sizeof(float));
                std::memcpy(b.data(), md->fusion_mlp_b[k], b.size() * sizeof(float));
            }
        BakeOptions opt;
        if (o) {
            if (o->cull_step > 0) opt.cull_step = o->cull_step;
            opt.cull_alpha_thresh = o->cull_alpha_thresh;
            opt.dilate_voxels = int(o->dilate_voxels);
        }
        BakedScene out = bake(model, bitgrid_from_words(train_words, train_res), opt);
        save_baked(out, path);
        return 0;
    } catch (const std::exception& e) {
        g_err = e.what();
        return 1;
    }
}

} // extern "C"
