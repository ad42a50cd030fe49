// ngprt_gpu.hpp — header-only C++ adapter from the reference's own types to the
// B200 C ABI (ngprt_cuda.h). This is the binding a maintainer of the reference
// adds to route its render path to the GPU:
//
//     #include "ngprt/baking.hpp"     // reference: BakedScene, PosedDataset, Image
//     #include "ngprt_gpu.hpp"
//     ngprt::gpu::Scene gs(baked);                  // upload once (ngprt_scene_create)
//     ngprt::Image img = gs.render(dataset, frame); // == render_ray over every pixel
//     ngprt::BakedScene b = ngprt::gpu::bake(model, train_grid, opts);  // == bake()
//     ngprt::gpu::MultiScene ms(baked, {0, 1, 2, 3});  // replicas, NCCL gather to GPU 0
//     ngprt::Image big = ms.render(dataset, frame);     // tiles over 4 GPUs, same Image
//
// Requires the reference headers (/root/reference/proj/include) on the include
// path and links against paper_2407_10482_b200/_lib/libngprt_cuda.so (and
// libcudart for MultiScene's device output buffer).
// Errors surface as std::runtime_error carrying ngprt_last_error(), like the
// reference's own exceptions.
#pragma once

#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "ngprt/baking.hpp"
#include "ngprt/config.hpp"
#include "ngprt/scene.hpp"

#include <cuda_runtime.h>  // MultiScene's devices[0] output buffer

#include "ngprt_cuda.h"

namespace ngprt::gpu {

struct RenderOptions {
    float step = float(kBaseStep);  // march step gamma * s0 (config.hpp:11)
    bool use_dist_grid = true;      // march(..., &distance, ...) vs nullptr
    bool max_step_rule = false;     // occupancy.hpp:272
    bool early_stop = true;         // volume.hpp:70
    int keep_level = 0;             // level_masked_fine (fusion.hpp:198-209); 0 = off
    bool exact_mlp = false;         // bit-exact CUDA-core shade instead of tcgen05
};

inline void check(ngprt_status s, const char* what) {
    if (s != NGPRT_OK) throw std::runtime_error(std::string(what) + ": " + ngprt_last_error());
}

// A BakedScene resident on one B200 (immutable).
class Scene {
public:
    // The C-ABI view of a reference BakedScene (pointers into `s`, plus the coarse
    // keys in row order, which SparseCoarseGrid keeps only in its hash map).
    struct Desc {
        ngprt_scene_desc desc{};
        std::vector<uint64_t> keys;
        explicit Desc(const BakedScene& s) {
            ngprt_scene_desc& d = desc;
            const int L = s.cfg.fine_levels;
            d.L = uint32_t(L);
            d.L_C = uint32_t(s.cfg.corner_grid_res);
            // SparseCoarseGrid (baking.hpp:11-50): keys in row order
            keys.resize(s.coarse.index.size());
            for (const auto& kv : s.coarse.index) keys[kv.second] = kv.first;
            d.n_coarse = keys.size();
            d.coarse_keys = keys.data();
            d.coarse_rows = s.coarse.rows.data();
            for (int l = 0; l < L; ++l) {
                d.fine_res[l] = uint32_t(s.fine[l].resolution);
                d.fine_table_len[l] = s.fine[l].table_len;
                d.fine_hashed[l] = s.fine[l].addressing == Addressing::Hashed ? 1 : 0;
                d.fine_tables[l] = s.fine[l].entries.value.data();
            }
            for (int k = 0; k < 3; ++k) {
                d.psi_w[k] = s.psi.weight[k].value.data();
                d.psi_b[k] = s.psi.bias[k].value.data();
            }
            d.fusion_tag = uint8_t(s.tag);
            d.att_globals = fusion_is_invariant(s.tag) ? s.fusion.global_pre.value.data() : nullptr;
            if (s.tag == FusionTag::Mlp)
                for (int k = 0; k < 2; ++k) {
                    d.fusion_mlp_w[k] = s.fusion.mlp.weight[k].value.data();
                    d.fusion_mlp_b[k] = s.fusion.mlp.bias[k].value.data();
                }
            d.occ_base_res = uint32_t(s.pyramid.levels[0].res);
            for (int k = 0; k < kPyramidLevels; ++k) d.pyramid_words[k] = s.pyramid.levels[k].words.data();
            d.dist_res = uint32_t(s.distance.resolution);
            d.dist_values = s.distance.values.empty() ? nullptr : s.distance.values.data();
        }
    };

    explicit Scene(const BakedScene& s, int device = 0) {
        Desc d(s);
        check(ngprt_scene_create(&d.desc, device, &h_), "ngprt_scene_create");
    }
    ~Scene() { ngprt_scene_destroy(h_); }
    Scene(const Scene&) = delete;
    Scene& operator=(const Scene&) = delete;

    // Renders frame `frame` of `ds` (scene.hpp:191-228 camera model) into an Image
    // (image.hpp:12-22); optionally returns the per-ray MarchCounters.
    Image render(const PosedDataset& ds, size_t frame, const RenderOptions& o = {},
                 std::vector<MarchCounters>* counters = nullptr) const {
        if (frame >= ds.frames.size()) throw std::out_of_range("render: bad frame index");
        const ngprt_camera cam = camera_of(ds, frame);
        const ngprt_render_opts ro = opts_of(o);
        Image img(ds.width, ds.height);
        std::vector<ngprt_ray_stats> st(counters ? size_t(ds.width) * ds.height : 0);
        check(ngprt_render_host(h_, &cam, 1, &ro, img.rgb.data(), counters ? st.data() : nullptr),
              "ngprt_render_host");
        if (counters) {
            counters->resize(st.size());
            for (size_t i = 0; i < st.size(); ++i) {
                (*counters)[i].marching_points = st[i].marching;
                (*counters)[i].occupied_points = st[i].occupied;
                (*counters)[i].occ_grid_accesses = st[i].occ_acc;
                (*counters)[i].dist_grid_accesses = st[i].dist_acc;
            }
        }
        return img;
    }

    // Serving: enqueue frame `frame` into `img` (sized ds.width x ds.height) and
    // return; the device->host copy overlaps the next enqueued frame's march
    // (ngprt_render_host_async). `img` must stay alive until wait().
    void render_async(const PosedDataset& ds, size_t frame, Image& img,
                      const RenderOptions& o = {}) const {
        if (frame >= ds.frames.size()) throw std::out_of_range("render: bad frame index");
        if (img.width != ds.width || img.height != ds.height) img = Image(ds.width, ds.height);
        const ngprt_camera cam = camera_of(ds, frame);
        const ngprt_render_opts ro = opts_of(o);
        check(ngprt_render_host_async(h_, &cam, 1, &ro, img.rgb.data(), nullptr),
              "ngprt_render_host_async");
    }
    void wait() const { check(ngprt_render_host_wait(h_), "ngprt_render_host_wait"); }

    ngprt_scene* handle() const { return h_; }

    static ngprt_camera camera_of(const PosedDataset& ds, size_t frame) {
        ngprt_camera cam{};
        for (int i = 0; i < 16; ++i) cam.c2w[i] = ds.frames[frame].c2w[i];
        cam.fx = ds.fx;
        cam.fy = ds.fy;
        cam.cx = ds.cx;
        cam.cy = ds.cy;
        cam.width = uint32_t(ds.width);
        cam.height = uint32_t(ds.height);
        return cam;
    }
    static ngprt_render_opts opts_of(const RenderOptions& o) {
        ngprt_render_opts ro{};
        ro.step = o.step;
        ro.use_dist_grid = o.use_dist_grid;
        ro.max_step_rule = o.max_step_rule;
        ro.early_stop = o.early_stop;
        ro.keep_level = int8_t(o.keep_level);
        ro.mlp_mode = o.exact_mlp ? NGPRT_MLP_EXACT : NGPRT_MLP_TENSOR;
        return ro;
    }

private:
    ngprt_scene* h_ = nullptr;
};

// A BakedScene replicated on several B200s driven from this one process
// (ngprt_multi_*): every frame is split into interleaved
// tile x tile tiles rendered by all devices at once (one launch per device),
// gathered to devices[0] over NCCL (ncclCommInitAll) and returned as one Image,
// identical to Scene::render's. render_cameras() gives each device whole frames.
class MultiScene {
public:
    MultiScene(const BakedScene& s, std::vector<int> devices) : devices_(std::move(devices)) {
        Scene::Desc d(s);
        check(ngprt_multi_create(&d.desc, devices_.data(), int(devices_.size()), &h_),
              "ngprt_multi_create");
    }
    ~MultiScene() { ngprt_multi_destroy(h_); }
    MultiScene(const MultiScene&) = delete;
    MultiScene& operator=(const MultiScene&) = delete;
    bool uses_nccl() const { return ngprt_multi_uses_nccl(h_) != 0; }

    Image render(const PosedDataset& ds, size_t frame, const RenderOptions& o = {},
                 uint32_t tile = 32) const {
        if (frame >= ds.frames.size()) throw std::out_of_range("render: bad frame index");
        const ngprt_camera cam = Scene::camera_of(ds, frame);
        const ngprt_render_opts ro = Scene::opts_of(o);
        return run(&cam, 1, [&](float* rgb) {
            return ngprt_multi_render_tiles(h_, &cam, 1, &ro, tile, rgb, nullptr, nullptr);
        })[0];
    }
    // Frames `frames` of ds, frame i rendered whole by device i % n (camera sharding).
    std::vector<Image> render_cameras(const PosedDataset& ds, const std::vector<size_t>& frames,
                                      const RenderOptions& o = {}) const {
        std::vector<ngprt_camera> cams;
        for (size_t f : frames) {
            if (f >= ds.frames.size()) throw std::out_of_range("render: bad frame index");
            cams.push_back(Scene::camera_of(ds, f));
        }
        const ngprt_render_opts ro = Scene::opts_of(o);
        return run(cams.data(), int(cams.size()), [&](float* rgb) {
            return ngprt_multi_render_cameras(h_, cams.data(), int(cams.size()), &ro, rgb, nullptr,
                                              nullptr);
        });
    }

private:
    // Renders into a devices[0] buffer (legacy stream) and copies the frames out.
    template <class F>
    std::vector<Image> run(const ngprt_camera* cams, int n, F&& call) const {
        const size_t px = size_t(cams[0].width) * cams[0].height;
        float* d = nullptr;
        if (cudaSetDevice(devices_[0]) != cudaSuccess || cudaMalloc(&d, px * n * 12) != cudaSuccess)
            throw std::runtime_error("MultiScene: device allocation failed");
        std::unique_ptr<float, cudaError_t (*)(void*)> guard(d, cudaFree);
        check(call(d), "ngprt_multi_render");
        std::vector<Image> out;
        for (int i = 0; i < n; ++i) {
            out.emplace_back(int(cams[0].width), int(cams[0].height));
            if (cudaMemcpy(out.back().rgb.data(), d + px * 3 * i, px * 12, cudaMemcpyDeviceToHost) !=
                cudaSuccess)
                throw std::runtime_error("MultiScene: device-to-host copy failed");
        }
        return out;
    }
    std::vector<int> devices_;
    ngprt_multi* h_ = nullptr;
};

// One-shot convenience: upload, render one frame.
inline Image render(const BakedScene& s, const PosedDataset& ds, size_t frame,
                    const RenderOptions& o = {}, int device = 0) {
    return Scene(s, device).render(ds, frame, o);
}

// bake (baking.hpp:107-202) on the GPU: the same model, training grid and
// options in, the same BakedScene out (save_baked writes the reference's file
// byte for byte; tests/test_bake.py, tests/cpp/adapter_demo.cpp).
inline BakedScene bake(const NgpRtModel<float>& model, const BitGrid& train_grid,
                       const BakeOptions& opt = {}, int device = 0) {
    const int L = model.cfg.fine_levels, lc = model.corner_res(), w = model.decoder_width();
    ngprt_model_desc d{};
    d.L = uint32_t(L);
    d.L_C = uint32_t(lc);
    d.coarse_table_len = model.cfg.coarse_table_len;
    for (int k = 0; k < kCoarseLevels; ++k) {
        d.coarse_res[k] = uint32_t(model.encoding.coarse[k].resolution);
        d.coarse_tables[k] = model.encoding.coarse[k].entries.value.data();
    }
    for (int k = 0; k < 2; ++k) {
        d.aux_w[k] = model.aux.weight[k].value.data();
        d.aux_b[k] = model.aux.bias[k].value.data();
    }
    for (int l = 0; l < L; ++l) {
        const auto& f = model.encoding.fine[l];
        d.fine_res[l] = uint32_t(f.resolution);
        d.fine_table_len[l] = f.table_len;
        d.fine_hashed[l] = f.addressing == Addressing::Hashed ? 1 : 0;
        d.fine_tables[l] = f.entries.value.data();
    }
    for (int k = 0; k < 3; ++k) {
        d.psi_w[k] = model.psi.weight[k].value.data();
        d.psi_b[k] = model.psi.bias[k].value.data();
    }
    d.fusion_tag = uint8_t(model.fusion_tag);
    if (fusion_is_invariant(model.fusion_tag)) d.att_globals = model.fusion.global_pre.value.data();
    if (model.fusion_tag == FusionTag::Mlp)
        for (int k = 0; k < 2; ++k) {
            d.fusion_mlp_w[k] = model.fusion.mlp.weight[k].value.data();
            d.fusion_mlp_b[k] = model.fusion.mlp.bias[k].value.data();
        }
    const ngprt_bake_opts o{opt.cull_step, opt.cull_alpha_thresh, uint32_t(opt.dilate_voxels), 0};
    ngprt_baked* raw = nullptr;
    check(ngprt_bake(&d, train_grid.words.data(), uint32_t(train_grid.res), &o, device, &raw),
          "ngprt_bake");
    std::unique_ptr<ngprt_baked, void (*)(ngprt_baked*)> b(raw, ngprt_baked_free);
    const ngprt_scene_desc& r = *ngprt_baked_desc(b.get());

    BakedScene out;  // assembled as bake() does (baking.hpp:114-116, 137-200)
    out.cfg = model.cfg;
    out.tag = model.fusion_tag;
    out.coarse.init(lc, L);
    out.coarse.rows.assign(r.coarse_rows, r.coarse_rows + r.n_coarse * size_t(w));
    out.coarse.index.reserve(r.n_coarse);
    for (uint64_t i = 0; i < r.n_coarse; ++i) out.coarse.index.emplace(r.coarse_keys[i], uint32_t(i));
    out.fine.resize(L);
    for (int l = 0; l < L; ++l) {
        const auto& f = model.encoding.fine[l];
        out.fine[l].resolution = f.resolution;
        out.fine[l].table_len = f.table_len;
        out.fine[l].feature_dim = f.feature_dim;
        out.fine[l].addressing = f.addressing;
        out.fine[l].entries.init("fine_l" + std::to_string(l + 1), f.entries.size(), false);
        out.fine[l].entries.value = f.entries.value;
    }
    Rng dummy(0);
    out.psi.init({kShadeInWidth, 64, 64, 3}, "psi", dummy, nullptr);
    for (int k = 0; k < out.psi.num_layers(); ++k) {
        out.psi.weight[k].value = model.psi.weight[k].value;
        out.psi.bias[k].value = model.psi.bias[k].value;
    }
    out.fusion.init(model.fusion_tag, L, dummy, nullptr);
    if (fusion_is_invariant(model.fusion_tag)) out.fusion.global_pre.value = model.fusion.global_pre.value;
    if (model.fusion_tag == FusionTag::Mlp)
        for (int k = 0; k < out.fusion.mlp.num_layers(); ++k) {
            out.fusion.mlp.weight[k].value = model.fusion.mlp.weight[k].value;
            out.fusion.mlp.bias[k].value = model.fusion.mlp.bias[k].value;
        }
    for (int k = 0; k < kPyramidLevels; ++k) {
        out.pyramid.levels[k] = BitGrid(int(r.occ_base_res) >> k);
        std::copy(r.pyramid_words[k], r.pyramid_words[k] + out.pyramid.levels[k].words.size(),
                  out.pyramid.levels[k].words.begin());
    }
    out.distance.resolution = int(r.dist_res);
    out.distance.voxel_size = Roi::extent / r.dist_res;
    out.distance.values.assign(r.dist_values,
                               r.dist_values + size_t(r.dist_res) * r.dist_res * r.dist_res);
    return out;
}

}  // namespace ngprt::gpu
