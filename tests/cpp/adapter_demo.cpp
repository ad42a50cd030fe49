// tests/cpp/adapter_demo.cpp — drop-in demonstration (test infrastructure).
//
// Builds a BakedScene entirely with the reference's own functions (make_scene,
// scene_occupancy, build_pyramid, build_distance_grid, HashLevel, TinyMlp,
// FusionMode), renders it (a) with the reference's render path composed on the
// CPU exactly as SURVEY.md §8(c) and (b) on the B200 through include/ngprt_gpu.hpp,
// and compares with the reference's own max_abs_diff / psnr (image.hpp:89-110).
// Then bakes a reference NgpRtModel (model.hpp:27-107) with the reference's
// bake() and with ngprt::gpu::bake() and compares the two save_baked files.
// Feature values are NOT fp16-representable, so the GPU picks f32 storage.
// Prints one JSON line; tests/test_gpu_adapter.py checks it.
#include "ngprt_gpu.hpp"

#include <cstdio>
#include <fstream>
#include <iterator>
#include <unistd.h>

using namespace ngprt;

static BakedScene make_baked(uint64_t seed) {
    BakedScene s;
    s.cfg.corner_grid_res = 64;
    s.cfg.fine_levels = 2;
    s.cfg.fine_table_len = size_t(1) << 14;
    s.tag = FusionTag::SeparateAttV;
    Rng rng(seed);
    const SynthScene sc = make_scene("toy");
    s.pyramid = build_pyramid(scene_occupancy(sc, 128));
    s.distance = build_distance_grid(s.pyramid.levels[1]);
    const int lc = s.cfg.corner_grid_res, L = s.cfg.fine_levels;
    s.coarse.init(lc, L);
    BitGrid occ = scene_occupancy(sc, lc), marks(lc + 1);
    for (int z = 0; z < lc; ++z)
        for (int y = 0; y < lc; ++y)
            for (int x = 0; x < lc; ++x)
                if (occ.get(x, y, z))
                    for (int k = 0; k < 8; ++k) marks.set(x + (k & 1), y + ((k >> 1) & 1), z + (k >> 2));
    for (int z = 0; z <= lc; ++z)
        for (int y = 0; y <= lc; ++y)
            for (int x = 0; x <= lc; ++x) {
                if (!marks.get(x, y, z)) continue;
                float* row = s.coarse.add_row(s.coarse.key_of({x, y, z}));
                row[0] = float(rng.uniform(1.0, 5.0));
                for (int c = 1; c < 8 + 2 * L; ++c) row[c] = float(rng.uniform(-1.5, 1.5));
            }
    s.fine.resize(L);
    for (int l = 0; l < L; ++l) {
        s.fine[l].init("fine_l" + std::to_string(l + 1), s.cfg.fine_resolution(l),
                       s.cfg.fine_table_len, kFineFeatureDim);
        for (auto& v : s.fine[l].entries.value) v = float(rng.uniform(-1.0, 1.0));
    }
    s.psi.init({kShadeInWidth, 64, 64, 3}, "psi", rng, nullptr);
    for (int k = 0; k < 3; ++k)
        for (auto& b : s.psi.bias[k].value) b = float(rng.uniform(-0.1, 0.1));
    s.fusion.init(s.tag, L, rng, nullptr);
    return s;
}

// The canonical render_ray composition with reference functions.
static Image cpu_render(const BakedScene& s, const PosedDataset& ds, size_t f,
                        std::vector<MarchCounters>& mcs) {
    Image img(ds.width, ds.height);
    mcs.assign(size_t(ds.width) * ds.height, MarchCounters{});
    const float step = float(kBaseStep);
    for (int py = 0; py < ds.height; ++py)
        for (int px = 0; px < ds.width; ++px) {
            Ray<float> ray;
            if (!generate_rays(ds, f, px + 0.5, py + 0.5, ray)) continue;
            std::vector<RaySample<float>> samples;
            float T = 1.f;
            auto emit = [&](float t) {
                Vec3f x = ray.at(t);
                for (int a = 0; a < 3; ++a) x[a] = ngprt::clamp(x[a], -1.f, 1.f);
                auto feat = decode_point_baked(s, x);
                samples.push_back({t, step, feat});
                T = T * (1.f - alpha_from_sigma(activate_density(feat.sigma_pre()), step));
                return !(T < float(kEarlyStopTransmittance));
            };
            mcs[size_t(py) * ds.width + px] = march(ray, s.pyramid, &s.distance, step, false, emit);
            auto acc = composite(std::span<const RaySample<float>>(samples), true);
            if (acc.final_t < 1.f) {
                Vec3f c = shade(acc, ray.dir, s.psi);
                float* p = img.pixel(px, py);
                p[0] = c[0];
                p[1] = c[1];
                p[2] = c[2];
            }
        }
    return img;
}

static std::string slurp(const std::string& path) {
    std::ifstream f(path, std::ios::binary);
    return std::string(std::istreambuf_iterator<char>(f), std::istreambuf_iterator<char>());
}

// Reference model in the "desk" geometry (config.hpp:60-68) with non-trivial
// parameters, its training grid, both bakes, byte comparison of the files.
static bool bake_identical(size_t* corners) {
    RunConfig rc = RunConfig::desk();
    NgpRtModel<float> m;
    m.init(rc.enc, FusionTag::SeparateAttV, 7);
    Rng rng(99);
    for (auto& lvl : m.encoding.coarse)
        for (auto& v : lvl.entries.value) v = float(rng.uniform(-1.0, 1.0));
    for (auto& lvl : m.encoding.fine)
        for (auto& v : lvl.entries.value) v = float(rng.uniform(-0.5, 0.5));
    m.aux.bias[1].value[0] = -0.5f;  // density offset: the cull keeps about half the voxels
    const BitGrid grid = scene_occupancy(make_scene("toy"), rc.train_grid_res);
    const BakedScene rb = bake(m, grid);
    const BakedScene gb = gpu::bake(m, grid);
    const std::string pa = "/tmp/adapter_demo_ref_" + std::to_string(getpid()) + ".ngrt";
    const std::string pb = "/tmp/adapter_demo_gpu_" + std::to_string(getpid()) + ".ngrt";
    save_baked(rb, pa);
    save_baked(gb, pb);
    const bool same = slurp(pa) == slurp(pb) && !slurp(pa).empty();
    std::remove(pa.c_str());
    std::remove(pb.c_str());
    *corners = gb.coarse.count();
    return same;
}

int main() {
    const BakedScene s = make_baked(2024);
    PosedDataset ds;
    ds.width = 64;
    ds.height = 48;
    ds.fx = ds.fy = 1.1 * ds.width;
    ds.cx = 0.5 * ds.width;
    ds.cy = 0.5 * ds.height;
    for (auto& m : sphere_views(3, 2.9)) ds.frames.push_back({"", m});
    gpu::Scene gs(s);
    double worst_exact = 0, worst_tc = 0, min_psnr_tc = 99;
    long counter_mismatch = 0;
    for (size_t f = 0; f < ds.frames.size(); ++f) {
        std::vector<MarchCounters> ref_mc, gpu_mc;
        const Image ref = cpu_render(s, ds, f, ref_mc);
        gpu::RenderOptions exact;
        exact.exact_mlp = true;
        const Image g_exact = gs.render(ds, f, exact, &gpu_mc);
        const Image g_tc = gs.render(ds, f);
        worst_exact = std::max(worst_exact, max_abs_diff(ref, g_exact));
        worst_tc = std::max(worst_tc, max_abs_diff(ref, g_tc));
        min_psnr_tc = std::min(min_psnr_tc, psnr(ref, g_tc));
        for (size_t i = 0; i < ref_mc.size(); ++i)
            counter_mismatch += ref_mc[i].marching_points != gpu_mc[i].marching_points ||
                                ref_mc[i].occupied_points != gpu_mc[i].occupied_points ||
                                ref_mc[i].occ_grid_accesses != gpu_mc[i].occ_grid_accesses ||
                                ref_mc[i].dist_grid_accesses != gpu_mc[i].dist_grid_accesses;
    }
    // serving path: every frame enqueued, one wait; equals the synchronous render
    long async_mismatch = 0;
    {
        std::vector<Image> imgs(ds.frames.size());
        for (size_t f = 0; f < ds.frames.size(); ++f) gs.render_async(ds, f, imgs[f]);
        gs.wait();
        for (size_t f = 0; f < ds.frames.size(); ++f) {
            const Image sync = gs.render(ds, f);
            async_mismatch += max_abs_diff(sync, imgs[f]) != 0.0;
        }
    }
    // multi-device drop-in (ngprt_multi_*): one device (NCCL communicator from
    // ncclCommInitAll) and two replicas on device 0 (peer-copy gather); tile and
    // camera sharding both equal the single-scene render
    long multi_mismatch = 0;
    bool multi_nccl = false;
    {
        gpu::RenderOptions exact;
        exact.exact_mlp = true;
        gpu::MultiScene one(s, {0});
        multi_nccl = one.uses_nccl();
        gpu::MultiScene two(s, {0, 0});
        std::vector<size_t> all;
        for (size_t f = 0; f < ds.frames.size(); ++f) all.push_back(f);
        const std::vector<Image> cams_one = one.render_cameras(ds, all, exact);
        const std::vector<Image> cams_two = two.render_cameras(ds, all, exact);
        for (size_t f = 0; f < ds.frames.size(); ++f) {
            const Image want = gs.render(ds, f, exact);
            multi_mismatch += max_abs_diff(want, one.render(ds, f, exact, 16)) != 0.0;
            multi_mismatch += max_abs_diff(want, two.render(ds, f, exact, 8)) != 0.0;
            multi_mismatch += max_abs_diff(want, cams_one[f]) != 0.0;
            multi_mismatch += max_abs_diff(want, cams_two[f]) != 0.0;
        }
    }
    ngprt_scene_info info{};
    ngprt_scene_info_get(gs.handle(), &info);
    size_t bake_corners = 0;
    const bool bake_same = bake_identical(&bake_corners);
    std::printf("{\"frames\": %zu, \"max_abs_exact\": %.9g, \"max_abs_tensor\": %.9g, "
                "\"psnr_tensor\": %.3f, \"counter_mismatch\": %ld, \"storage\": %d, "
                "\"bake_identical\": %s, \"bake_corners\": %zu, \"async_mismatch\": %ld, "
                "\"multi_mismatch\": %ld, \"multi_nccl\": %s}\n",
                ds.frames.size(), worst_exact, worst_tc, min_psnr_tc, counter_mismatch,
                int(info.storage), bake_same ? "true" : "false", bake_corners, async_mismatch,
                multi_mismatch, multi_nccl ? "true" : "false");
    return 0;
}
