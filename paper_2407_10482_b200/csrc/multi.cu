// multi.cu — interleaved-tile shard assembly and single-process multi-device
// rendering (include/ngprt_cuda.h: ngprt_shard_*, ngprt_multi_*).
//
// rays are independent and the scene is read-only
// (SPEC.md:329-330), so the path shards with no data-path collective. Each
// device holds a scene replica and renders either its interleaved tiles of the
// frame (one K0/K1/K2 launch into a compact per-rank buffer, see
// ngprt_render_opts.shard_*) or whole cameras; the only exchange is the gather
// of finished pixels to devices[0]: grouped ncclSend/ncclRecv issued on the
// render streams, so each device's transfer starts as soon as its own render
// ends. NCCL is loaded at run time (dlopen libnccl.so.2); the render path
// itself never links it.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <mutex>
#include <string>
#include <vector>

#include "render.cuh"

namespace ngprt_host {
void set_error(const std::string& msg);
}

namespace {

using ngprt_host::set_error;

ngprt_status fail(ngprt_status s, const std::string& msg) {
    set_error(msg);
    return s;
}

#define MG_CUDA(call)                                                                 \
    do {                                                                              \
        cudaError_t e_ = (call);                                                      \
        if (e_ != cudaSuccess)                                                        \
            return fail(e_ == cudaErrorMemoryAllocation ? NGPRT_ENOMEM : NGPRT_ECUDA, \
                        std::string(#call) + ": " + cudaGetErrorString(e_));          \
    } while (0)

uint64_t shard_pixels(uint32_t w, uint32_t h, uint32_t world, uint32_t tile) {
    const uint64_t t = tile ? tile : 32u, n = world ? world : 1u;
    const uint64_t tiles = ((w + t - 1) / t) * ((h + t - 1) / t);
    return (tiles + n - 1) / n * t * t;
}

// frames[cam][y][x][c] <- shards[rank][cam][local tile j][ly][lx][c] with global
// tile T = (y / tile) * tiles_x + x / tile, rank = T % world, j = T / world.
// One thread per output element; reads are contiguous along x inside a tile row.
__global__ void shard_assemble_kernel(const float* __restrict__ shards, uint32_t world,
                                      uint32_t n_cams, uint32_t w, uint32_t h, uint32_t tile,
                                      uint32_t ch, uint64_t per_cam, float* __restrict__ frames) {
    const uint64_t n = uint64_t(n_cams) * h * w * ch;
    const uint32_t tiles_x = (w + tile - 1) / tile;
    for (uint64_t i = blockIdx.x * uint64_t(blockDim.x) + threadIdx.x; i < n;
         i += uint64_t(gridDim.x) * blockDim.x) {
        const uint32_t c = uint32_t(i % ch);
        const uint64_t pix = i / ch;
        const uint32_t x = uint32_t(pix % w);
        const uint64_t r = pix / w;
        const uint32_t y = uint32_t(r % h), cam = uint32_t(r / h);
        const uint32_t T = (y / tile) * tiles_x + x / tile;
        const uint32_t rank = T % world, j = T / world;
        const uint64_t src = ((uint64_t(rank) * n_cams + cam) * per_cam + uint64_t(j) * tile * tile +
                              uint64_t(y % tile) * tile + (x % tile)) * ch + c;
        frames[i] = shards[src];
    }
}

// ---- NCCL, resolved at run time ----
struct Nccl {
    bool ok = false;
    std::string why;
    ncclResult_t (*CommInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    const char* (*ErrorString)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = nullptr;
        for (const char* name : {"libnccl.so.2", "libnccl.so"})
            if ((h = dlopen(name, RTLD_NOW | RTLD_GLOBAL))) break;
        if (!h) {
            n.why = std::string("dlopen libnccl.so.2 failed: ") + dlerror();
            return;
        }
        auto sym = [&](auto& fp, const char* s) {
            fp = reinterpret_cast<std::remove_reference_t<decltype(fp)>>(dlsym(h, s));
            return fp != nullptr;
        };
        n.ok = sym(n.CommInitAll, "ncclCommInitAll") && sym(n.CommDestroy, "ncclCommDestroy") &&
               sym(n.GroupStart, "ncclGroupStart") && sym(n.GroupEnd, "ncclGroupEnd") &&
               sym(n.Send, "ncclSend") && sym(n.Recv, "ncclRecv") &&
               sym(n.ErrorString, "ncclGetErrorString");
        if (!n.ok) n.why = "libnccl.so.2 lacks a needed symbol";
    });
    return n;
}

#define MG_NCCL(call)                                                                        \
    do {                                                                                     \
        ncclResult_t r_ = (call);                                                            \
        if (r_ != ncclSuccess)                                                               \
            return fail(NGPRT_ENCCL, std::string(#call) + ": " + nccl().ErrorString(r_));    \
    } while (0)

template <class T>
ngprt_status grow(int dev, T** p, size_t* cap, size_t n) {
    if (*cap >= n) return NGPRT_OK;
    MG_CUDA(cudaSetDevice(dev));
    if (*p) cudaFree(*p);
    *p = nullptr;
    *cap = 0;
    MG_CUDA(cudaMalloc(p, n * sizeof(T)));
    *cap = n;
    return NGPRT_OK;
}

}  // namespace

struct ngprt_multi {
    std::vector<int> dev;
    std::vector<ngprt_scene*> scene;
    std::vector<cudaStream_t> st;      // render + transfer stream per device ([0] unused: caller's)
    std::vector<cudaEvent_t> rendered; // per device, for the peer-copy gather
    cudaEvent_t start = nullptr;       // on the caller's stream: the other devices wait for it
    bool use_nccl = false;
    std::vector<ncclComm_t> comm;
    std::vector<float*> rgb;           // per-device compact outputs ([0] unused for tiles)
    std::vector<size_t> rgb_cap;
    std::vector<ngprt_ray_stats*> stats;
    std::vector<size_t> stats_cap;
    float* grgb = nullptr;             // devices[0]: gathered shard outputs
    size_t grgb_cap = 0;
    ngprt_ray_stats* gstats = nullptr;
    size_t gstats_cap = 0;
    std::mutex mu;                     // one multi-device call at a time

    ~ngprt_multi() {
        for (size_t i = 0; i < dev.size(); ++i) {
            cudaSetDevice(dev[i]);
            if (i < st.size() && st[i]) cudaStreamSynchronize(st[i]);
        }
        if (use_nccl)
            for (ncclComm_t c : comm)
                if (c) nccl().CommDestroy(c);
        for (size_t i = 0; i < dev.size(); ++i) {
            cudaSetDevice(dev[i]);
            if (i < st.size() && st[i]) cudaStreamDestroy(st[i]);
            if (i < rendered.size() && rendered[i]) cudaEventDestroy(rendered[i]);
            if (i < rgb.size() && rgb[i]) cudaFree(rgb[i]);
            if (i < stats.size() && stats[i]) cudaFree(stats[i]);
            if (i < scene.size() && scene[i]) ngprt_scene_destroy(scene[i]);
        }
        if (!dev.empty()) {
            cudaSetDevice(dev[0]);
            if (start) cudaEventDestroy(start);
            if (grgb) cudaFree(grgb);
            if (gstats) cudaFree(gstats);
        }
    }
};

namespace {

// The other devices' streams wait for the caller's stream (their buffers may still
// be read by the previous call's gather, which stream0 has already ordered).
ngprt_status fork(ngprt_multi* m, cudaStream_t s0) {
    MG_CUDA(cudaSetDevice(m->dev[0]));
    MG_CUDA(cudaEventRecord(m->start, s0));
    for (size_t i = 1; i < m->dev.size(); ++i) {
        MG_CUDA(cudaSetDevice(m->dev[i]));
        MG_CUDA(cudaStreamWaitEvent(m->st[i], m->start, 0));
    }
    return NGPRT_OK;
}

// Copy `bytes` from device i's buffer to devices[0] (peer path, repeated devices).
ngprt_status peer_copy(ngprt_multi* m, size_t i, void* dst0, const void* src, size_t bytes,
                       cudaStream_t s0) {
    MG_CUDA(cudaSetDevice(m->dev[0]));
    MG_CUDA(cudaStreamWaitEvent(s0, m->rendered[i], 0));
    MG_CUDA(cudaMemcpyPeerAsync(dst0, m->dev[0], src, m->dev[i], bytes, s0));
    return NGPRT_OK;
}

}  // namespace

extern "C" {

uint64_t ngprt_shard_pixels(uint32_t w, uint32_t h, uint32_t world, uint32_t tile) {
    return shard_pixels(w, h, world, tile);
}

ngprt_status ngprt_shard_assemble(const float* shards, uint32_t world, uint32_t n_cams, uint32_t w,
                                  uint32_t h, uint32_t tile, uint32_t channels, float* frames,
                                  void* stream) {
    if (!shards || !frames || world == 0 || channels == 0)
        return fail(NGPRT_EINVAL, "ngprt_shard_assemble: bad argument");
    tile = tile ? tile : 32u;
    if (tile % 8) return fail(NGPRT_EINVAL, "ngprt_shard_assemble: tile must be a multiple of 8");
    if (!n_cams || !w || !h) return NGPRT_OK;
    const uint64_t per_cam = shard_pixels(w, h, world, tile);
    const uint64_t n = uint64_t(n_cams) * w * h * channels;
    const unsigned blocks = unsigned(std::min<uint64_t>((n + 255) / 256, 148 * 16));
    shard_assemble_kernel<<<blocks, 256, 0, static_cast<cudaStream_t>(stream)>>>(
        shards, world, n_cams, w, h, tile, channels, per_cam, frames);
    MG_CUDA(cudaGetLastError());
    return NGPRT_OK;
}

ngprt_status ngprt_multi_create(const ngprt_scene_desc* desc, const int* devices, int n_dev,
                                ngprt_multi** out) {
    const ngprt_dev::DeviceRestore keep;
    if (!desc || !devices || n_dev < 1 || !out) return fail(NGPRT_EINVAL, "ngprt_multi_create: bad argument");
    *out = nullptr;
    auto* m = new ngprt_multi;
    m->dev.assign(devices, devices + n_dev);
    m->scene.assign(n_dev, nullptr);
    m->st.assign(n_dev, nullptr);
    m->rendered.assign(n_dev, nullptr);
    m->rgb.assign(n_dev, nullptr);
    m->rgb_cap.assign(n_dev, 0);
    m->stats.assign(n_dev, nullptr);
    m->stats_cap.assign(n_dev, 0);
    auto bail = [&](ngprt_status s) {
        delete m;
        return s;
    };
    for (int i = 0; i < n_dev; ++i) {
        if (const ngprt_status s = ngprt_scene_create(desc, devices[i], &m->scene[i])) return bail(s);
        if (cudaSetDevice(devices[i]) != cudaSuccess ||
            cudaStreamCreateWithFlags(&m->st[i], cudaStreamNonBlocking) != cudaSuccess ||
            cudaEventCreateWithFlags(&m->rendered[i], cudaEventDisableTiming) != cudaSuccess)
            return bail(fail(NGPRT_ECUDA, "ngprt_multi_create: stream/event creation failed"));
    }
    cudaSetDevice(devices[0]);
    if (cudaEventCreateWithFlags(&m->start, cudaEventDisableTiming) != cudaSuccess)
        return bail(fail(NGPRT_ECUDA, "ngprt_multi_create: event creation failed"));
    // NCCL needs distinct devices; replicas sharing a GPU gather by peer copies
    std::vector<int> sorted(m->dev);
    std::sort(sorted.begin(), sorted.end());
    const bool distinct = std::adjacent_find(sorted.begin(), sorted.end()) == sorted.end();
    if (distinct) {
        const Nccl& n = nccl();
        if (!n.ok) return bail(fail(NGPRT_ENCCL, n.why));
        m->comm.assign(n_dev, nullptr);
        const ncclResult_t r = n.CommInitAll(m->comm.data(), n_dev, devices);
        if (r != ncclSuccess) {
            m->comm.clear();
            return bail(fail(NGPRT_ENCCL, std::string("ncclCommInitAll: ") + n.ErrorString(r)));
        }
        m->use_nccl = true;
    }
    *out = m;
    return NGPRT_OK;
}

void ngprt_multi_destroy(ngprt_multi* m) {
    const ngprt_dev::DeviceRestore keep;
    delete m;
}

int ngprt_multi_uses_nccl(const ngprt_multi* m) { return m && m->use_nccl ? 1 : 0; }

const ngprt_scene* ngprt_multi_scene(const ngprt_multi* m, int i) {
    return (m && i >= 0 && i < int(m->scene.size())) ? m->scene[i] : nullptr;
}

ngprt_status ngprt_multi_render_tiles(ngprt_multi* m, const ngprt_camera* cams, int n_cams,
                                      const ngprt_render_opts* opts, uint32_t tile, float* rgb0,
                                      ngprt_ray_stats* stats0, void* stream0) {
    const ngprt_dev::DeviceRestore keep;
    const ngprt_dev::NvtxRange range("ngprt_multi_render_tiles");
    if (!m || !cams || n_cams <= 0 || !opts || !rgb0)
        return fail(NGPRT_EINVAL, "ngprt_multi_render_tiles: bad argument");
    tile = tile ? tile : 32u;
    std::lock_guard<std::mutex> lock(m->mu);
    const int n = int(m->dev.size());
    const cudaStream_t s0 = static_cast<cudaStream_t>(stream0);
    const bool window = opts->w && opts->h;
    const uint32_t W = window ? opts->w : cams[0].width, H = window ? opts->h : cams[0].height;
    const size_t per = size_t(shard_pixels(W, H, uint32_t(n), tile)) * size_t(n_cams);  // pixels per rank
    if (ngprt_status e = grow(m->dev[0], &m->grgb, &m->grgb_cap, per * 3 * n)) return e;
    if (stats0)
        if (ngprt_status e = grow(m->dev[0], &m->gstats, &m->gstats_cap, per * n)) return e;
    for (int i = 1; i < n; ++i) {
        if (ngprt_status e = grow(m->dev[i], &m->rgb[i], &m->rgb_cap[i], per * 3)) return e;
        if (stats0)
            if (ngprt_status e = grow(m->dev[i], &m->stats[i], &m->stats_cap[i], per)) return e;
    }
    if (ngprt_status e = fork(m, s0)) return e;
    // every device renders its tiles: one K0/K1/K2 launch each; devices[0] writes
    // straight into its slot of the gather buffer
    for (int i = 0; i < n; ++i) {
        ngprt_render_opts o = *opts;
        o.shard_world = uint32_t(n);
        o.shard_rank = uint32_t(i);
        o.shard_tile = tile;
        float* out = i == 0 ? m->grgb : m->rgb[i];
        ngprt_ray_stats* st = stats0 ? (i == 0 ? m->gstats : m->stats[i]) : nullptr;
        if (ngprt_status e = ngprt_render(m->scene[i], cams, n_cams, &o, out, st, i == 0 ? stream0 : m->st[i]))
            return e;
        if (i > 0) {
            MG_CUDA(cudaSetDevice(m->dev[i]));
            MG_CUDA(cudaEventRecord(m->rendered[i], m->st[i]));
        }
    }
    // gather to devices[0]: rank i's compact buffer lands at slot i
    if (n > 1) {
        if (m->use_nccl) {
            const Nccl& nc = nccl();
            MG_NCCL(nc.GroupStart());
            for (int i = 1; i < n; ++i) {
                MG_NCCL(nc.Send(m->rgb[i], per * 3, ncclFloat32, 0, m->comm[i], m->st[i]));
                MG_NCCL(nc.Recv(m->grgb + per * 3 * i, per * 3, ncclFloat32, i, m->comm[0], s0));
                if (stats0) {
                    MG_NCCL(nc.Send(m->stats[i], per * 4, ncclUint32, 0, m->comm[i], m->st[i]));
                    MG_NCCL(nc.Recv(m->gstats + per * i, per * 4, ncclUint32, i, m->comm[0], s0));
                }
            }
            MG_NCCL(nc.GroupEnd());
        } else {
            for (int i = 1; i < n; ++i) {
                if (ngprt_status e = peer_copy(m, i, m->grgb + per * 3 * i, m->rgb[i], per * 12, s0))
                    return e;
                if (stats0)
                    if (ngprt_status e = peer_copy(m, i, m->gstats + per * i, m->stats[i],
                                                   per * sizeof(ngprt_ray_stats), s0))
                        return e;
            }
        }
    }
    MG_CUDA(cudaSetDevice(m->dev[0]));
    if (ngprt_status e = ngprt_shard_assemble(m->grgb, uint32_t(n), uint32_t(n_cams), W, H, tile, 3,
                                              rgb0, stream0))
        return e;
    if (stats0)
        if (ngprt_status e = ngprt_shard_assemble(reinterpret_cast<const float*>(m->gstats), uint32_t(n),
                                                  uint32_t(n_cams), W, H, tile, 4,
                                                  reinterpret_cast<float*>(stats0), stream0))
            return e;
    return NGPRT_OK;
}

ngprt_status ngprt_multi_render_cameras(ngprt_multi* m, const ngprt_camera* cams, int n_cams,
                                        const ngprt_render_opts* opts, float* rgb0,
                                        ngprt_ray_stats* stats0, void* stream0) {
    const ngprt_dev::DeviceRestore keep;
    const ngprt_dev::NvtxRange range("ngprt_multi_render_cameras");
    if (!m || !cams || n_cams <= 0 || !opts || !rgb0)
        return fail(NGPRT_EINVAL, "ngprt_multi_render_cameras: bad argument");
    if (opts->shard_world) return fail(NGPRT_EINVAL, "ngprt_multi_render_cameras: opts are sharded");
    std::lock_guard<std::mutex> lock(m->mu);
    const int n = int(m->dev.size());
    const cudaStream_t s0 = static_cast<cudaStream_t>(stream0);
    const bool window = opts->w && opts->h;
    const uint32_t W = window ? opts->w : cams[0].width, H = window ? opts->h : cams[0].height;
    const size_t frame = size_t(W) * H;
    if (ngprt_status e = fork(m, s0)) return e;
    std::vector<std::vector<ngprt_camera>> mine(n);
    for (int c = 0; c < n_cams; ++c) mine[c % n].push_back(cams[c]);
    // device i renders cameras i, i + n, ... as one call; devices[0]'s frames are
    // rendered straight into place when it owns every camera (n == 1)
    for (int i = 0; i < n; ++i) {
        if (mine[i].empty()) continue;
        const size_t k = mine[i].size();
        float* out;
        ngprt_ray_stats* st = nullptr;
        if (n == 1) {
            out = rgb0;
            st = stats0;
        } else {
            if (ngprt_status e = grow(m->dev[i], &m->rgb[i], &m->rgb_cap[i], k * frame * 3)) return e;
            if (stats0)
                if (ngprt_status e = grow(m->dev[i], &m->stats[i], &m->stats_cap[i], k * frame)) return e;
            out = m->rgb[i];
            st = stats0 ? m->stats[i] : nullptr;
        }
        if (ngprt_status e = ngprt_render(m->scene[i], mine[i].data(), int(k), opts, out, st,
                                          i == 0 ? stream0 : m->st[i]))
            return e;
        if (i > 0) {
            MG_CUDA(cudaSetDevice(m->dev[i]));
            MG_CUDA(cudaEventRecord(m->rendered[i], m->st[i]));
        }
    }
    if (n == 1) return NGPRT_OK;
    // gather: camera c (local frame c / n of device c % n) to rgb0 + c * frame
    MG_CUDA(cudaSetDevice(m->dev[0]));
    for (int c = 0; c < n_cams; c += n) {  // devices[0]'s own frames: device-local copies
        MG_CUDA(cudaMemcpyAsync(rgb0 + size_t(c) * frame * 3, m->rgb[0] + size_t(c / n) * frame * 3,
                                frame * 12, cudaMemcpyDeviceToDevice, s0));
        if (stats0)
            MG_CUDA(cudaMemcpyAsync(stats0 + size_t(c) * frame, m->stats[0] + size_t(c / n) * frame,
                                    frame * sizeof(ngprt_ray_stats), cudaMemcpyDeviceToDevice, s0));
    }
    if (m->use_nccl) {
        const Nccl& nc = nccl();
        MG_NCCL(nc.GroupStart());
        for (int c = 0; c < n_cams; ++c) {
            const int i = c % n;
            if (i == 0) continue;
            const size_t j = size_t(c / n);
            MG_NCCL(nc.Send(m->rgb[i] + j * frame * 3, frame * 3, ncclFloat32, 0, m->comm[i], m->st[i]));
            MG_NCCL(nc.Recv(rgb0 + size_t(c) * frame * 3, frame * 3, ncclFloat32, i, m->comm[0], s0));
            if (stats0) {
                MG_NCCL(nc.Send(m->stats[i] + j * frame, frame * 4, ncclUint32, 0, m->comm[i], m->st[i]));
                MG_NCCL(nc.Recv(stats0 + size_t(c) * frame, frame * 4, ncclUint32, i, m->comm[0], s0));
            }
        }
        MG_NCCL(nc.GroupEnd());
    } else {
        for (int c = 0; c < n_cams; ++c) {
            const int i = c % n;
            if (i == 0) continue;
            const size_t j = size_t(c / n);
            if (ngprt_status e = peer_copy(m, i, rgb0 + size_t(c) * frame * 3, m->rgb[i] + j * frame * 3,
                                           frame * 12, s0))
                return e;
            if (stats0)
                if (ngprt_status e = peer_copy(m, i, stats0 + size_t(c) * frame, m->stats[i] + j * frame,
                                               frame * sizeof(ngprt_ray_stats), s0))
                    return e;
        }
    }
    return NGPRT_OK;
}

}  // extern "C"
