// baked.hpp — host-side BakedScene container shared by the .ngrt reader/writer
// (ngrt_io.cpp) and the GPU bake (bake.cu). Internal; the public view is
// ngprt_scene_desc via ngprt_baked_desc().
#pragma once

#include <sys/mman.h>

#include <cstdlib>
#include <cstring>
#include <new>
#include <string>
#include <vector>

#include "ngprt_cuda.h"

// Large host arrays of a BakedScene: uninitialised on resize (the bake and the
// loader overwrite every element) and 2 MiB-aligned with transparent huge pages
// advised, so filling a multi-GB corner-row array is not dominated by page
// faults and zero-fill.
template <class T>
struct HostBuf {
    T* p = nullptr;
    size_t n = 0;
    HostBuf() = default;
    HostBuf(const HostBuf&) = delete;
    HostBuf& operator=(const HostBuf&) = delete;
    ~HostBuf() { std::free(p); }
    void resize(size_t m) {  // contents are not preserved
        std::free(p);
        p = nullptr;
        n = m;
        if (!m) return;
        constexpr size_t kHuge = size_t(2) << 20;
        const size_t bytes = (m * sizeof(T) + kHuge - 1) / kHuge * kHuge;
        p = static_cast<T*>(std::aligned_alloc(kHuge, bytes));
        if (!p) throw std::bad_alloc();
        madvise(p, bytes, MADV_HUGEPAGE);
    }
    void assign(const T* a, const T* b) {
        resize(size_t(b - a));
        if (n) std::memcpy(p, a, n * sizeof(T));
    }
    T* data() { return p; }
    const T* data() const { return p; }
    size_t size() const { return n; }
    bool empty() const { return n == 0; }
    T& operator[](size_t i) { return p[i]; }
    const T& operator[](size_t i) const { return p[i]; }
};

struct ngprt_baked {
    ngprt_scene_desc desc{};
    HostBuf<uint64_t> keys;
    HostBuf<float> rows;
    HostBuf<float> fine[NGPRT_MAX_FINE_LEVELS];
    std::vector<float> psi_w[3], psi_b[3];
    std::vector<float> att;
    std::vector<float> fmlp_w[2], fmlp_b[2];
    HostBuf<uint64_t> pyramid[NGPRT_PYRAMID_LEVELS];
    HostBuf<uint8_t> dist;
    uint32_t pyramid_base = 512;

    // Points desc at the owned arrays (call after filling them).
    void finalize() {
        ngprt_scene_desc& d = desc;
        const uint32_t L = d.L;
        d.n_coarse = keys.size();
        d.coarse_keys = keys.data();
        d.coarse_rows = rows.data();
        for (uint32_t l = 0; l < L; ++l) d.fine_tables[l] = fine[l].data();
        for (int k = 0; k < 3; ++k) {
            d.psi_w[k] = psi_w[k].data();
            d.psi_b[k] = psi_b[k].data();
        }
        d.att_globals = att.empty() ? nullptr : att.data();
        for (int k = 0; k < 2; ++k) {
            d.fusion_mlp_w[k] = fmlp_w[k].empty() ? nullptr : fmlp_w[k].data();
            d.fusion_mlp_b[k] = fmlp_b[k].empty() ? nullptr : fmlp_b[k].data();
        }
        d.occ_base_res = pyramid_base;
        for (int k = 0; k < NGPRT_PYRAMID_LEVELS; ++k) d.pyramid_words[k] = pyramid[k].data();
        d.dist_res = dist.empty() ? 0 : (pyramid_base >> 1);
        d.dist_values = dist.empty() ? nullptr : dist.data();
        d.storage = NGPRT_STORAGE_AUTO;
    }
};

namespace ngprt_host {
void set_error(const std::string& msg);  // ngprt_abi.cu (ngprt_last_error)
}
