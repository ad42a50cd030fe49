// ngrt_io.cpp — host-side reader of the reference's baked-scene file format
// (".ngrt", written by save_baked, read by load_baked: baking.hpp:229-485).
//
// Layout (little-endian): "NGRT", u32 version = 1, header { u32 L_C, u32 L,
// u32 fine_res[L], u64 table_lens[6 + L], u8 fusion_tag, zero pad to an 8-byte
// multiple }, then sections { u32 id, u64 byte_len, payload, u32 crc32(payload) }.
// The parse mirrors load_baked's checks and error texts (with byte offsets) and
// yields an ngprt_scene_desc whose pyramid levels and distance grid are the
// file's own (512..32 and 256^3, baking.hpp:435-447).
#include <algorithm>
#include <cstdio>
#include <cstring>
#include <memory>
#include <stdexcept>
#include <string>
#include <vector>

#include "baked.hpp"

namespace {

constexpr uint32_t kVersion = 1;
constexpr int kCoarseLevels = 6;

struct Reader {  // detail::ByteReader, training.hpp:464-479
    const unsigned char* p;
    size_t len, off = 0;
    void read(void* dst, size_t n, const char* what) {
        if (n > len - off)  // off <= len always; no wrap for huge n
            throw std::runtime_error(std::string("checkpoint: truncated reading ") + what +
                                     " at offset " + std::to_string(off));
        std::memcpy(dst, p + off, n);
        off += n;
    }
    template <class V>
    V pod(const char* what) {
        V v;
        read(&v, sizeof v, what);
        return v;
    }
};

void read_mlp(Reader& pr, const char* tag, std::vector<float>* w, std::vector<float>* b) {
    const uint32_t nd = pr.pod<uint32_t>("mlp ndims");
    if (nd > 16) throw std::runtime_error(std::string("load_baked: ") + tag + " has too many layers");
    std::vector<int> dims(nd);
    for (auto& d : dims) d = int(pr.pod<uint32_t>("mlp dim"));
    const std::vector<int> want = {23, 64, 64, 3};  // shade requires 23 -> 3 (volume.hpp:121-122)
    if (dims != want)
        throw std::runtime_error(std::string("load_baked: ") + tag +
                                 " must be 23-64-64-3 (shade, volume.hpp:121-122)");
    for (int k = 0; k < 3; ++k) {
        w[k].resize(size_t(dims[k]) * dims[k + 1]);
        b[k].resize(size_t(dims[k + 1]));
        pr.read(w[k].data(), w[k].size() * 4, "mlp weights");
        pr.read(b[k].data(), b[k].size() * 4, "mlp biases");
    }
}

}  // namespace

extern "C" {

ngprt_status ngprt_baked_load(const char* path, ngprt_baked** out) {
    if (!path || !out) {
        ngprt_host::set_error("ngprt_baked_load: null argument");
        return NGPRT_EINVAL;
    }
    *out = nullptr;
    try {
        std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "rb"), &std::fclose);
        if (!f) throw std::runtime_error(std::string("load_baked: cannot open ") + path);
        std::vector<unsigned char> buf;
        unsigned char chunk[1 << 16];
        size_t n;
        while ((n = std::fread(chunk, 1, sizeof chunk, f.get())) > 0) buf.insert(buf.end(), chunk, chunk + n);
        if (buf.size() < 8 || std::memcmp(buf.data(), "NGRT", 4) != 0)
            throw std::runtime_error("load_baked: bad magic at offset 0");
        Reader r{buf.data() + 4, buf.size() - 4};
        if (r.pod<uint32_t>("version") != kVersion)
            throw std::runtime_error("load_baked: unsupported version at offset 4");

        auto b = std::make_unique<ngprt_baked>();
        ngprt_scene_desc& d = b->desc;
        const size_t header_start = r.off;
        const uint32_t lc = r.pod<uint32_t>("L_C");
        const uint32_t L = r.pod<uint32_t>("L");
        if (L < 2 || L > 4) throw std::runtime_error("load_baked: L out of range");
        d.L = L;
        d.L_C = lc;
        for (uint32_t l = 0; l < L; ++l) d.fine_res[l] = r.pod<uint32_t>("fine resolution");
        std::vector<uint64_t> lens(kCoarseLevels + L);
        for (auto& v : lens) v = r.pod<uint64_t>("table length");
        for (uint32_t l = 0; l < L; ++l) {
            d.fine_table_len[l] = lens[kCoarseLevels + l];
            d.fine_hashed[l] = 1;  // load_baked: Addressing::Hashed (baking.hpp:384)
            // bounds the reference leaves unchecked: a crafted length would make the
            // section-2 size arithmetic wrap and the device hash read out of bounds
            if (d.fine_table_len[l] == 0 || d.fine_table_len[l] > (uint64_t(1) << 32))
                throw std::runtime_error("load_baked: fine table length out of range (1..2^32)");
            if (d.fine_res[l] == 0 || d.fine_res[l] > (1u << 20))
                throw std::runtime_error("load_baked: fine resolution out of range (1..2^20)");
        }
        if (lc == 0 || lc > 4096) throw std::runtime_error("load_baked: L_C out of range (1..4096)");
        d.fusion_tag = r.pod<uint8_t>("fusion tag");
        while ((r.off - header_start) % 8 != 0) r.pod<uint8_t>("pad");
        const int w = 8 + 2 * int(L);

        bool saw[8] = {};
        while (r.off < r.len) {
            const size_t sec_off = r.off;
            const uint32_t id = r.pod<uint32_t>("section id");
            const uint64_t len = r.pod<uint64_t>("section length");
            if (len > r.len - r.off || r.len - r.off - len < 4)  // no u64 wrap
                throw std::runtime_error("load_baked: truncated section " + std::to_string(id) +
                                         " at offset " + std::to_string(sec_off));
            const unsigned char* payload = r.p + r.off;
            r.off += len;
            const uint32_t crc = r.pod<uint32_t>("section crc");
            if (ngprt_crc32(payload, len, 0) != crc)
                throw std::runtime_error("load_baked: checksum failure in section " +
                                         std::to_string(id) + " at offset " +
                                         std::to_string(sec_off));
            Reader pr{payload, len};
            switch (id) {
                case 1: {  // coarse corner map, sorted by key
                    const uint64_t count = pr.pod<uint64_t>("corner count");
                    if (count > (pr.len - pr.off) / (8 + sizeof(float) * w))
                        throw std::runtime_error("load_baked: corner count exceeds section 1 at offset " +
                                                 std::to_string(sec_off));
                    b->keys.resize(count);
                    b->rows.resize(count * w);
                    for (uint64_t i = 0; i < count; ++i) {
                        b->keys[i] = pr.pod<uint64_t>("corner index");
                        pr.read(b->rows.data() + i * w, sizeof(float) * w, "corner row");
                    }
                    break;
                }
                case 2: {
                    uint64_t want = 0;
                    for (uint32_t l = 0; l < L; ++l) want += d.fine_table_len[l] * 32;
                    if (want != len)
                        throw std::runtime_error("load_baked: fine table section size mismatch at offset " +
                                                 std::to_string(sec_off));
                    for (uint32_t l = 0; l < L; ++l) {
                        b->fine[l].resize(d.fine_table_len[l] * 8);
                        pr.read(b->fine[l].data(), b->fine[l].size() * 4, "fine table");
                    }
                    break;
                }
                case 3:
                    read_mlp(pr, "view MLP", b->psi_w, b->psi_b);
                    break;
                case 4:
                    for (int k = 0; k < NGPRT_PYRAMID_LEVELS; ++k) {
                        const size_t res = size_t(512) >> k;
                        b->pyramid[k].resize((res * res * res + 63) / 64);
                        pr.read(b->pyramid[k].data(), b->pyramid[k].size() * 8, "pyramid");
                    }
                    break;
                case 5:
                    b->dist.resize(size_t(256) * 256 * 256);
                    pr.read(b->dist.data(), b->dist.size(), "distance grid");
                    break;
                case 6:
                    b->att.resize(size_t(2) * L);
                    pr.read(b->att.data(), b->att.size() * 4, "attention globals");
                    break;
                case 7: {  // fusion MLP {8L, 64, 8} (baking.hpp:452-466)
                    const uint32_t nd = pr.pod<uint32_t>("fusion mlp ndims");
                    if (nd > 16) throw std::runtime_error("load_baked: fusion MLP has too many layers");
                    std::vector<int> dims(nd);
                    for (auto& dd : dims) dd = int(pr.pod<uint32_t>("fusion mlp dim"));
                    if (dims != std::vector<int>{8 * int(L), 64, 8})
                        throw std::runtime_error("load_baked: fusion MLP must be 8L-64-8 (fusion.hpp:101)");
                    for (int k = 0; k < 2; ++k) {
                        b->fmlp_w[k].resize(size_t(dims[k]) * dims[k + 1]);
                        b->fmlp_b[k].resize(size_t(dims[k + 1]));
                        pr.read(b->fmlp_w[k].data(), b->fmlp_w[k].size() * 4, "fusion mlp weights");
                        pr.read(b->fmlp_b[k].data(), b->fmlp_b[k].size() * 4, "fusion mlp biases");
                    }
                    break;
                }
                default:
                    throw std::runtime_error("load_baked: unknown section id " + std::to_string(id) +
                                             " at offset " + std::to_string(sec_off));
            }
            if (pr.off != pr.len)
                throw std::runtime_error("load_baked: section " + std::to_string(id) +
                                         " length mismatch at offset " + std::to_string(sec_off));
            if (id <= 7) saw[id] = true;
        }
        for (uint32_t id : {1u, 2u, 3u, 4u, 5u})
            if (!saw[id]) throw std::runtime_error("load_baked: missing section " + std::to_string(id));
        const bool inv = d.fusion_tag == NGPRT_FUSION_SHARED_ATT_INV ||
                         d.fusion_tag == NGPRT_FUSION_SEPARATE_ATT_INV;
        if (inv && !saw[6]) throw std::runtime_error("load_baked: missing attention globals section");
        if (d.fusion_tag == NGPRT_FUSION_MLP && !saw[7])
            throw std::runtime_error("load_baked: missing fusion MLP section");

        b->pyramid_base = 512;
        b->finalize();
        *out = b.release();
        return NGPRT_OK;
    } catch (const std::exception& e) {
        ngprt_host::set_error(e.what());
        return NGPRT_EINVAL;
    }
}

const ngprt_scene_desc* ngprt_baked_desc(const ngprt_baked* b) { return b ? &b->desc : nullptr; }

void ngprt_baked_free(ngprt_baked* b) { delete b; }

ngprt_status ngprt_scene_load(const char* path, int device, ngprt_scene** out) {
    ngprt_baked* b = nullptr;
    ngprt_status st = ngprt_baked_load(path, &b);
    if (st != NGPRT_OK) return st;
    st = ngprt_scene_create(&b->desc, device, out);
    ngprt_baked_free(b);
    return st;
}

}  // extern "C"

namespace {
void put_bytes(std::vector<unsigned char>& out, const void* p, size_t n) {
    const auto* b = static_cast<const unsigned char*>(p);
    out.insert(out.end(), b, b + n);
}
template <class V>
void put_pod(std::vector<unsigned char>& out, const V& v) {
    put_bytes(out, &v, sizeof v);
}
void put_section(std::vector<unsigned char>& out, uint32_t id, const std::vector<unsigned char>& p) {
    put_pod(out, id);
    put_pod(out, uint64_t(p.size()));
    put_bytes(out, p.data(), p.size());
    put_pod(out, ngprt_crc32(p.data(), p.size(), 0));
}
}  // namespace

extern "C" ngprt_status ngprt_baked_save(const ngprt_baked* b, const char* path) {
    // save_baked, baking.hpp:266-349 (coarse table lengths of the header are the
    // EncodingConfig defaults: the render path does not use them).
    if (!b || !path) {
        ngprt_host::set_error("ngprt_baked_save: null argument");
        return NGPRT_EINVAL;
    }
    const ngprt_scene_desc& d = b->desc;
    if (d.occ_base_res != 512 || d.dist_res != 256 || !d.dist_values) {
        ngprt_host::set_error("save_baked: the format fixes a 512 pyramid and a 256^3 distance grid");
        return NGPRT_EINVAL;
    }
    const int L = int(d.L), w = 8 + 2 * L;
    std::vector<unsigned char> out;
    put_bytes(out, "NGRT", 4);
    put_pod(out, kVersion);
    const size_t header_start = out.size();
    put_pod(out, uint32_t(d.L_C));
    put_pod(out, uint32_t(L));
    for (int l = 0; l < L; ++l) put_pod(out, uint32_t(d.fine_res[l]));
    const int cres[kCoarseLevels] = {16, 32, 64, 128, 256, 512};
    for (int k = 0; k < kCoarseLevels; ++k) {
        const uint64_t corners = uint64_t(cres[k] + 1) * (cres[k] + 1) * (cres[k] + 1);
        put_pod(out, corners < (uint64_t(1) << 21) ? corners : (uint64_t(1) << 21));
    }
    for (int l = 0; l < L; ++l) put_pod(out, uint64_t(d.fine_table_len[l]));
    put_pod(out, uint8_t(d.fusion_tag));
    while ((out.size() - header_start) % 8 != 0) out.push_back(0);
    {
        std::vector<size_t> order(d.n_coarse);
        for (size_t i = 0; i < order.size(); ++i) order[i] = i;
        std::sort(order.begin(), order.end(),
                  [&](size_t x, size_t y) { return d.coarse_keys[x] < d.coarse_keys[y]; });
        std::vector<unsigned char> p;
        put_pod(p, uint64_t(d.n_coarse));
        for (size_t i : order) {
            put_pod(p, uint64_t(d.coarse_keys[i]));
            put_bytes(p, d.coarse_rows + i * w, sizeof(float) * w);
        }
        put_section(out, 1, p);
    }
    {
        std::vector<unsigned char> p;
        for (int l = 0; l < L; ++l) put_bytes(p, d.fine_tables[l], d.fine_table_len[l] * 8 * sizeof(float));
        put_section(out, 2, p);
    }
    {
        std::vector<unsigned char> p;
        const uint32_t dims[4] = {23, 64, 64, 3};
        put_pod(p, uint32_t(4));
        for (uint32_t v : dims) put_pod(p, v);
        for (int k = 0; k < 3; ++k) {
            put_bytes(p, d.psi_w[k], sizeof(float) * dims[k] * dims[k + 1]);
            put_bytes(p, d.psi_b[k], sizeof(float) * dims[k + 1]);
        }
        put_section(out, 3, p);
    }
    {
        std::vector<unsigned char> p;
        for (int k = 0; k < NGPRT_PYRAMID_LEVELS; ++k) {
            const size_t res = size_t(512) >> k;
            put_bytes(p, d.pyramid_words[k], ((res * res * res + 63) / 64) * 8);
        }
        put_section(out, 4, p);
    }
    {
        std::vector<unsigned char> p;
        put_bytes(p, d.dist_values, size_t(256) * 256 * 256);
        put_section(out, 5, p);
    }
    if (d.fusion_tag == NGPRT_FUSION_SHARED_ATT_INV || d.fusion_tag == NGPRT_FUSION_SEPARATE_ATT_INV) {
        std::vector<unsigned char> p;
        put_bytes(p, d.att_globals, sizeof(float) * 2 * L);
        put_section(out, 6, p);
    }
    if (d.fusion_tag == NGPRT_FUSION_MLP) {
        std::vector<unsigned char> p;
        const uint32_t dims[3] = {uint32_t(8 * L), 64, 8};
        put_pod(p, uint32_t(3));
        for (uint32_t v : dims) put_pod(p, v);
        for (int k = 0; k < 2; ++k) {
            put_bytes(p, d.fusion_mlp_w[k], sizeof(float) * dims[k] * dims[k + 1]);
            put_bytes(p, d.fusion_mlp_b[k], sizeof(float) * dims[k + 1]);
        }
        put_section(out, 7, p);
    }
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen(path, "wb"), &std::fclose);
    if (!f || std::fwrite(out.data(), 1, out.size(), f.get()) != out.size()) {
        ngprt_host::set_error(std::string("save_baked: cannot write ") + path);
        return NGPRT_EINVAL;
    }
    return NGPRT_OK;
}
