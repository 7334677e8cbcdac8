// Packed-KV wire / disk format (include/ekv_capi.h, "EKVPACK1" family): the
// compressed cloud layers of an assembled context as one self-describing,
// checksummed byte stream -- what crosses the cloud -> edge link (the transfer
// the reference simulates in Sim::submit_transfer, sim.cpp:417-449, sized by
// deep_layer_bytes, sim.cpp:714) or is kept as the historical cache
// (sim.cpp:885-895).  Checksums are the reference's fnv1a64 (rng.cpp:7-15).
//
// Version 2 (written here): each of a layer's four arrays (K codes, V codes,
// K scales, V scales) is cut into 4 KiB chunks; the layer checksum is
// FNV-1a 64 over the little-endian u64 FNV-1a 64 of every chunk, in payload
// order.  The chunk hashes are independent, so the device hashes a layer in
// microseconds (one thread per chunk) right where the bytes are: export hashes
// the context storage before the D2H copy, import hashes a staging copy in HBM
// before committing it (a corrupted pack never reaches the context).  Version 1
// packs (FNV-1a over the whole layer payload) are still accepted.
#include <algorithm>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "ekv_objects.h"

using namespace ekv;

namespace {
constexpr char kPackMagic[8] = {'E', 'K', 'V', 'P', 'A', 'C', 'K', '1'};
constexpr uint32_t kPackVersion = 2;
constexpr size_t kChunk = 4096;
constexpr uint64_t kFnvOffset = 14695981039346656037ull, kFnvPrime = 1099511628211ull;

struct PackHeader {  // 64 bytes, little-endian
    char magic[8];
    uint32_t version, n_layers, H, S, d_e, d_c, bits, group, header_bytes, reserved[3];
    uint64_t header_fnv;  // fnv1a64 of [0, header_bytes) with this field zero
};
static_assert(sizeof(PackHeader) == 64, "pack header layout");

uint64_t fnv1a(const void* data, size_t len, uint64_t h = kFnvOffset) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= kFnvPrime;
    }
    return h;
}

// ---- device chunk hashing -----------------------------------------------------
constexpr int kMaxHashArrays = 128;  // 32 layers x 4 arrays per launch
struct HashTable {
    int n_arrays;
    const uint8_t* base[kMaxHashArrays];
    unsigned long long len[kMaxHashArrays];
    int first[kMaxHashArrays + 1];  // prefix sum of chunk counts
};

__global__ void chunk_fnv_kernel(const __grid_constant__ HashTable t, uint64_t* __restrict__ out) {
    const int c = blockIdx.x * blockDim.x + threadIdx.x;
    if (c >= t.first[t.n_arrays]) return;
    int a = 0;
    while (t.first[a + 1] <= c) ++a;
    const size_t off = (size_t)(c - t.first[a]) * kChunk;
    const size_t len = min((size_t)kChunk, (size_t)t.len[a] - off);
    const uint8_t* p = t.base[a] + off;
    uint64_t h = kFnvOffset;
    size_t i = 0;
    for (; i + 16 <= len; i += 16) {  // 16-byte loads, bytes hashed in address order
        const uint4 v = *reinterpret_cast<const uint4*>(p + i);
        const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
        for (int k = 0; k < 4; ++k)
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                h ^= (w[k] >> (8 * b)) & 0xFFu;
                h *= kFnvPrime;
            }
    }
    for (; i < len; ++i) {
        h ^= p[i];
        h *= kFnvPrime;
    }
    out[c] = h;
}

size_t chunks_of(size_t len) { return (len + kChunk - 1) / kChunk; }

size_t pack_row_bytes(int d_e, int bits) { return (size_t)d_e * bits / 8; }
size_t pack_layer_bytes(int H, int S, int d_e, int bits, int group) {
    const size_t rows = (size_t)H * S;
    return 2 * rows * pack_row_bytes(d_e, bits) + 2 * rows * (size_t)(d_e / group) * 4;
}
size_t pack_header_bytes(int n, int d_e) {
    const size_t b = sizeof(PackHeader) + (size_t)n * 4 * 2 + (size_t)d_e * 4 + (size_t)n * 8;
    return (b + 255) / 256 * 256;
}
void pack_check_shape(int n, int H, int S, int d_e, int bits, int group) {
    require(n >= 1, "kvpack: no layers");
    require(H >= 1 && S >= 1 && d_e >= 1, "kvpack: empty shape");
    require(bits == 8 || bits == 4, "kvpack: bits must be 8 or 4");
    require(group >= 1 && d_e % group == 0, "kvpack: group must divide d_e");
    require(d_e * bits % 8 == 0, "kvpack: d_e * bits must be whole bytes");
}

// The four arrays of one layer payload: K codes, V codes, K scales, V scales.
struct LayerArrays {
    size_t cb, sb;
    size_t size(int a) const { return a < 2 ? cb : sb; }
    size_t offset(int a) const { return a == 0 ? 0 : a == 1 ? cb : a == 2 ? 2 * cb : 2 * cb + sb; }
    size_t chunks() const { return 2 * chunks_of(cb) + 2 * chunks_of(sb); }
};

// Layer checksums (version 2) from device arrays: arrays[4*i + a] of layer i.
// Hashes on `st`, returns after the chunk hashes are back on the host.
void device_layer_fnvs(const std::vector<const void*>& arrays, const LayerArrays& la, int n,
                       uint64_t* out, ekv_ctx_s* c, cudaStream_t st) {
    std::vector<uint64_t> ch(la.chunks() * n);
    uint64_t* dch = nullptr;
    EKV_CUDA(cudaMallocAsync((void**)&dch, sizeof(uint64_t) * ch.size(), st));
    size_t done = 0;
    for (int l0 = 0; l0 < n; l0 += kMaxHashArrays / 4) {
        const int nl = std::min(n - l0, kMaxHashArrays / 4);
        HashTable t{};
        t.n_arrays = 4 * nl;
        t.first[0] = 0;
        for (int i = 0; i < 4 * nl; ++i) {
            t.base[i] = (const uint8_t*)arrays[4 * l0 + i];
            t.len[i] = la.size(i % 4);
            t.first[i + 1] = t.first[i] + (int)chunks_of(t.len[i]);
        }
        const int total = t.first[4 * nl];
        chunk_fnv_kernel<<<(total + 127) / 128, 128, 0, st>>>(t, dch + done);
        EKV_CUDA(cudaGetLastError());
        count_launches(1);
        done += total;
    }
    EKV_CUDA(cudaMemcpyAsync(ch.data(), dch, sizeof(uint64_t) * ch.size(), cudaMemcpyDeviceToHost, st));
    EKV_CUDA(cudaFreeAsync(dch, st));
    EKV_CUDA(cudaStreamSynchronize(st));
    (void)c;
    const size_t per = la.chunks();
    for (int i = 0; i < n; ++i) out[i] = fnv1a(ch.data() + i * per, sizeof(uint64_t) * per);
}

// Version-2 layer checksums of a host payload (chunks hashed on parallel threads).
void host_layer_fnvs_v2(const unsigned char* payload, int n, const LayerArrays& la, size_t lb,
                        uint64_t* out) {
    const size_t per = la.chunks();
    std::vector<uint64_t> ch(per * n);
    std::vector<std::pair<const unsigned char*, size_t>> jobs;
    for (int i = 0; i < n; ++i)
        for (int a = 0; a < 4; ++a) {
            const unsigned char* base = payload + (size_t)i * lb + la.offset(a);
            for (size_t off = 0; off < la.size(a); off += kChunk)
                jobs.emplace_back(base + off, std::min(kChunk, la.size(a) - off));
        }
    const int nt = std::max(1, std::min((int)jobs.size(), (int)std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([&, t] {
            for (size_t j = t; j < jobs.size(); j += nt) ch[j] = fnv1a(jobs[j].first, jobs[j].second);
        });
    for (auto& th : pool) th.join();
    for (int i = 0; i < n; ++i) out[i] = fnv1a(ch.data() + i * per, sizeof(uint64_t) * per);
}

void host_layer_fnvs_v1(const unsigned char* payload, int n, size_t lb, uint64_t* out) {
    const int nt = std::max(1, std::min(n, (int)std::thread::hardware_concurrency()));
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; ++t)
        pool.emplace_back([=] {
            for (int i = t; i < n; i += nt) out[i] = fnv1a(payload + (size_t)i * lb, lb);
        });
    for (auto& th : pool) th.join();
}

// validated view of a pack in host memory
struct PackView {
    const PackHeader* hd;
    const int32_t* edge;
    const int32_t* cloud;
    const int32_t* kept;
    const uint64_t* lfnv;
    const unsigned char* payload;
    size_t layer_bytes;
    LayerArrays la;
};

// Header checks (magic, version, shape, sizes, header checksum); with
// verify_payload the layer checksums too (on host threads).
PackView pack_view(const void* src, size_t bytes, bool verify_payload) {
    require(src != nullptr, "kvpack: null buffer");
    require(bytes >= sizeof(PackHeader), "kvpack: truncated header");
    PackView v{};
    v.hd = (const PackHeader*)src;
    require(std::memcmp(v.hd->magic, kPackMagic, 8) == 0, "kvpack: bad magic");
    require(v.hd->version == 1 || v.hd->version == 2,
            "kvpack: unsupported version " + std::to_string(v.hd->version));
    const int n = (int)v.hd->n_layers, H = (int)v.hd->H, S = (int)v.hd->S, de = (int)v.hd->d_e;
    pack_check_shape(n, H, S, de, (int)v.hd->bits, (int)v.hd->group);
    require(v.hd->header_bytes == pack_header_bytes(n, de), "kvpack: header size mismatch");
    require(bytes >= v.hd->header_bytes, "kvpack: truncated header");
    {
        std::vector<unsigned char> tmp((const unsigned char*)src, (const unsigned char*)src + v.hd->header_bytes);
        reinterpret_cast<PackHeader*>(tmp.data())->header_fnv = 0;
        require(fnv1a(tmp.data(), tmp.size()) == v.hd->header_fnv, "kvpack: header checksum mismatch");
    }
    const unsigned char* b = (const unsigned char*)src + sizeof(PackHeader);
    v.edge = (const int32_t*)b;
    v.cloud = v.edge + n;
    v.kept = v.cloud + n;
    v.lfnv = (const uint64_t*)(v.kept + de);
    v.payload = (const unsigned char*)src + v.hd->header_bytes;
    v.layer_bytes = pack_layer_bytes(H, S, de, (int)v.hd->bits, (int)v.hd->group);
    const size_t rows = (size_t)H * S;
    v.la = LayerArrays{rows * pack_row_bytes(de, (int)v.hd->bits), rows * (de / v.hd->group) * 4};
    require(bytes >= v.hd->header_bytes + (size_t)n * v.layer_bytes, "kvpack: truncated payload");
    if (verify_payload) {
        std::vector<uint64_t> got(n);
        if (v.hd->version == 1)
            host_layer_fnvs_v1(v.payload, n, v.layer_bytes, got.data());
        else
            host_layer_fnvs_v2(v.payload, n, v.la, v.layer_bytes, got.data());
        for (int i = 0; i < n; ++i)
            require(got[i] == v.lfnv[i], "kvpack: checksum mismatch in layer " + std::to_string(v.edge[i]));
    }
    return v;
}

void check_pack_fits(const PackView& v, ekv_kvctx_s* c) {
    const int H = c->model->cfg.num_heads, de = d_of(c->model);
    require((int)v.hd->H == H && (int)v.hd->d_e == de && (int)v.hd->S == c->S,
            "kvpack: dim mismatch (pack H=" + std::to_string(v.hd->H) + " S=" + std::to_string(v.hd->S) +
                " d=" + std::to_string(v.hd->d_e) + ", context H=" + std::to_string(H) +
                " S=" + std::to_string(c->S) + " d=" + std::to_string(de) + ")");
    for (uint32_t i = 0; i < v.hd->n_layers; ++i) {
        const int l = v.edge[i];
        require(l >= 0 && l < (int)c->seg.size(), "missing layer " + std::to_string(l));
        const ekv_segment& sg = c->seg[l];
        require(sg.format == (int)v.hd->bits && sg.group == (int)v.hd->group,
                "kvpack: layer " + std::to_string(l) + " format differs from the context's");
    }
}

void* dst_array(const ekv_segment& sg, int a) {
    return (void*)(a == 0 ? sg.k : a == 1 ? sg.v : a == 2 ? (const void*)sg.k_scales : (const void*)sg.v_scales);
}
}  // namespace

extern "C" {

int ekv_fnv1a64(const void* data, size_t len, uint64_t seed, uint64_t* out) {
    return guard([&] {
        require(out && (data || len == 0), "ekv_fnv1a64: null argument");
        *out = fnv1a(data, len, seed);
    });
}

int ekv_kvpack_size(int n_layers, int H, int S, int d_e, int bits, int group, size_t* bytes) {
    return guard([&] {
        require(bytes != nullptr, "ekv_kvpack_size: null argument");
        pack_check_shape(n_layers, H, S, d_e, bits, group);
        *bytes = pack_header_bytes(n_layers, d_e) + (size_t)n_layers * pack_layer_bytes(H, S, d_e, bits, group);
    });
}

int ekv_kvpack_export(ekv_kvctx_t c, const int* layers, const int* cloud_layers, int n, const int* kept, int d_c,
                      void* dst, size_t capacity) {
    return guard([&] {
        require(c && layers && cloud_layers && kept && dst, "ekv_kvpack_export: null argument");
        require(n >= 1, "kvpack: no layers");
        const ekv_segment& s0 = c->seg.at(layers[0]);
        const int H = c->model->cfg.num_heads, S = c->S, de = d_of(c->model);
        const int bits = s0.format, group = s0.group;
        require(bits == EKV_KV_INT8 || bits == EKV_KV_INT4, "kvpack: layer " + std::to_string(layers[0]) +
                                                                " is not a compressed layer");
        pack_check_shape(n, H, S, de, bits, group);
        for (int i = 0; i < n; ++i) {
            require(layers[i] >= 0 && layers[i] < (int)c->seg.size(), "missing layer " + std::to_string(layers[i]));
            const ekv_segment& sg = c->seg[layers[i]];
            require(sg.format == bits && sg.group == group,
                    "kvpack: layer " + std::to_string(layers[i]) + " format differs from layer " +
                        std::to_string(layers[0]));
        }
        const size_t hb = pack_header_bytes(n, de), lb = pack_layer_bytes(H, S, de, bits, group);
        require(capacity >= hb + (size_t)n * lb, "kvpack: destination too small");
        ekv_ctx_s* ctx = c->model->ctx;
        set_dev(ctx);
        cudaStream_t st = ctx->stream;
        unsigned char* out = (unsigned char*)dst;
        std::memset(out, 0, hb);
        PackHeader* hd = (PackHeader*)out;
        std::memcpy(hd->magic, kPackMagic, 8);
        hd->version = kPackVersion;
        hd->n_layers = n;
        hd->H = H;
        hd->S = S;
        hd->d_e = de;
        hd->d_c = d_c;
        hd->bits = bits;
        hd->group = group;
        hd->header_bytes = (uint32_t)hb;
        int32_t* edge = (int32_t*)(out + sizeof(PackHeader));
        int32_t* cloud = edge + n;
        int32_t* kp = cloud + n;
        uint64_t* lfnv = (uint64_t*)(kp + de);
        const size_t rows = (size_t)H * S;
        const LayerArrays la{rows * pack_row_bytes(de, bits), rows * (de / group) * 4};
        std::vector<const void*> arrays;
        for (int i = 0; i < n; ++i) {
            edge[i] = layers[i];
            cloud[i] = cloud_layers[i];
            const ekv_segment& sg = c->seg[layers[i]];
            unsigned char* p = out + hb + (size_t)i * lb;
            for (int a = 0; a < 4; ++a) {
                arrays.push_back(dst_array(sg, a));
                EKV_CUDA(cudaMemcpyAsync(p + la.offset(a), dst_array(sg, a), la.size(a),
                                         cudaMemcpyDeviceToHost, st));
            }
        }
        for (int j = 0; j < de; ++j) kp[j] = kept[j];
        device_layer_fnvs(arrays, la, n, lfnv, ctx, st);  // hashes the device copy (synchronises)
        hd->header_fnv = 0;
        hd->header_fnv = fnv1a(out, hb);
    });
}

int ekv_kvpack_parse(const void* src, size_t bytes, ekv_kvpack_info* info, int* layers, int* cloud_layers,
                     int* kept) {
    return guard([&] {
        const PackView v = pack_view(src, bytes, true);
        if (info) {
            info->n_layers = (int)v.hd->n_layers;
            info->H = (int)v.hd->H;
            info->S = (int)v.hd->S;
            info->d_e = (int)v.hd->d_e;
            info->d_c = (int)v.hd->d_c;
            info->bits = (int)v.hd->bits;
            info->group = (int)v.hd->group;
            info->bytes = v.hd->header_bytes + (size_t)v.hd->n_layers * v.layer_bytes;
        }
        for (uint32_t i = 0; i < v.hd->n_layers; ++i) {
            if (layers) layers[i] = v.edge[i];
            if (cloud_layers) cloud_layers[i] = v.cloud[i];
        }
        if (kept)
            for (uint32_t j = 0; j < v.hd->d_e; ++j) kept[j] = v.kept[j];
    });
}

int ekv_kvpack_import(ekv_kvctx_t c, const void* src, size_t bytes) {
    return guard([&] {
        require(c != nullptr, "ekv_kvpack_import: null context");
        const PackView hv = pack_view(src, bytes, false);
        const bool v2 = hv.hd->version == 2;
        const PackView v = v2 ? hv : pack_view(src, bytes, true);  // v1: verify on the host
        check_pack_fits(v, c);
        ekv_ctx_s* ctx = c->model->ctx;
        set_dev(ctx);
        cudaStream_t st = ctx->stream;
        const int n = (int)v.hd->n_layers;
        if (!v2) {
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < 4; ++a)
                    EKV_CUDA(cudaMemcpyAsync(dst_array(c->seg[v.edge[i]], a),
                                             v.payload + (size_t)i * v.layer_bytes + v.la.offset(a), v.la.size(a),
                                             cudaMemcpyHostToDevice, st));
            EKV_CUDA(cudaStreamSynchronize(st));
            return;
        }
        // v2: land the payload in an HBM staging buffer, hash it there, commit on success
        const size_t total = (size_t)n * v.layer_bytes;
        uint8_t* stage = nullptr;
        EKV_CUDA(cudaMallocAsync((void**)&stage, total, st));
        try {
            EKV_CUDA(cudaMemcpyAsync(stage, v.payload, total, cudaMemcpyHostToDevice, st));
            std::vector<const void*> arrays;
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < 4; ++a) arrays.push_back(stage + (size_t)i * v.layer_bytes + v.la.offset(a));
            std::vector<uint64_t> got(n);
            device_layer_fnvs(arrays, v.la, n, got.data(), ctx, st);
            for (int i = 0; i < n; ++i)
                require(got[i] == v.lfnv[i], "kvpack: checksum mismatch in layer " + std::to_string(v.edge[i]));
            for (int i = 0; i < n; ++i)
                for (int a = 0; a < 4; ++a)
                    EKV_CUDA(cudaMemcpyAsync(dst_array(c->seg[v.edge[i]], a), arrays[4 * i + a], v.la.size(a),
                                             cudaMemcpyDeviceToDevice, st));
        } catch (...) {
            cudaFreeAsync(stage, st);
            cudaStreamSynchronize(st);
            throw;
        }
        EKV_CUDA(cudaFreeAsync(stage, st));
        EKV_CUDA(cudaStreamSynchronize(st));
    });
}

int ekv_session_forward_pack(ekv_session_t s, const float* emb_dev, int n, float* out_dev, const void* src,
                             size_t bytes) {
    return guard([&] {
        require(s && emb_dev, "ekv_session_forward_pack: null argument");
        require(n >= 1, "ekv_session_forward_pack: n must be >= 1");
        const PackView v = pack_view(src, bytes, false);
        require(v.hd->version == 2, "kvpack: the streamed import needs a version-2 pack");
        ekv_kvctx_s* c = s->kv;
        check_pack_fits(v, c);
        ekv_model_s* m = s->model;
        ekv_ctx_s* ctx = m->ctx;
        check_overflow(s, n);
        set_dev(ctx);
        cudaStream_t st = ctx->stream, cp = ctx->copy, hs = ctx->aux;
        const int L = m->cfg.num_layers, nl = (int)v.hd->n_layers;
        std::vector<cudaEvent_t> ready(L, nullptr);
        cudaEvent_t start = nullptr;
        uint64_t* dch = nullptr;
        auto cleanup = [&] {
            for (auto& e : ready)
                if (e) cudaEventDestroy(e);
            if (start) cudaEventDestroy(start);
        };
        try {
            EKV_CUDA(cudaEventCreateWithFlags(&start, cudaEventDisableTiming));
            EKV_CUDA(cudaEventRecord(start, st));
            EKV_CUDA(cudaStreamWaitEvent(cp, start, 0));
            // per layer on the copy stream: upload into the context and release the layer to
            // the compute stream (Eq. 20: upload l overlaps compute < l); the checksum of
            // layer l runs on a third stream behind its upload, off both critical paths
            const size_t per = v.la.chunks();
            EKV_CUDA(cudaMallocAsync((void**)&dch, sizeof(uint64_t) * per * nl, cp));
            EKV_CUDA(cudaEventRecord(start, cp));
            EKV_CUDA(cudaStreamWaitEvent(hs, start, 0));
            for (int i = 0; i < nl; ++i) {
                const int l = v.edge[i];
                HashTable t{};
                t.n_arrays = 4;
                for (int a = 0; a < 4; ++a) {
                    void* dst = dst_array(c->seg[l], a);
                    EKV_CUDA(cudaMemcpyAsync(dst, v.payload + (size_t)i * v.layer_bytes + v.la.offset(a),
                                             v.la.size(a), cudaMemcpyHostToDevice, cp));
                    t.base[a] = (const uint8_t*)dst;
                    t.len[a] = v.la.size(a);
                    t.first[a + 1] = t.first[a] + (int)chunks_of(t.len[a]);
                }
                EKV_CUDA(cudaEventCreateWithFlags(&ready[l], cudaEventDisableTiming));
                EKV_CUDA(cudaEventRecord(ready[l], cp));
                EKV_CUDA(cudaStreamWaitEvent(hs, ready[l], 0));
                chunk_fnv_kernel<<<(t.first[4] + 127) / 128, 128, 0, hs>>>(t, dch + (size_t)i * per);
                EKV_CUDA(cudaGetLastError());
                count_launches(1);
            }
            streamed_forward(s, emb_dev, n, out_dev, ready.data(), nullptr, nullptr, nullptr);
            std::vector<uint64_t> ch(per * nl);
            EKV_CUDA(cudaMemcpyAsync(ch.data(), dch, sizeof(uint64_t) * ch.size(), cudaMemcpyDeviceToHost, hs));
            EKV_CUDA(cudaFreeAsync(dch, hs));
            dch = nullptr;
            EKV_CUDA(cudaStreamSynchronize(hs));
            EKV_CUDA(cudaStreamSynchronize(cp));
            EKV_CUDA(cudaStreamSynchronize(st));
            for (int i = 0; i < nl; ++i)
                require(fnv1a(ch.data() + (size_t)i * per, sizeof(uint64_t) * per) == v.lfnv[i],
                        "kvpack: checksum mismatch in layer " + std::to_string(v.edge[i]) +
                            " (the forward's outputs and the context's layers are invalid)");
        } catch (...) {
            cudaStreamSynchronize(hs);
            if (dch) cudaFreeAsync(dch, cp);
            cudaStreamSynchronize(cp);
            cudaStreamSynchronize(st);
            cleanup();
            throw;
        }
        cleanup();
    });
}

}  // extern "C"
