// C++ mirror of the reference interface (include/edgekv_b200.hpp) over the
// B200 C ABI (include/ekv_capi.h).  Host-side work here is marshalling,
// validation with the reference's messages and the scalar arithmetic the
// reference does on the host; every tensor operation runs on the device.
#include "edgekv_b200.hpp"

#include <algorithm>
#include <cmath>
#include <cstring>
#include <memory>
#include <mutex>
#include <numeric>
#include <set>
#include <stdexcept>
#include <string>

#include "ekv_capi.h"

namespace edgekv {

namespace {

std::string shape_str(const Matrix& m) {
    return std::to_string(m.rows) + "x" + std::to_string(m.cols);
}

void check(int rc) {
    if (rc != EKV_OK) throw std::invalid_argument(ekv_last_error());
}


uint16_t to_bf16(double x) {
    float f = static_cast<float>(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x7FFFFFu)) return static_cast<uint16_t>((u >> 16) | 0x40);
    u += 0x7FFFu + ((u >> 16) & 1u);
    return static_cast<uint16_t>(u >> 16);
}

ekv_ctx_t device_ctx();

// Device buffer owned by the mirror (allocated through the C ABI).
struct DevBuf {
    void* p = nullptr;
    size_t n = 0;
    explicit DevBuf(size_t bytes) : n(bytes) { check(ekv_device_alloc(device_ctx(), bytes ? bytes : 1, &p)); }
    ~DevBuf() { ekv_device_free(device_ctx(), p); }
    DevBuf(const DevBuf&) = delete;
    DevBuf& operator=(const DevBuf&) = delete;
    void put(const void* host) { check(ekv_copy(device_ctx(), p, host, n, 0)); }
    void get(void* host, size_t bytes) const { check(ekv_copy(device_ctx(), host, p, bytes, 1)); }
};

struct Runtime {
    std::mutex mu;
    int device = 0;
    ekv_ctx_t ctx = nullptr;
    // device copies of Model objects, keyed by a hash of ALL their weight data
    // (a reference caller may mutate weights in place), least recently used first
    struct ModelEntry {
        uint64_t signature = 0;
        ekv_model_t handle = nullptr;
    };
    static constexpr size_t kMaxModels = 4;
    std::vector<ModelEntry> models;

    ekv_ctx_t get() {
        if (!ctx) {
            check(ekv_ctx_create(device, nullptr, &ctx));
        }
        return ctx;
    }
    void* stream() {
        void* s = nullptr;
        check(ekv_ctx_stream(get(), &s));
        return s;
    }
};

Runtime& rt() {
    static Runtime r;
    return r;
}

ekv_ctx_t device_ctx() { return rt().get(); }

// 64-bit hash of every weight word of the model (word-wise multiply-xorshift:
// the same coverage as the reference's fnv1a checksum, transformer.cpp:118-131,
// at ~1 ns per double).
uint64_t signature(const Model& m) {
    uint64_t h = 0x9E3779B97F4A7C15ull;
    auto mixw = [&](uint64_t u) {
        h ^= u + 0x9E3779B97F4A7C15ull + (h << 6) + (h >> 2);
        h *= 0xBF58476D1CE4E5B9ull;
    };
    auto mixv = [&](const std::vector<double>& v) {
        mixw(v.size());
        for (double x : v) {
            uint64_t u;
            std::memcpy(&u, &x, 8);
            mixw(u);
        }
    };
    const ModelConfig& c = m.config;
    mixw((uint64_t)c.num_layers), mixw((uint64_t)c.num_heads), mixw((uint64_t)c.head_dim),
        mixw((uint64_t)c.max_positions);
    for (const LayerWeights& lw : m.layers) {
        for (const HeadWeights& w : lw.heads)
            for (const Matrix* x : {&w.wq, &w.wk, &w.wv}) mixv(x->data);
        mixv(lw.out_proj.data);
        mixv(lw.gamma);
        mixv(lw.bias);
    }
    mixv(m.pos_embedding.data);
    return h;
}

// fp64 reference layout -> bf16 B200 layout (wqkvT [3h][h], woT [h][h]).
ekv_model_t upload_model(ekv_ctx_t ctx, const Model& m) {
    const ModelConfig& c = m.config;
    c.validate();
    const int L = c.num_layers, H = c.num_heads, d = c.head_dim, h = c.hidden_size;
    ekv_model_config cfg{L, H, d, c.max_positions};
    ekv_model_t mh = nullptr;
    check(ekv_model_create(ctx, &cfg, &mh));
    std::vector<uint16_t> wqkv((size_t)3 * h * h), wo((size_t)h * h);
    for (int l = 0; l < L; ++l) {
        const LayerWeights& lw = m.layers[l];
        for (int hd = 0; hd < H; ++hd) {
            const HeadWeights& w = lw.heads[hd];
            const Matrix* parts[3] = {&w.wq, &w.wk, &w.wv};
            for (int part = 0; part < 3; ++part)
                for (int cix = 0; cix < d; ++cix) {
                    uint16_t* row = wqkv.data() + (size_t)(part * h + hd * d + cix) * h;
                    for (int k = 0; k < h; ++k) row[k] = to_bf16((*parts[part])(k, cix));
                }
        }
        for (int j = 0; j < h; ++j)
            for (int i = 0; i < h; ++i) wo[(size_t)j * h + i] = to_bf16(lw.out_proj(i, j));
        check(ekv_model_set_layer(mh, l, wqkv.data(), wo.data()));
    }
    std::vector<float> gamma(h), bias(h);
    for (int i = 0; i < h; ++i) {
        gamma[i] = static_cast<float>(m.layers[0].gamma[i]);
        bias[i] = static_cast<float>(m.layers[0].bias[i]);
    }
    std::vector<uint16_t> pos((size_t)c.max_positions * h);
    for (size_t i = 0; i < pos.size(); ++i) pos[i] = to_bf16(m.pos_embedding.data[i]);
    check(ekv_model_set_io(mh, gamma.data(), bias.data(), pos.data()));
    return mh;
}

// The device copy of `m` (uploaded on first use, re-uploaded when any weight
// changed; at most Runtime::kMaxModels kept).  Caller holds rt().mu.
ekv_model_t device_model(const Model& m) {
    Runtime& r = rt();
    const uint64_t sig = signature(m);
    for (size_t i = 0; i < r.models.size(); ++i)
        if (r.models[i].signature == sig) {
            Runtime::ModelEntry e = r.models[i];
            r.models.erase(r.models.begin() + (long)i);
            r.models.push_back(e);  // most recently used last
            return e.handle;
        }
    if (r.models.size() >= Runtime::kMaxModels) {
        ekv_model_destroy(r.models.front().handle);
        r.models.erase(r.models.begin());
    }
    ekv_model_t h = upload_model(r.get(), m);
    r.models.push_back(Runtime::ModelEntry{sig, h});
    return h;
}

std::vector<uint16_t> head_major_bf16(const std::vector<Matrix>& per_head, int S, int d) {
    std::vector<uint16_t> out((size_t)per_head.size() * S * d);
    for (size_t hd = 0; hd < per_head.size(); ++hd)
        for (size_t i = 0; i < (size_t)S * d; ++i) out[hd * S * d + i] = to_bf16(per_head[hd].data[i]);
    return out;
}

}  // namespace

// ---------------------------------------------------------------- value types
void ModelConfig::validate() const {
    if (num_layers < 1) throw std::invalid_argument("ModelConfig: num_layers must be >= 1");
    if (head_dim < 1) throw std::invalid_argument("ModelConfig: head_dim must be >= 1");
    if (num_heads < 1) throw std::invalid_argument("ModelConfig: num_heads must be >= 1");
    if (max_positions < 1) throw std::invalid_argument("ModelConfig: max_positions must be >= 1");
    if (hidden_size != num_heads * head_dim)
        throw std::invalid_argument("ModelConfig: hidden_size " + std::to_string(hidden_size) +
                                    " != num_heads*head_dim " + std::to_string(num_heads * head_dim));
}

KVCache KVCache::empty_for(int layers, int heads, int dim) {
    KVCache c;
    c.num_layers = layers;
    c.num_heads = heads;
    c.head_dim = dim;
    c.keys.assign(layers, std::vector<Matrix>(heads, Matrix(0, dim)));
    c.values.assign(layers, std::vector<Matrix>(heads, Matrix(0, dim)));
    return c;
}

PruneSpec PruneSpec::from_lambda(double lambda, int head_dim) {
    int retained = 0;
    check(ekv_prune_retained(lambda, head_dim, &retained));
    PruneSpec s;
    s.lambda = lambda;
    s.head_dim = head_dim;
    s.retained = retained;
    s.validate();
    return s;
}

void PruneSpec::validate() const {
    if (lambda < 0.0 || lambda > 1.0) throw std::invalid_argument("PruneSpec: lambda outside [0,1]");
    if (head_dim < 1) throw std::invalid_argument("PruneSpec: head_dim must be >= 1");
    int budget = 0;
    check(ekv_prune_retained(lambda, head_dim, &budget));
    if (retained != budget)
        throw std::invalid_argument("PruneSpec: retained " + std::to_string(retained) +
                                    " != floor((1-lambda)*head_dim) = " + std::to_string(budget));
}

void ChannelMask::validate() const {
    int prev = -1;
    for (int c : kept) {
        if (c <= prev || c < 0 || c >= head_dim)
            throw std::invalid_argument(
                "ChannelMask: kept channels must be unique, ascending and < head_dim");
        prev = c;
    }
}

ChannelMask ChannelMask::full(int head_dim) {
    ChannelMask m;
    m.head_dim = head_dim;
    m.kept.resize(head_dim);
    std::iota(m.kept.begin(), m.kept.end(), 0);
    return m;
}

double SegmentAttention::sigma_raw() const { return sigma * std::exp(shift); }

void SimilarityConfig::validate() const {
    if (theta_cka < 0.0) throw std::invalid_argument("SimilarityConfig: theta_cka must be >= 0");
    if (theta_rsa < -1.0) throw std::invalid_argument("SimilarityConfig: theta_rsa must be >= -1");
    if (num_probe_samples < 2)
        throw std::invalid_argument("SimilarityConfig: num_probe_samples must be >= 2");
}

// ---------------------------------------------------------------- alignment
ChannelMask select_channels(const Matrix& q, const Matrix& k, const PruneSpec& spec) {
    spec.validate();
    if (q.cols != k.cols || static_cast<int>(q.cols) != spec.head_dim)
        throw std::invalid_argument("select_channels: dim mismatch (Q " + shape_str(q) + ", K " +
                                    shape_str(k) + ", spec dim " + std::to_string(spec.head_dim) + ")");
    std::lock_guard<std::mutex> g(rt().mu);
    ekv_ctx_t ctx = rt().get();
    const int d = spec.head_dim;
    // column sums of squares in fp64 on the device (no rounding of Q / K)
    DevBuf sums(sizeof(double) * 2 * d);
    check(ekv_memset(ctx, sums.p, 0, sums.n));
    for (int which = 0; which < 2; ++which) {
        const Matrix& m = which ? k : q;
        if (m.rows == 0) continue;
        DevBuf dev(m.data.size() * 8);
        dev.put(m.data.data());
        check(ekv_colsq_f64(ctx, (const double*)dev.p, (int64_t)m.rows, d, (double*)sums.p + which * d));
        check(ekv_ctx_synchronize(ctx));
    }
    std::vector<double> both(2 * d);
    sums.get(both.data(), sizeof(double) * 2 * d);
    ChannelMask mask;
    mask.head_dim = d;
    mask.kept.resize(spec.retained);
    check(ekv_rank_channels(both.data(), both.data() + d, d, spec.retained, mask.kept.data(), nullptr));
    return mask;
}

KVCache prune_cache(const KVCache& cache, const ChannelMask& mask) {
    if (mask.head_dim != cache.head_dim)
        throw std::invalid_argument("prune_cache: mask dim " + std::to_string(mask.head_dim) +
                                    " != cache head_dim " + std::to_string(cache.head_dim));
    mask.validate();
    const int d_c = cache.head_dim, d_e = static_cast<int>(mask.kept.size());
    KVCache out = KVCache::empty_for(cache.num_layers, cache.num_heads, d_e);
    out.positions = cache.positions;
    if (d_e == 0) return out;
    std::lock_guard<std::mutex> g(rt().mu);
    ekv_ctx_t ctx = rt().get();
    DevBuf kept(sizeof(int) * d_e);
    kept.put(mask.kept.data());
    for (int l = 0; l < cache.num_layers; ++l)
        for (int h = 0; h < cache.num_heads; ++h)
            for (int kv = 0; kv < 2; ++kv) {
                const Matrix& src = kv ? cache.values[l][h] : cache.keys[l][h];
                Matrix& dst = kv ? out.values[l][h] : out.keys[l][h];
                dst = Matrix(src.rows, d_e);
                if (src.rows == 0) continue;
                DevBuf a(src.data.size() * 8), b(dst.data.size() * 8);
                a.put(src.data.data());
                check(ekv_gather_columns(ctx, a.p, (int64_t)src.rows, d_c, (const int*)kept.p, d_e, 8, b.p));
                check(ekv_ctx_synchronize(ctx));
                b.get(dst.data.data(), b.n);
            }
    return out;
}

// ---------------------------------------------------------------- transformer
QkvRows project_qkv(const Model& model, const Matrix& x, int layer, int head) {
    const ModelConfig& cfg = model.config;
    if (layer < 0 || layer >= cfg.num_layers)
        throw std::invalid_argument("project_qkv: layer " + std::to_string(layer) + " out of range [0," +
                                    std::to_string(cfg.num_layers - 1) + "]");
    if (head < 0 || head >= cfg.num_heads)
        throw std::invalid_argument("project_qkv: head " + std::to_string(head) + " out of range [0," +
                                    std::to_string(cfg.num_heads - 1) + "]");
    if (static_cast<int>(x.cols) != cfg.hidden_size)
        throw std::invalid_argument("project_qkv: input has " + std::to_string(x.cols) +
                                    " cols, expected hidden_size " + std::to_string(cfg.hidden_size));
    const HeadWeights& w = model.layers[layer].heads[head];
    const int n = (int)x.rows, h = cfg.hidden_size, d = cfg.head_dim;
    QkvRows r{Matrix(n, d), Matrix(n, d), Matrix(n, d)};
    if (n == 0) return r;
    std::lock_guard<std::mutex> g(rt().mu);
    ekv_ctx_t ctx = rt().get();
    DevBuf dx(x.data.size() * 8), dw((size_t)h * d * 8), dout((size_t)n * d * 8);
    dx.put(x.data.data());
    const Matrix* ws[3] = {&w.wq, &w.wk, &w.wv};
    Matrix* outs[3] = {&r.q, &r.k, &r.v};
    for (int i = 0; i < 3; ++i) {
        dw.put(ws[i]->data.data());
        check(ekv_matmul_f64(ctx, (const double*)dx.p, (const double*)dw.p, n, h, d, (double*)dout.p));
        check(ekv_ctx_synchronize(ctx));
        dout.get(outs[i]->data.data(), dout.n);
    }
    return r;
}

std::vector<Matrix> forward_rows(const Model& model, KVCache& cache, const Matrix& embeddings,
                                 PositionKind kind, FlopCounts* fc) {
    const ModelConfig& cfg = model.config;
    if (cache.num_layers != cfg.num_layers || cache.num_heads != cfg.num_heads ||
        cache.head_dim != cfg.head_dim)
        throw std::invalid_argument("forward_rows: cache shape does not match model");
    if (static_cast<int>(embeddings.cols) != cfg.hidden_size)
        throw std::invalid_argument("forward_rows: embeddings have " + std::to_string(embeddings.cols) +
                                    " cols, expected hidden_size " + std::to_string(cfg.hidden_size));
    const int n = static_cast<int>(embeddings.rows);
    const int old = cache.size();
    if (old + n > cfg.max_positions)
        throw std::invalid_argument("position overflow: " + std::to_string(old + n) +
                                    " > max_positions " + std::to_string(cfg.max_positions));
    const int L = cfg.num_layers, H = cfg.num_heads, d = cfg.head_dim, h = cfg.hidden_size;
    std::vector<Matrix> outs;
    if (n == 0) {
        for (int l = 0; l < L; ++l) outs.emplace_back(0, h);
        return outs;
    }
    std::vector<float> lo((size_t)L * n * h);
    std::vector<uint16_t> kb((size_t)L * H * n * d), vb(kb.size());
    {
        std::lock_guard<std::mutex> g(rt().mu);
        ekv_ctx_t ctx = rt().get();
        ekv_model_t mh = device_model(model);
        ekv_kvctx_t kvc = nullptr;
        std::unique_ptr<ekv_kvctx_s, int (*)(ekv_kvctx_t)> kguard(nullptr, ekv_kvctx_destroy);
        if (old > 0) {  // the cached rows become the context the new rows attend to
            std::vector<int> fmt(L, EKV_KV_BF16);
            check(ekv_kvctx_create(mh, old, fmt.data(), d, &kvc));
            kguard.reset(kvc);
            for (int l = 0; l < L; ++l) {
                auto k = head_major_bf16(cache.keys[l], old, d);
                auto v = head_major_bf16(cache.values[l], old, d);
                check(ekv_kvctx_upload_bf16(kvc, l, k.data(), v.data()));
            }
        }
        std::vector<float> e(embeddings.data.begin(), embeddings.data.end());
        DevBuf de(e.size() * 4), dlo(lo.size() * 4), dk(kb.size() * 2), dv(vb.size() * 2);
        de.put(e.data());
        check(ekv_forward_rows(mh, kvc, (const float*)de.p, n, (float*)dlo.p, nullptr, dk.p, dv.p));
        dlo.get(lo.data(), dlo.n);
        dk.get(kb.data(), dk.n);
        dv.get(vb.data(), dv.n);
    }
    auto f = [](uint16_t b) {
        const uint32_t u = (uint32_t)b << 16;
        float x;
        std::memcpy(&x, &u, 4);
        return (double)x;
    };
    for (int l = 0; l < L; ++l) {
        Matrix x(n, h);
        for (size_t i = 0; i < x.data.size(); ++i) x.data[i] = lo[(size_t)l * n * h + i];
        outs.push_back(std::move(x));
        for (int hd = 0; hd < H; ++hd) {
            Matrix& ck = cache.keys[l][hd];
            Matrix& cv = cache.values[l][hd];
            const size_t base = ((size_t)l * H + hd) * n * d;
            ck.data.reserve(ck.data.size() + (size_t)n * d);
            cv.data.reserve(cv.data.size() + (size_t)n * d);
            for (size_t i = 0; i < (size_t)n * d; ++i) {
                ck.data.push_back(f(kb[base + i]));
                cv.data.push_back(f(vb[base + i]));
            }
            ck.rows += n;
            cv.rows += n;
            ck.cols = cv.cols = d;
        }
    }
    for (int i = 0; i < n; ++i) cache.positions.push_back(PositionTag{kind, old + i});
    if (fc) {  // the reference's closed-form counts (transformer.cpp:267-283)
        const int64_t k = H;
        fc->proj += 3ll * n * h + (int64_t)L * n * k * 3 * d * (2ll * h - 1);
        for (int l = 0; l < L; ++l)
            for (int i = 0; i < n; ++i) {
                const int64_t vis = old + i + 1;
                fc->score += k * vis * (2ll * d - 1);
                fc->softmax += k * (3 * vis + 1);
                fc->value += k * (vis * 2 * d + d);
            }
        fc->out_proj += (int64_t)L * n * h * (2ll * h - 1);
    }
    return outs;
}

PrefillResult prefill(const Model& model, const Matrix& embeddings, FlopCounts* fc, PositionKind kind) {
    PrefillResult res;
    res.cache = KVCache::empty_for(model.config.num_layers, model.config.num_heads, model.config.head_dim);
    res.layer_outputs = forward_rows(model, res.cache, embeddings, kind, fc);
    return res;
}

Vec decode_step(const Model& model, KVCache& cache, const Vec& embedding, FlopCounts* fc,
                PositionKind kind) {
    if (static_cast<int>(embedding.size()) != model.config.hidden_size)
        throw std::invalid_argument("decode_step: embedding size " + std::to_string(embedding.size()) +
                                    " != hidden_size " + std::to_string(model.config.hidden_size));
    Matrix row(1, embedding.size());
    row.data = embedding;
    std::vector<Matrix> outs = forward_rows(model, cache, row, kind, fc);
    return outs.back().row(0);
}

// ---------------------------------------------------------------- decode attention
SegmentAttention segment_attention(const Vec& q, const Matrix& k, const Matrix& v) {
    if (k.rows == 0 || v.rows == 0) throw std::invalid_argument("segment_attention: empty segment");
    if (k.rows != v.rows)
        throw std::invalid_argument("segment_attention: K/V row mismatch (" + shape_str(k) + " vs " +
                                    shape_str(v) + ")");
    if (q.size() != k.cols)
        throw std::invalid_argument("segment_attention: q has " + std::to_string(q.size()) +
                                    " dims, K has " + std::to_string(k.cols));
    const int d = static_cast<int>(k.cols), n = static_cast<int>(k.rows), vd = static_cast<int>(v.cols);
    std::lock_guard<std::mutex> g(rt().mu);
    ekv_ctx_t ctx = rt().get();
    DevBuf dq(q.size() * 8), dk(k.data.size() * 8), dv(v.data.size() * 8), dout((size_t)vd * 8);
    dq.put(q.data());
    dk.put(k.data.data());
    dv.put(v.data.data());
    SegmentAttention res;
    check(ekv_segment_attention_f64(ctx, (const double*)dq.p, (const double*)dk.p, (const double*)dv.p, n,
                                    d, vd, (double*)dout.p, &res.sigma, &res.shift));
    res.o.resize(vd);
    dout.get(res.o.data(), dout.n);
    return res;
}

MergedAttention merge_attention(const SegmentAttention& ctx, const SegmentAttention& user) {
    if (ctx.o.size() != user.o.size())
        throw std::invalid_argument("merge_attention: head_dim mismatch (" +
                                    std::to_string(ctx.o.size()) + " vs " +
                                    std::to_string(user.o.size()) + ")");
    if (!(ctx.sigma > 0.0) || !(user.sigma > 0.0) || !std::isfinite(ctx.sigma) ||
        !std::isfinite(user.sigma))
        throw std::invalid_argument("merge_attention: non-positive or non-finite sigma");
    const double m = std::max(ctx.shift, user.shift);
    const double sc = ctx.sigma * std::exp(ctx.shift - m);
    const double su = user.sigma * std::exp(user.shift - m);
    MergedAttention r;
    r.weights.alpha_ctx = sc / (sc + su);
    r.weights.alpha_user = su / (sc + su);
    r.o.resize(ctx.o.size());
    for (size_t i = 0; i < r.o.size(); ++i)
        r.o[i] = r.weights.alpha_ctx * ctx.o[i] + r.weights.alpha_user * user.o[i];
    return r;
}

AssembledContext assemble_context(const std::map<int, LayerKV>& shared,
                                  const std::map<int, LayerKV>& local,
                                  const std::map<int, CacheOrigin>& shared_origins,
                                  int expected_layers) {
    const int total = expected_layers >= 0 ? expected_layers
                                           : static_cast<int>(shared.size() + local.size());
    if (total == 0) throw std::invalid_argument("assemble_context: no layers supplied");
    std::vector<const LayerKV*> by(total, nullptr);
    std::vector<CacheOrigin> prov(total, CacheOrigin::local);
    auto place = [&](int layer, const LayerKV& kv, CacheOrigin o) {
        if (layer < 0 || layer >= total)
            throw std::invalid_argument("assemble_context: layer " + std::to_string(layer) +
                                        " outside 0.." + std::to_string(total - 1));
        if (by[layer]) throw std::invalid_argument("assemble_context: duplicate layer " + std::to_string(layer));
        by[layer] = &kv;
        prov[layer] = o;
    };
    for (const auto& [l, kv] : local) place(l, kv, CacheOrigin::local);
    for (const auto& [l, kv] : shared) {
        auto it = shared_origins.find(l);
        place(l, kv, it == shared_origins.end() ? CacheOrigin::cloud : it->second);
    }
    for (int l = 0; l < total; ++l)
        if (!by[l]) throw std::invalid_argument("assemble_context: missing layer " + std::to_string(l));
    if (by[0]->keys.empty()) throw std::invalid_argument("assemble_context: layer 0 has no heads");
    const int heads = static_cast<int>(by[0]->keys.size());
    const int dim = static_cast<int>(by[0]->keys[0].cols);
    const int pos = static_cast<int>(by[0]->keys[0].rows);
    AssembledContext out;
    out.cache = KVCache::empty_for(total, heads, dim);
    out.provenance = prov;
    for (int l = 0; l < total; ++l) {
        const LayerKV& kv = *by[l];
        if ((int)kv.keys.size() != heads || (int)kv.values.size() != heads)
            throw std::invalid_argument("assemble_context: layer " + std::to_string(l) +
                                        " head count mismatch");
        for (int h = 0; h < heads; ++h) {
            const Matrix& k = kv.keys[h];
            const Matrix& v = kv.values[h];
            if ((int)k.cols != dim || (int)v.cols != dim || k.rows != v.rows || (int)k.rows != pos)
                throw std::invalid_argument("assemble_context: layer " + std::to_string(l) +
                                            " dim mismatch (K " + shape_str(k) + ", V " + shape_str(v) +
                                            ", expected " + std::to_string(pos) + "x" +
                                            std::to_string(dim) + ")");
            out.cache.keys[l][h] = k;
            out.cache.values[l][h] = v;
        }
    }
    for (int p = 0; p < pos; ++p) out.cache.positions.push_back(PositionTag{PositionKind::context, p});
    return out;
}

CollaborativeResult collaborative_decode(const Model& edge_model, const AssembledContext& context,
                                         const Matrix& user_embeddings, int steps) {
    const ModelConfig& cfg = edge_model.config;
    if (steps < 1) throw std::invalid_argument("collaborative_decode: steps must be >= 1");
    const int S = context.cache.size();
    if (S > 0) {
        if (context.cache.num_layers != cfg.num_layers)
            throw std::invalid_argument("collaborative_decode: context has " +
                                        std::to_string(context.cache.num_layers) + " layers, model has " +
                                        std::to_string(cfg.num_layers));
        if (context.cache.num_heads != cfg.num_heads || context.cache.head_dim != cfg.head_dim)
            throw std::invalid_argument(
                "collaborative_decode: context dims (heads " + std::to_string(context.cache.num_heads) +
                ", dim " + std::to_string(context.cache.head_dim) +
                ") do not match model; align with head pruning first");
    }
    const int U = static_cast<int>(user_embeddings.rows);
    if (S + U + steps > cfg.max_positions)
        throw std::invalid_argument("position overflow: " + std::to_string(S + U + steps) +
                                    " > max_positions " + std::to_string(cfg.max_positions));
    std::lock_guard<std::mutex> g(rt().mu);
    ekv_ctx_t ctx = rt().get();
    ekv_model_t mh = device_model(edge_model);
    const int L = cfg.num_layers, H = cfg.num_heads, d = cfg.head_dim, h = cfg.hidden_size;
    std::vector<int> fmt(L, EKV_KV_BF16);
    ekv_kvctx_t kvc = nullptr;
    check(ekv_kvctx_create(mh, S, fmt.data(), d, &kvc));
    std::unique_ptr<ekv_kvctx_s, int (*)(ekv_kvctx_t)> kguard(kvc, ekv_kvctx_destroy);
    for (int l = 0; l < L && S > 0; ++l) {
        auto kb = head_major_bf16(context.cache.keys[l], S, d);
        auto vb = head_major_bf16(context.cache.values[l], S, d);
        check(ekv_kvctx_upload_bf16(kvc, l, kb.data(), vb.data()));
    }
    ekv_session_t sess = nullptr;
    check(ekv_session_create(mh, kvc, U + steps, &sess));
    std::unique_ptr<ekv_session_s, int (*)(ekv_session_t)> sguard(sess, ekv_session_destroy);
    std::vector<float> ue((size_t)U * h), pre((size_t)std::max(U, 1) * h), st((size_t)steps * h);
    for (size_t i = 0; i < ue.size(); ++i) ue[i] = static_cast<float>(user_embeddings.data[i]);
    check(ekv_collaborative_decode(sess, ue.data(), U, steps, pre.data(), st.data()));
    CollaborativeResult r;
    for (int i = 0; i < U; ++i) r.prefill_outputs.emplace_back(pre.begin() + (size_t)i * h, pre.begin() + (size_t)(i + 1) * h);
    for (int t = 0; t < steps; ++t) r.step_outputs.emplace_back(st.begin() + (size_t)t * h, st.begin() + (size_t)(t + 1) * h);
    (void)H;
    return r;
}

// ---------------------------------------------------------------- layer matching
LayerMatchReport match_layers(const std::vector<Matrix>& edge_outputs,
                              const std::vector<Matrix>& cloud_outputs,
                              const SimilarityConfig& cfg) {
    cfg.validate();
    if (edge_outputs.empty() || cloud_outputs.empty())
        throw std::invalid_argument("match_layers: empty layer output list");
    const size_t n = edge_outputs[0].rows;
    for (const auto* list : {&edge_outputs, &cloud_outputs})
        for (const Matrix& m : *list)
            if (m.rows != n)
                throw std::invalid_argument("match_layers: probe row-count mismatch (" +
                                            std::to_string(m.rows) + " vs " + std::to_string(n) + ")");
    const int me = (int)edge_outputs.size(), nc = (int)cloud_outputs.size();
    const int ce = (int)edge_outputs[0].cols, cc = (int)cloud_outputs[0].cols;
    std::vector<double> e, c;
    for (const Matrix& m : edge_outputs) e.insert(e.end(), m.data.begin(), m.data.end());
    for (const Matrix& m : cloud_outputs) c.insert(c.end(), m.data.begin(), m.data.end());
    LayerMatchReport r;
    r.config = cfg;
    r.cka = Matrix(me, nc);
    r.rsa = Matrix(me, nc);
    std::vector<int> best(me);
    {
        std::lock_guard<std::mutex> g(rt().mu);
        check(ekv_match_layers(rt().get(), e.data(), me, ce, c.data(), nc, cc, (int)n, cfg.theta_cka,
                               cfg.theta_rsa, r.cka.data.data(), r.rsa.data.data(), best.data()));
    }
    r.best.assign(me, std::nullopt);
    for (int le = 0; le < me; ++le)
        if (best[le] >= 0) {
            r.best[le] = best[le];
            r.matches.push_back(LayerMatch{le, best[le], r.cka(le, best[le]), r.rsa(le, best[le])});
            r.shared_layers.push_back(le);
        }
    return r;
}

// ---------------------------------------------------------------- scheduler
CacheSource cache_source(int layer, double cost_local, double cost_peer, int boundary, int m) {
    int s = 0;
    check(ekv_cache_source(layer, cost_local, cost_peer, boundary, m, &s));
    return static_cast<CacheSource>(s);
}

ScheduleTrace pipeline_schedule(const std::vector<LayerTimes>& layers,
                                const std::vector<CacheSource>& sources) {
    if (!sources.empty() && sources.size() != layers.size())
        throw std::invalid_argument("pipeline_schedule: sources size mismatch");
    const int n = (int)layers.size();
    std::vector<double> comm(n), comp(n), pip(std::max(n, 1));
    for (int i = 0; i < n; ++i) {
        comm[i] = layers[i].t_comm;
        comp[i] = layers[i].t_comp;
    }
    ScheduleTrace t;
    check(ekv_pipeline_schedule(comm.data(), comp.data(), n, pip.data(), &t.sequential_total,
                                &t.pipelined_total));
    t.layers.resize(n);
    for (int i = 0; i < n; ++i)
        t.layers[i] = ScheduleEntry{sources.empty() ? CacheSource::local : sources[i], comm[i], comp[i], pip[i]};
    return t;
}

// ---------------------------------------------------------------- extensions
namespace b200 {

void set_device(int device) {
    std::lock_guard<std::mutex> g(rt().mu);
    if (rt().ctx) throw std::invalid_argument("b200::set_device: the device is already in use");
    rt().device = device;
}

void invalidate(const Model& model) {
    std::lock_guard<std::mutex> g(rt().mu);
    const uint64_t sig = signature(model);
    auto& ms = rt().models;
    for (size_t i = 0; i < ms.size(); ++i)
        if (ms[i].signature == sig) {
            ekv_model_destroy(ms[i].handle);
            ms.erase(ms.begin() + (long)i);
            return;
        }
}

std::vector<QuantizedLayer> compress_cache(const KVCache& cache, const ChannelMask& mask, int bits,
                                           int group) {
    if (mask.head_dim != cache.head_dim)
        throw std::invalid_argument("prune_cache: mask dim " + std::to_string(mask.head_dim) +
                                    " != cache head_dim " + std::to_string(cache.head_dim));
    mask.validate();
    const int d_c = cache.head_dim, d_e = (int)mask.kept.size(), H = cache.num_heads;
    if (group == 0) group = bits == 8 ? d_e : 32;
    std::lock_guard<std::mutex> g(rt().mu);
    ekv_ctx_t ctx = rt().get();
    DevBuf kept(sizeof(int) * d_e);
    kept.put(mask.kept.data());
    std::vector<QuantizedLayer> out(cache.num_layers);
    const int S = cache.size();
    for (int l = 0; l < cache.num_layers; ++l) {
        QuantizedLayer& q = out[l];
        q.bits = bits;
        q.group = group;
        q.head_dim = d_e;
        q.positions = S;
        const size_t rows = (size_t)H * S;
        q.k_codes.resize(rows * d_e * bits / 8);
        q.v_codes.resize(q.k_codes.size());
        q.k_scales.resize(rows * (d_e / group));
        q.v_scales.resize(q.k_scales.size());
        if (rows == 0) continue;
        for (int kv = 0; kv < 2; ++kv) {
            auto src = head_major_bf16(kv ? cache.values[l] : cache.keys[l], S, d_c);
            DevBuf ds(src.size() * 2), dc(q.k_codes.size()), dsc(q.k_scales.size() * 4);
            ds.put(src.data());
            check(ekv_kv_compress(ctx, ds.p, (int64_t)rows, d_c, (const int*)kept.p, d_e, bits, group,
                                  dc.p, (float*)dsc.p));
            check(ekv_ctx_synchronize(ctx));
            dc.get(kv ? q.v_codes.data() : q.k_codes.data(), dc.n);
            dsc.get(kv ? q.v_scales.data() : q.k_scales.data(), dsc.n);
        }
    }
    return out;
}

LayerKV dequantize(const QuantizedLayer& q, int num_heads) {
    LayerKV kv;
    const int d = q.head_dim, S = q.positions;
    const size_t rows = (size_t)num_heads * S;
    if (q.k_codes.size() != rows * d * q.bits / 8 || q.k_scales.size() != rows * (d / q.group))
        throw std::invalid_argument("dequantize: code / scale sizes do not match the layer shape");
    std::vector<double> k(rows * d), v(rows * d);
    if (rows > 0) {
        std::lock_guard<std::mutex> g(rt().mu);
        ekv_ctx_t ctx = rt().get();
        DevBuf dc(q.k_codes.size()), ds(q.k_scales.size() * 4), out(rows * d * 8);
        for (int which = 0; which < 2; ++which) {
            dc.put(which ? q.v_codes.data() : q.k_codes.data());
            ds.put(which ? q.v_scales.data() : q.k_scales.data());
            check(ekv_kv_dequant_f64(ctx, dc.p, (const float*)ds.p, (int64_t)rows, d, q.bits, q.group,
                                     (double*)out.p));
            check(ekv_ctx_synchronize(ctx));
            out.get(which ? v.data() : k.data(), out.n);
        }
    }
    for (int h = 0; h < num_heads; ++h) {
        Matrix km(S, d), vm(S, d);
        std::copy(k.begin() + (size_t)h * S * d, k.begin() + (size_t)(h + 1) * S * d, km.data.begin());
        std::copy(v.begin() + (size_t)h * S * d, v.begin() + (size_t)(h + 1) * S * d, vm.data.begin());
        kv.keys.push_back(std::move(km));
        kv.values.push_back(std::move(vm));
    }
    return kv;
}

DeepKV build_deep_kv(const Model& cloud_model, const PrefillResult& cloud_prefill,
                     const Matrix& ctx_emb_cloud, const std::map<int, int>& match,
                     const PruneSpec& spec) {
    spec.validate();
    const ModelConfig& cc = cloud_model.config;
    if (spec.head_dim != cc.head_dim)
        throw std::invalid_argument("select_channels: dim mismatch (spec dim " +
                                    std::to_string(spec.head_dim) + ", cloud head_dim " +
                                    std::to_string(cc.head_dim) + ")");
    const int S = cloud_prefill.cache.size(), H = cc.num_heads, dc = cc.head_dim, hc = cc.hidden_size;
    if ((int)ctx_emb_cloud.rows != S || (int)ctx_emb_cloud.cols != hc)
        throw std::invalid_argument("build_deep_kv: context embeddings do not match the cloud prefill");
    std::set<int> layers;
    for (const auto& [le, lc] : match) {
        if (lc < 0 || lc >= cc.num_layers)
            throw std::invalid_argument("build_deep_kv: matched cloud layer " + std::to_string(lc) +
                                        " out of range");
        layers.insert(lc);
    }
    DeepKV out;
    if (match.empty()) return out;
    const std::vector<int> lcs(layers.begin(), layers.end());
    const int m = (int)lcs.size();
    if (spec.retained == dc) {
        out.mask = ChannelMask::full(dc);
        out.cut_margin = INFINITY;
    } else {
        // X_lc (bf16) = x0 for lc == 0 (sim.cpp:224-234), else the cloud prefill's layer lc-1 output
        std::vector<uint16_t> xb((size_t)m * S * hc);
        for (int i = 0; i < m; ++i) {
            uint16_t* dst = xb.data() + (size_t)i * S * hc;
            if (lcs[i] == 0) {
                for (int r = 0; r < S; ++r)
                    for (int c = 0; c < hc; ++c)
                        dst[(size_t)r * hc + c] = to_bf16(cloud_model.layers[0].gamma[c] *
                                                              (ctx_emb_cloud(r, c) + cloud_model.pos_embedding(r, c)) +
                                                          cloud_model.layers[0].bias[c]);
            } else {
                const Matrix& x = cloud_prefill.layer_outputs[lcs[i] - 1];
                for (size_t j = 0; j < x.data.size(); ++j) dst[j] = to_bf16(x.data[j]);
            }
        }
        std::lock_guard<std::mutex> g(rt().mu);
        ekv_ctx_t ctx = rt().get();
        ekv_model_t mh = device_model(cloud_model);
        void* w0 = nullptr;
        void* wo = nullptr;
        check(ekv_model_weights(mh, 0, &w0, &wo));
        DevBuf dx(xb.size() * 2);
        dx.put(xb.data());
        std::vector<std::unique_ptr<DevBuf>> kbuf;
        std::vector<const void*> kp;
        for (int lc : lcs) {
            auto kb = head_major_bf16(cloud_prefill.cache.keys[lc], S, dc);
            kbuf.push_back(std::make_unique<DevBuf>(kb.size() * 2));
            kbuf.back()->put(kb.data());
            kp.push_back(kbuf.back()->p);
        }
        ekv_cloud_kv cl{};
        cl.m = m;
        cl.S = S;
        cl.H = H;
        cl.d_c = dc;
        cl.x = dx.p;
        cl.wq = w0;
        cl.wq_stride = (int64_t)4 * hc * hc;
        cl.wq_index = lcs.data();
        cl.k = kp.data();
        cl.v = kp.data();
        out.mask.head_dim = dc;
        out.mask.kept.resize(spec.retained);
        check(ekv_align_select(ctx, &cl, spec.lambda, out.mask.kept.data(), &out.cut_margin));
    }
    const KVCache pruned = prune_cache(cloud_prefill.cache, out.mask);
    for (const auto& [le, lc] : match) {
        LayerKV kv;
        kv.keys = pruned.keys[lc];
        kv.values = pruned.values[lc];
        out.deep_kv[le] = std::move(kv);
    }
    return out;
}

}  // namespace b200
}  // namespace edgekv
