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
    struct ModelEntry {
        ekv_model_t handle = nullptr;
        uint64_t signature = 0;
    };
    std::map<const Model*, ModelEntry> models;

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

uint64_t signature(const Model& m) {
    uint64_t h = 1469598103934665603ull;
    auto mix = [&](double v) {
        uint64_t u;
        std::memcpy(&u, &v, 8);
        h = (h ^ u) * 1099511628211ull;
    };
    const ModelConfig& c = m.config;
    mix(c.num_layers), mix(c.num_heads), mix(c.head_dim), mix(c.max_positions);
    for (const LayerWeights& lw : m.layers) {
        for (const HeadWeights& w : lw.heads)
            for (const Matrix* x : {&w.wq, &w.wk, &w.wv})
                if (!x->data.empty()) mix(x->data.front()), mix(x->data.back());
        if (!lw.out_proj.data.empty()) mix(lw.out_proj.data.front()), mix(lw.out_proj.data.back());
    }
    if (!m.pos_embedding.data.empty()) mix(m.pos_embedding.data.back());
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
    std::vector<double> qsq(d, 0.0), ksq(d, 0.0);
    DevBuf sums(sizeof(double) * 2 * d);
    check(ekv_memset(ctx, sums.p, 0, sums.n));
    for (int which = 0; which < 2; ++which) {
        const Matrix& m = which ? k : q;
        if (m.rows == 0) continue;
        std::vector<uint16_t> b(m.data.size());
        for (size_t i = 0; i < b.size(); ++i) b[i] = to_bf16(m.data[i]);
        DevBuf dev(b.size() * 2);
        dev.put(b.data());
        check(ekv_kv_colnorm(ctx, dev.p, (int64_t)m.rows, d, (double*)sums.p + which * d));
        check(ekv_ctx_synchronize(ctx));
    }
    std::vector<double> both(2 * d);
    sums.get(both.data(), sizeof(double) * 2 * d);
    std::copy(both.begin(), both.begin() + d, qsq.begin());
    std::copy(both.begin() + d, both.end(), ksq.begin());
    ChannelMask mask;
    mask.head_dim = d;
    mask.kept.resize(spec.retained);
    check(ekv_rank_channels(qsq.data(), ksq.data(), d, spec.retained, mask.kept.data(), nullptr));
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

// ---------------------------------------------------------------- decode attention
SegmentAttention segment_attention(const Vec& q, const Matrix& k, const Matrix& v) {
    if (k.rows == 0 || v.rows == 0) throw std::invalid_argument("segment_attention: empty segment");
    if (k.rows != v.rows)
        throw std::invalid_argument("segment_attention: K/V row mismatch (" + shape_str(k) + " vs " +
                                    shape_str(v) + ")");
    if (q.size() != k.cols)
        throw std::invalid_argument("segment_attention: q has " + std::to_string(q.size()) +
                                    " dims, K has " + std::to_string(k.cols));
    const int d = static_cast<int>(k.cols), n = static_cast<int>(k.rows);
    if (v.cols != k.cols || !(d == 32 || d == 64 || d == 128))
        throw std::invalid_argument("segment_attention: head_dim " + std::to_string(d) +
                                    " has no B200 kernel (32, 64 or 128)");
    std::lock_guard<std::mutex> g(rt().mu);
    ekv_ctx_t ctx = rt().get();
    // the whole segment is the "user" segment of a one-row attention with no context
    std::vector<uint16_t> kb(k.data.size()), vb(v.data.size());
    for (size_t i = 0; i < kb.size(); ++i) kb[i] = to_bf16(k.data[i]);
    for (size_t i = 0; i < vb.size(); ++i) vb[i] = to_bf16(v.data[i]);
    std::vector<float> qf(q.begin(), q.end());
    DevBuf dk(kb.size() * 2), dv(vb.size() * 2), dq(qf.size() * 4), dout(qf.size() * 4), dlse(4);
    dk.put(kb.data());
    dv.put(vb.data());
    dq.put(qf.data());
    ekv_segment none{EKV_KV_BF16, 0, d, nullptr, nullptr, nullptr, nullptr};
    check(ekv_decode_attention(ctx, 1, 1, d, (const float*)dq.p, &none, dk.p, dv.p, n, n - 1,
                               (float*)dout.p, (float*)dlse.p));
    check(ekv_ctx_synchronize(ctx));
    std::vector<float> o(d);
    float lse = 0.0f;
    dout.get(o.data(), dout.n);
    dlse.get(&lse, 4);
    SegmentAttention res;
    res.o.assign(o.begin(), o.end());
    // the normaliser as (mantissa, shift) = (1, log-sum-exp): the same
    // sigma_raw = sigma * e^shift the reference carries, and merge_attention
    // only ever uses sigma * e^(shift - m)
    res.shift = lse;
    res.sigma = 1.0;
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
    Runtime::ModelEntry& me = rt().models[&edge_model];
    const uint64_t sig = signature(edge_model);
    if (!me.handle || me.signature != sig) {
        if (me.handle) ekv_model_destroy(me.handle);
        me.handle = upload_model(ctx, edge_model);
        me.signature = sig;
    }
    const int L = cfg.num_layers, H = cfg.num_heads, d = cfg.head_dim, h = cfg.hidden_size;
    std::vector<int> fmt(L, EKV_KV_BF16);
    ekv_kvctx_t kvc = nullptr;
    check(ekv_kvctx_create(me.handle, S, fmt.data(), d, &kvc));
    std::unique_ptr<ekv_kvctx_s, int (*)(ekv_kvctx_t)> kguard(kvc, ekv_kvctx_destroy);
    for (int l = 0; l < L && S > 0; ++l) {
        auto kb = head_major_bf16(context.cache.keys[l], S, d);
        auto vb = head_major_bf16(context.cache.values[l], S, d);
        check(ekv_kvctx_upload_bf16(kvc, l, kb.data(), vb.data()));
    }
    ekv_session_t sess = nullptr;
    check(ekv_session_create(me.handle, kvc, U + steps, &sess));
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
    check(ekv_match_layers(e.data(), me, ce, c.data(), nc, cc, (int)n, cfg.theta_cka, cfg.theta_rsa,
                           r.cka.data.data(), r.rsa.data.data(), best.data()));
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
    auto it = rt().models.find(&model);
    if (it != rt().models.end()) {
        ekv_model_destroy(it->second.handle);
        rt().models.erase(it);
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
    const int d = q.head_dim, S = q.positions, ng = d / q.group, rb = d * q.bits / 8;
    auto code = [&](const std::vector<std::uint8_t>& c, size_t row, int col) {
        if (q.bits == 8) return (int)(int8_t)c[row * rb + col];
        const int nib = (c[row * rb + (col >> 1)] >> ((col & 1) * 4)) & 0xF;
        return nib >= 8 ? nib - 16 : nib;
    };
    for (int h = 0; h < num_heads; ++h) {
        Matrix k(S, d), v(S, d);
        for (int i = 0; i < S; ++i)
            for (int c = 0; c < d; ++c) {
                const size_t row = (size_t)h * S + i;
                k(i, c) = (double)code(q.k_codes, row, c) * (double)q.k_scales[row * ng + c / q.group];
                v(i, c) = (double)code(q.v_codes, row, c) * (double)q.v_scales[row * ng + c / q.group];
            }
        kv.keys.push_back(std::move(k));
        kv.values.push_back(std::move(v));
    }
    return kv;
}

}  // namespace b200
}  // namespace edgekv
