// ref_capi.cpp -- TEST INFRASTRUCTURE ONLY.
//
// A thin extern "C" shim over the UNMODIFIED reference library (edgekv_core,
// compiled from /root/reference/proj/src by oracle/Makefile into oracle/_ref/).
// It lets the Python tests pin the C restatement (oracle/ekv_oracle.c) against
// the real reference, lets tests/golden/make_golden.py emit golden vectors,
// and gives bench.py a "reference" CPU baseline (ref_bench_decode).
// Nothing here is product code; the product never links it.
//
// Weight layout translation: callers pass the B200 layout (wqkvT [L][3h][h],
// woT [L][h][h]); we populate edgekv::Model directly
// (transformer.hpp:76-83), exactly as SURVEY.md section 0 prescribes for
// scaled-init models.
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <set>
#include <string>
#include <thread>
#include <vector>

#include "edgekv/cache_merge.hpp"
#include "edgekv/cost_model.hpp"
#include "edgekv/head_prune.hpp"
#include "edgekv/layer_match.hpp"
#include "edgekv/matrix.hpp"
#include "edgekv/rng.hpp"
#include "edgekv/transformer.hpp"

using namespace edgekv;

namespace {
thread_local std::string g_err;

template <class F>
int guarded(F&& f) {
    try {
        return f();
    } catch (const std::exception& e) {
        g_err = e.what();
        return -1;
    }
}

Matrix to_matrix(const double* p, std::size_t r, std::size_t c) {
    Matrix m(r, c);
    if (r * c) std::memcpy(m.data.data(), p, sizeof(double) * r * c);
    return m;
}

// B200 layout -> edgekv::Model (reference layout).
Model make_model(int L, int H, int d, int max_pos, const double* wqkvT, const double* woT,
                 const double* gamma, const double* bias, const double* pos) {
    const int h = H * d;
    Model m;
    m.config.num_layers = L;
    m.config.num_heads = H;
    m.config.head_dim = d;
    m.config.hidden_size = h;
    m.config.max_positions = max_pos;
    m.config.validate();
    m.layers.resize(L);
    for (int l = 0; l < L; ++l) {
        LayerWeights& lw = m.layers[l];
        lw.heads.resize(H);
        const double* W = wqkvT + (std::size_t)l * 3 * h * h;
        for (int hd = 0; hd < H; ++hd) {
            HeadWeights& w = lw.heads[hd];
            w.wq = Matrix(h, d);
            w.wk = Matrix(h, d);
            w.wv = Matrix(h, d);
            for (int k = 0; k < h; ++k)
                for (int c = 0; c < d; ++c) {
                    w.wq(k, c) = W[(std::size_t)(0 * h + hd * d + c) * h + k];
                    w.wk(k, c) = W[(std::size_t)(1 * h + hd * d + c) * h + k];
                    w.wv(k, c) = W[(std::size_t)(2 * h + hd * d + c) * h + k];
                }
        }
        lw.out_proj = Matrix(h, h);
        const double* Wo = woT + (std::size_t)l * h * h;
        for (int i = 0; i < h; ++i)
            for (int j = 0; j < h; ++j) lw.out_proj(i, j) = Wo[(std::size_t)j * h + i];
        lw.gamma.assign(gamma, gamma + h);
        lw.bias.assign(bias, bias + h);
    }
    m.pos_embedding = to_matrix(pos, max_pos, h);
    return m;
}

// ctx_k/ctx_v: [L][H][S][d]; layers < boundary are "local", the rest "cloud".
AssembledContext make_context(int L, int H, int d, int S, const double* ck, const double* cv,
                              int boundary) {
    if (S == 0) {
        AssembledContext ctx;
        ctx.cache = KVCache::empty_for(L, H, d);
        return ctx;
    }
    std::map<int, LayerKV> local, shared;
    std::map<int, CacheOrigin> origins;
    for (int l = 0; l < L; ++l) {
        LayerKV kv;
        for (int hd = 0; hd < H; ++hd) {
            const std::size_t off = ((std::size_t)l * H + hd) * S * d;
            kv.keys.push_back(to_matrix(ck + off, S, d));
            kv.values.push_back(to_matrix(cv + off, S, d));
        }
        if (l < boundary) {
            local[l] = std::move(kv);
        } else {
            shared[l] = std::move(kv);
            origins[l] = CacheOrigin::cloud;
        }
    }
    return assemble_context(shared, local, origins, L);
}
}  // namespace

extern "C" {

const char* ref_last_error() { return g_err.c_str(); }

uint64_t ref_mix(uint64_t a, uint64_t b) { return Rng::mix(a, b); }

void ref_mt64_stream(uint64_t seed, int64_t n, uint64_t* out) {
    Rng r(seed);
    for (int64_t i = 0; i < n; ++i) out[i] = r.next_u64();
}

uint64_t ref_fnv1a64(const void* p, std::size_t n, uint64_t h) { return fnv1a64(p, n, h); }

// init_model (transformer.cpp:82-115) exported in the reference layout.
int ref_init_model(int L, int H, int d, int max_pos, uint64_t seed, double* wq, double* wk,
                   double* wv, double* out_proj, double* pos, uint64_t* checksum) {
    return guarded([&] {
        ModelConfig cfg;
        cfg.num_layers = L;
        cfg.num_heads = H;
        cfg.head_dim = d;
        cfg.hidden_size = H * d;
        cfg.max_positions = max_pos;
        cfg.seed = seed;
        Model m = init_model(cfg);
        const std::size_t hd_sz = (std::size_t)H * d * d;
        for (int l = 0; l < L; ++l) {
            for (int hd = 0; hd < H; ++hd) {
                const HeadWeights& w = m.layers[l].heads[hd];
                std::memcpy(wq + ((std::size_t)l * H + hd) * hd_sz, w.wq.data.data(), hd_sz * 8);
                std::memcpy(wk + ((std::size_t)l * H + hd) * hd_sz, w.wk.data.data(), hd_sz * 8);
                std::memcpy(wv + ((std::size_t)l * H + hd) * hd_sz, w.wv.data.data(), hd_sz * 8);
            }
            std::memcpy(out_proj + (std::size_t)l * H * d * H * d, m.layers[l].out_proj.data.data(),
                        (std::size_t)H * d * H * d * 8);
        }
        std::memcpy(pos, m.pos_embedding.data.data(), (std::size_t)max_pos * H * d * 8);
        *checksum = m.checksum();
        return 0;
    });
}

int ref_generate_embeddings(uint64_t seed, int n, int h, double* out) {
    return guarded([&] {
        Matrix m = generate_embeddings(seed, n, h);
        std::memcpy(out, m.data.data(), sizeof(double) * m.data.size());
        return 0;
    });
}

int ref_prune_retained(double lambda, int head_dim) {
    return guarded([&] { return PruneSpec::from_lambda(lambda, head_dim).retained; });
}

// select_channels (head_prune.cpp:83-108); returns the kept count.
int ref_select_channels(const double* q, int64_t q_rows, const double* k, int64_t k_rows, int d,
                        double lambda, int* kept) {
    return guarded([&] {
        ChannelMask m = select_channels(to_matrix(q, q_rows, d), to_matrix(k, k_rows, d),
                                        PruneSpec::from_lambda(lambda, d));
        for (std::size_t i = 0; i < m.kept.size(); ++i) kept[i] = m.kept[i];
        return (int)m.kept.size();
    });
}

double ref_prune_objective(const double* q, int64_t q_rows, const double* k, int64_t k_rows,
                           int d, const int* kept, int n_kept) {
    ChannelMask m;
    m.head_dim = d;
    m.kept.assign(kept, kept + n_kept);
    return prune_objective(to_matrix(q, q_rows, d), to_matrix(k, k_rows, d), m);
}

// prune_cache (head_prune.cpp:170-197) on a [L][H][S][d_c] cache.
int ref_prune_cache(int L, int H, int S, int d_c, const double* keys, const double* values,
                    const int* kept, int d_e, double* out_k, double* out_v) {
    return guarded([&] {
        KVCache c = KVCache::empty_for(L, H, d_c);
        for (int l = 0; l < L; ++l)
            for (int hd = 0; hd < H; ++hd) {
                const std::size_t off = ((std::size_t)l * H + hd) * S * d_c;
                c.keys[l][hd] = to_matrix(keys + off, S, d_c);
                c.values[l][hd] = to_matrix(values + off, S, d_c);
            }
        for (int p = 0; p < S; ++p) c.positions.push_back(PositionTag{PositionKind::context, p});
        ChannelMask m;
        m.head_dim = d_c;
        m.kept.assign(kept, kept + d_e);
        KVCache o = prune_cache(c, m);
        for (int l = 0; l < L; ++l)
            for (int hd = 0; hd < H; ++hd) {
                const std::size_t off = ((std::size_t)l * H + hd) * S * d_e;
                std::memcpy(out_k + off, o.keys[l][hd].data.data(), sizeof(double) * S * d_e);
                std::memcpy(out_v + off, o.values[l][hd].data.data(), sizeof(double) * S * d_e);
            }
        return 0;
    });
}

int ref_segment_attention(const double* q, const double* k, const double* v, int rows, int d,
                          int vd, double* o, double* sigma, double* shift) {
    return guarded([&] {
        Vec qv(q, q + d);
        SegmentAttention s = segment_attention(qv, to_matrix(k, rows, d), to_matrix(v, rows, vd));
        std::memcpy(o, s.o.data(), sizeof(double) * vd);
        *sigma = s.sigma;
        *shift = s.shift;
        return 0;
    });
}

int ref_merge_attention(const double* o_c, double sigma_c, double shift_c, const double* o_u,
                        double sigma_u, double shift_u, int d, double* o, double* alpha_ctx,
                        double* alpha_user) {
    return guarded([&] {
        SegmentAttention c, u;
        c.o.assign(o_c, o_c + d);
        c.sigma = sigma_c;
        c.shift = shift_c;
        u.o.assign(o_u, o_u + d);
        u.sigma = sigma_u;
        u.shift = shift_u;
        MergedAttention m = merge_attention(c, u);
        std::memcpy(o, m.o.data(), sizeof(double) * d);
        *alpha_ctx = m.weights.alpha_ctx;
        *alpha_user = m.weights.alpha_user;
        return 0;
    });
}

// collaborative_decode (cache_merge.cpp:230-273) on a B200-layout model.
int ref_collaborative_decode(int L, int H, int d, int max_pos, const double* wqkvT,
                             const double* woT, const double* gamma, const double* bias,
                             const double* pos, int S, const double* ctx_k, const double* ctx_v,
                             int boundary, const double* user_emb, int U, int steps,
                             double* prefill_out, double* step_out) {
    return guarded([&] {
        Model m = make_model(L, H, d, max_pos, wqkvT, woT, gamma, bias, pos);
        AssembledContext ctx = make_context(L, H, d, S, ctx_k, ctx_v, boundary);
        CollaborativeResult r = collaborative_decode(m, ctx, to_matrix(user_emb, U, H * d), steps);
        for (std::size_t i = 0; i < r.prefill_outputs.size(); ++i)
            std::memcpy(prefill_out + i * H * d, r.prefill_outputs[i].data(), sizeof(double) * H * d);
        for (std::size_t t = 0; t < r.step_outputs.size(); ++t)
            std::memcpy(step_out + t * H * d, r.step_outputs[t].data(), sizeof(double) * H * d);
        return 0;
    });
}

// prefill (transformer.cpp:244-251): per-layer outputs [L][n][h], K/V [L][H][n][d].
int ref_prefill(int L, int H, int d, int max_pos, const double* wqkvT, const double* woT,
                const double* gamma, const double* bias, const double* pos, const double* emb,
                int n, double* layer_out, double* k_out, double* v_out) {
    return guarded([&] {
        Model m = make_model(L, H, d, max_pos, wqkvT, woT, gamma, bias, pos);
        PrefillResult p = prefill(m, to_matrix(emb, n, H * d));
        const int h = H * d;
        for (int l = 0; l < L; ++l) {
            std::memcpy(layer_out + (std::size_t)l * n * h, p.layer_outputs[l].data.data(),
                        sizeof(double) * n * h);
            for (int hd = 0; hd < H; ++hd) {
                const std::size_t off = ((std::size_t)l * H + hd) * n * d;
                if (k_out) std::memcpy(k_out + off, p.cache.keys[l][hd].data.data(), sizeof(double) * n * d);
                if (v_out) std::memcpy(v_out + off, p.cache.values[l][hd].data.data(), sizeof(double) * n * d);
            }
        }
        return 0;
    });
}

int ref_cka(const double* oe, int ce, const double* oc, int cc, int n, double* out) {
    return guarded([&] {
        *out = cka(to_matrix(oe, n, ce), to_matrix(oc, n, cc));
        return 0;
    });
}

int ref_rsa(const double* oe, int ce, const double* oc, int cc, int n, double* out) {
    return guarded([&] {
        *out = rsa(to_matrix(oe, n, ce), to_matrix(oc, n, cc));
        return 0;
    });
}

int ref_match_layers(const double* edge_outs, int me, int ce, const double* cloud_outs, int nc,
                     int cc, int n, double theta_cka, double theta_rsa, double* cka_out,
                     double* rsa_out, int* best) {
    return guarded([&] {
        std::vector<Matrix> e, c;
        for (int l = 0; l < me; ++l) e.push_back(to_matrix(edge_outs + (std::size_t)l * n * ce, n, ce));
        for (int l = 0; l < nc; ++l) c.push_back(to_matrix(cloud_outs + (std::size_t)l * n * cc, n, cc));
        SimilarityConfig cfg;
        cfg.theta_cka = theta_cka;
        cfg.theta_rsa = theta_rsa;
        cfg.num_probe_samples = n;
        LayerMatchReport r = match_layers(e, c, cfg);
        std::memcpy(cka_out, r.cka.data.data(), sizeof(double) * me * nc);
        std::memcpy(rsa_out, r.rsa.data.data(), sizeof(double) * me * nc);
        for (int l = 0; l < me; ++l) best[l] = r.best[l].has_value() ? r.best[l].value() : -1;
        return 0;
    });
}

int ref_cache_source(int layer, double cost_local, double cost_peer, int boundary, int m) {
    return guarded([&] { return (int)cache_source(layer, cost_local, cost_peer, boundary, m); });
}

int ref_pipeline_schedule(const double* t_comm, const double* t_comp, int n, double* t_pip,
                          double* seq_total, double* pip_total) {
    return guarded([&] {
        std::vector<LayerTimes> lt(n);
        for (int i = 0; i < n; ++i) lt[i] = LayerTimes{t_comm[i], t_comp[i]};
        ScheduleTrace t = pipeline_schedule(lt);
        for (int i = 0; i < n; ++i) t_pip[i] = t.layers[i].t_pip;
        *seq_total = t.sequential_total;
        *pip_total = t.pipelined_total;
        return 0;
    });
}

// CPU baseline: the reference's own collaborative_decode (fp64, one session
// per thread) on an edge model of the given shape with random scaled weights
// (populating edgekv::Model directly) and a random
// S-row assembled context (layers < boundary local, the rest "cloud").
struct RefBench {
    Model model;
    AssembledContext ctx;
    int h = 0;
};

void* ref_bench_setup(int L, int H, int d, int S, int boundary, int max_pos, uint64_t seed) {
    try {
        auto* b = new RefBench();
        const int h = H * d;
        b->h = h;
        Model& m = b->model;
        m.config.num_layers = L;
        m.config.num_heads = H;
        m.config.head_dim = d;
        m.config.hidden_size = h;
        m.config.max_positions = max_pos;
        Rng rng(seed);
        const double a = std::sqrt(3.0 / (double)h);
        m.layers.resize(L);
        for (int l = 0; l < L; ++l) {
            m.layers[l].heads.resize(H);
            for (auto& w : m.layers[l].heads) {
                for (Matrix* p : {&w.wq, &w.wk, &w.wv}) {
                    *p = Matrix(h, d);
                    for (double& v : p->data) v = rng.uniform(-a, a);
                }
            }
            m.layers[l].out_proj = Matrix(h, h);
            for (double& v : m.layers[l].out_proj.data) v = rng.uniform(-a, a);
            m.layers[l].gamma.assign(h, 1.0);
            m.layers[l].bias.assign(h, 0.0);
        }
        m.pos_embedding = Matrix(max_pos, h);
        for (double& v : m.pos_embedding.data) v = rng.uniform(-0.1, 0.1);
        std::map<int, LayerKV> local, shared;
        std::map<int, CacheOrigin> origins;
        for (int l = 0; l < L; ++l) {
            LayerKV kv;
            for (int hd = 0; hd < H; ++hd) {
                Matrix k(S, d), v(S, d);
                for (double& x : k.data) x = rng.uniform(-1, 1);
                for (double& x : v.data) x = rng.uniform(-1, 1);
                kv.keys.push_back(std::move(k));
                kv.values.push_back(std::move(v));
            }
            if (l < boundary) {
                local[l] = std::move(kv);
            } else {
                shared[l] = std::move(kv);
                origins[l] = CacheOrigin::cloud;
            }
        }
        b->ctx = assemble_context(shared, local, origins, L);
        return b;
    } catch (const std::exception& e) {
        g_err = e.what();
        return nullptr;
    }
}

// `threads` sessions in parallel, each running `calls` collaborative_decode
// calls (U user rows + `steps` generated rows).  Reports wall seconds and the
// forward rows processed (each row = one token through every layer).
int ref_bench_run(void* handle, int U, int steps, int threads, int calls, double* seconds,
                  int64_t* rows) {
    return guarded([&] {
        auto* b = static_cast<RefBench*>(handle);
        Matrix user = generate_embeddings(7, U, b->h);
        std::atomic<int64_t> total{0};
        std::string err;
        const auto t0 = std::chrono::steady_clock::now();
        std::vector<std::thread> pool;
        for (int t = 0; t < threads; ++t)
            pool.emplace_back([&] {
                for (int c = 0; c < calls; ++c) {
                    CollaborativeResult r = collaborative_decode(b->model, b->ctx, user, steps);
                    total += (int64_t)(r.prefill_outputs.size() + r.step_outputs.size());
                }
            });
        for (auto& t : pool) t.join();
        *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        *rows = total.load();
        return 0;
    });
}

void ref_bench_free(void* handle) { delete static_cast<RefBench*>(handle); }

// The reference's whole CE-LSLM value path for one request, composed from its
// public API in the order of Artifacts (sim.cpp:100-265): probe prefill of both
// models -> match_layers -> deep map; context prefill of both models;
// build_deep_kv (x0, project_qkv of every distinct matched cloud layer and head,
// select_channels, prune_cache); assembled_context; collaborative_decode of the
// user prompt.  Models in the B200 layout (populated directly).
// times[8] (seconds): probe prefill, match, edge ctx prefill, cloud ctx prefill,
// Q/K restack (project_qkv), select_channels, prune + assemble, decode.
// kept_out[retained], deep_map_out[deep], step_out[steps][h_e] (may be null).
int ref_full_path(int Le, int He, int de, int Lc, int Hc, int dc, int max_pos, const double* e_wqkvT,
                  const double* e_woT, const double* e_gamma, const double* e_bias, const double* e_pos,
                  const double* c_wqkvT, const double* c_woT, const double* c_gamma, const double* c_bias,
                  const double* c_pos, uint64_t seed, int n_probe, double theta_cka, double theta_rsa,
                  int S, int deep, double lambda, int U, int steps, double* times, int* kept_out,
                  int* deep_map_out, double* step_out) {
    return guarded([&] {
        using clk = std::chrono::steady_clock;
        auto sec = [](clk::time_point a, clk::time_point b) {
            return std::chrono::duration<double>(b - a).count();
        };
        const Model edge = make_model(Le, He, de, max_pos, e_wqkvT, e_woT, e_gamma, e_bias, e_pos);
        const Model cloud = make_model(Lc, Hc, dc, max_pos, c_wqkvT, c_woT, c_gamma, c_bias, c_pos);
        const int he = He * de, hc = Hc * dc;
        auto t0 = clk::now();
        Matrix pe = generate_embeddings(Rng::mix(seed, 0x9B0BE), n_probe, he);
        Matrix pc = generate_embeddings(Rng::mix(seed, 0x9B0BE), n_probe, hc);
        std::vector<Matrix> eo = prefill(edge, pe).layer_outputs;
        std::vector<Matrix> co = prefill(cloud, pc).layer_outputs;
        auto t1 = clk::now();
        SimilarityConfig cfg;
        cfg.theta_cka = theta_cka;
        cfg.theta_rsa = theta_rsa;
        cfg.num_probe_samples = n_probe;
        LayerMatchReport rep = match_layers(eo, co, cfg);
        const int boundary = Le - deep;
        std::map<int, int> match;
        for (int l = boundary; l < Le; ++l) {
            if (!rep.best[l].has_value())
                throw std::invalid_argument("ce_lslm: edge layer " + std::to_string(l) +
                                            " has no matched cloud layer under the configured thresholds");
            match[l] = rep.best[l].value();
            if (deep_map_out) deep_map_out[l - boundary] = match[l];
        }
        auto t2 = clk::now();
        const std::uint64_t eseed = Rng::mix(seed, 0xC7E20000ull);
        Matrix emb_e = generate_embeddings(eseed, S, he);
        Matrix emb_c = generate_embeddings(eseed, S, hc);
        PrefillResult epf = prefill(edge, emb_e);
        auto t3 = clk::now();
        PrefillResult cpf = prefill(cloud, emb_c);
        auto t4 = clk::now();
        std::set<int> cls;
        for (const auto& [le, lc] : match) cls.insert(lc);
        Matrix x0((std::size_t)S, (std::size_t)hc);
        for (int i = 0; i < S; ++i)
            for (int c = 0; c < hc; ++c)
                x0(i, c) = cloud.layers[0].gamma[c] * (emb_c(i, c) + cloud.pos_embedding(i, c)) +
                           cloud.layers[0].bias[c];
        const std::size_t blocks = cls.size() * (std::size_t)Hc;
        Matrix q_stack(blocks * S, dc), k_stack(blocks * S, dc);
        std::size_t block = 0;
        for (int lc : cls) {
            const Matrix& input = lc == 0 ? x0 : cpf.layer_outputs[lc - 1];
            for (int h = 0; h < Hc; ++h) {
                QkvRows qkv = project_qkv(cloud, input, lc, h);
                for (int i = 0; i < S; ++i)
                    for (int c = 0; c < dc; ++c) {
                        q_stack(block * S + i, c) = qkv.q(i, c);
                        k_stack(block * S + i, c) = qkv.k(i, c);
                    }
                ++block;
            }
        }
        auto t5 = clk::now();
        const PruneSpec spec = PruneSpec::from_lambda(lambda, dc);
        const ChannelMask mask =
            spec.retained == dc ? ChannelMask::full(dc) : select_channels(q_stack, k_stack, spec);
        if (kept_out) std::copy(mask.kept.begin(), mask.kept.end(), kept_out);
        auto t6 = clk::now();
        const KVCache pruned = prune_cache(cpf.cache, mask);
        std::map<int, LayerKV> local, shared;
        std::map<int, CacheOrigin> origins;
        for (int l = 0; l < boundary; ++l) {
            LayerKV kv;
            kv.keys = epf.cache.keys[l];
            kv.values = epf.cache.values[l];
            local[l] = std::move(kv);
        }
        for (const auto& [le, lc] : match) {
            LayerKV kv;
            kv.keys = pruned.keys[lc];
            kv.values = pruned.values[lc];
            shared[le] = std::move(kv);
            origins[le] = CacheOrigin::cloud;
        }
        AssembledContext ctx = assemble_context(shared, local, origins, Le);
        auto t7 = clk::now();
        Matrix user = generate_embeddings(Rng::mix(seed, 0x55E20000ull), U, he);
        CollaborativeResult r = collaborative_decode(edge, ctx, user, steps);
        auto t8 = clk::now();
        if (step_out)
            for (int t = 0; t < steps; ++t) std::copy(r.step_outputs[t].begin(), r.step_outputs[t].end(),
                                                      step_out + (std::size_t)t * he);
        times[0] = sec(t0, t1);  // probe prefill
        times[1] = sec(t1, t2);  // match_layers
        times[2] = sec(t2, t3);  // edge context prefill
        times[3] = sec(t3, t4);  // cloud context prefill
        times[4] = sec(t4, t5);  // Q/K restack (project_qkv)
        times[5] = sec(t5, t6);  // select_channels
        times[6] = sec(t6, t7);  // prune + assemble
        times[7] = sec(t7, t8);  // collaborative_decode
        return 0;
    });
}

}  // extern "C"
