// Tests of the C++ mirror (include/edgekv_b200.hpp) written like the
// reference's own doctest suites (cache_merge_test.cpp, head_prune_test.cpp,
// layer_match_test.cpp, cost_model_test.cpp), with the reference's message
// substrings, checked against the C oracle (oracle/ekv_oracle.c, linked as
// test infrastructure).  Built and run by tests/test_gpu_cpp_mirror.py.
#include <cmath>
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <algorithm>
#include <functional>
#include <stdexcept>
#include <string>
#include <vector>

#include "edgekv_b200.hpp"

extern "C" {
// oracle/ekv_oracle.c (TEST INFRASTRUCTURE)
void ekvo_fill_uniform_bf16(uint64_t seed, uint64_t stream, int64_t n, double lo, double hi,
                            uint16_t* out);
void ekvo_generate_embeddings(uint64_t seed, int n, int h, double* out);
void ekvo_segment_attention(const double* q, const double* k, const double* v, int visible, int d,
                            int vd, double* o, double* sigma, double* shift);
int ekvo_collaborative_decode(int L, int H, int d, int max_pos, const double* wqkvT,
                              const double* woT, const double* gamma, const double* bias,
                              const double* pos, int S, const double* ctx_k_all,
                              const double* ctx_v_all, const double* user_emb, int U, int steps,
                              const double* teacher, int user_kv_bf16, double* prefill_out,
                              double* step_out);
void ekvo_select_channels(const double* q, int64_t q_rows, const double* k, int64_t k_rows, int d,
                          int retained, int* kept, double* score_out);
void ekvo_prefill_ex(int L, int H, int d, int max_pos, const double* wqkvT, const double* woT,
                     const double* gamma, const double* bias, const double* pos, const double* emb,
                     int n, int kv_bf16, double* layer_out, double* k_out, double* v_out);
}

using namespace edgekv;

static int g_fail = 0, g_checks = 0;
#define CHECK(cond)                                                                  \
    do {                                                                             \
        ++g_checks;                                                                  \
        if (!(cond)) {                                                               \
            ++g_fail;                                                                \
            std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #cond);              \
        }                                                                            \
    } while (0)
#define CHECK_THROWS_WITH(expr, substr)                                              \
    do {                                                                             \
        ++g_checks;                                                                  \
        bool ok = false;                                                             \
        try {                                                                        \
            expr;                                                                    \
        } catch (const std::exception& e) {                                          \
            ok = std::string(e.what()).find(substr) != std::string::npos;            \
            if (!ok) std::printf("  threw: %s\n", e.what());                         \
        }                                                                            \
        if (!ok) {                                                                   \
            ++g_fail;                                                                \
            std::printf("FAIL %s:%d: %s does not throw \"%s\"\n", __FILE__, __LINE__, \
                        #expr, substr);                                              \
        }                                                                            \
    } while (0)

static double bf16(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    std::memcpy(&f, &u, 4);
    return f;
}

static Matrix rand_matrix(uint64_t seed, uint64_t stream, size_t r, size_t c, double s = 1.0) {
    std::vector<uint16_t> b(r * c);
    ekvo_fill_uniform_bf16(seed, stream, (int64_t)b.size(), -s, s, b.data());
    Matrix m(r, c);
    for (size_t i = 0; i < b.size(); ++i) m.data[i] = bf16(b[i]);  // bf16-exact values
    return m;
}

static double normwise(const Vec& got, const std::vector<double>& want, size_t off = 0) {
    double e = 0, w = 0;
    for (size_t i = 0; i < got.size(); ++i) {
        e = std::max(e, std::abs(got[i] - want[off + i]));
        w = std::max(w, std::abs(want[off + i]));
    }
    return e / w;
}

// B200 weight layout of a mirror Model, exact fp64 (for the oracle)
static void b200_layout(const Model& m, std::vector<double>& wqkvT, std::vector<double>& woT,
                        std::vector<double>& gamma, std::vector<double>& bias) {
    const int L = m.config.num_layers, H = m.config.num_heads, d = m.config.head_dim,
              h = m.config.hidden_size;
    wqkvT.assign((size_t)L * 3 * h * h, 0.0);
    woT.assign((size_t)L * h * h, 0.0);
    for (int l = 0; l < L; ++l) {
        for (int hd = 0; hd < H; ++hd) {
            const HeadWeights& w = m.layers[l].heads[hd];
            const Matrix* parts[3] = {&w.wq, &w.wk, &w.wv};
            for (int p = 0; p < 3; ++p)
                for (int c = 0; c < d; ++c)
                    for (int k = 0; k < h; ++k)
                        wqkvT[((size_t)l * 3 * h + p * h + hd * d + c) * h + k] = (*parts[p])(k, c);
        }
        for (int j = 0; j < h; ++j)
            for (int i = 0; i < h; ++i) woT[((size_t)l * h + j) * h + i] = m.layers[l].out_proj(i, j);
    }
    gamma = m.layers[0].gamma;
    bias = m.layers[0].bias;
}

static Model make_model(int L, int H, int d, int max_pos, uint64_t seed) {
    Model m;
    m.config = ModelConfig{L, H, d, H * d, max_pos, seed};
    const int h = H * d;
    const double a = std::sqrt(3.0 / h);
    m.layers.resize(L);
    uint64_t s = 0;
    for (int l = 0; l < L; ++l) {
        for (int hd = 0; hd < H; ++hd) {
            HeadWeights w;
            w.wq = rand_matrix(seed, s++, h, d, a / std::sqrt((double)d));
            w.wk = rand_matrix(seed, s++, h, d, a);
            w.wv = rand_matrix(seed, s++, h, d, a);
            m.layers[l].heads.push_back(w);
        }
        m.layers[l].out_proj = rand_matrix(seed, s++, h, h, a);
        m.layers[l].gamma.assign(h, 1.0);
        m.layers[l].bias.assign(h, 0.0);
    }
    m.pos_embedding = rand_matrix(seed, s++, max_pos, h, 0.1);
    return m;
}

static void test_prune_spec_and_tie_break() {
    // head_prune_test.cpp:66-81, 160-167
    CHECK(PruneSpec::from_lambda(0.2, 80).retained == 64);
    CHECK(PruneSpec::from_lambda(1.0 / 3.0, 6).retained == 4);
    CHECK(PruneSpec::from_lambda(0.5, 7).retained == 3);
    CHECK_THROWS_WITH(PruneSpec::from_lambda(-0.1, 4), "lambda outside");
    PruneSpec bad;
    bad.lambda = 0.5;
    bad.head_dim = 6;
    bad.retained = 4;
    CHECK_THROWS_WITH(bad.validate(), "floor");
    Matrix q(2, 3), k(2, 3);
    q.data = {1, 1, 1, 0, 0, 0};
    k.data = {1, 1, 1, 0, 0, 0};
    ChannelMask m = select_channels(q, k, PruneSpec::from_lambda(1.0 / 3.0, 3));
    CHECK((m.kept == std::vector<int>{0, 1}));
}

static void test_select_channels_matches_reference_rule() {
    // heterogeneous channel scales: a clear cut, so bf16 inputs decide it like fp64
    const int d = 64, rows = 512;
    Matrix q = rand_matrix(3, 1, rows, d), k = rand_matrix(3, 2, rows, d);
    for (size_t i = 0; i < (size_t)rows; ++i)
        for (int c = 0; c < d; ++c) {
            const double s = (c % 2) ? 4.0 : 1.0;
            q(i, c) *= s;
        }
    const PruneSpec spec = PruneSpec::from_lambda(0.5, d);
    ChannelMask got = select_channels(q, k, spec);
    std::vector<int> want(spec.retained);
    ekvo_select_channels(q.data.data(), rows, k.data.data(), rows, d, spec.retained, want.data(), nullptr);
    CHECK(got.kept == want);
}

static void test_prune_cache_is_an_exact_slice() {
    // head_prune_test.cpp:225-258
    KVCache c = KVCache::empty_for(2, 2, 6);
    for (int l = 0; l < 2; ++l)
        for (int h = 0; h < 2; ++h) {
            c.keys[l][h] = rand_matrix(l, h, 4, 6);
            c.values[l][h] = rand_matrix(l, 10 + h, 4, 6);
            c.keys[l][h](1, 3) = 0.1234567891234;  // not bf16-representable: must survive
        }
    for (int p = 0; p < 4; ++p) c.positions.push_back(PositionTag{PositionKind::context, p});
    ChannelMask mask;
    mask.head_dim = 6;
    mask.kept = {0, 2, 3, 5};
    KVCache out = prune_cache(c, mask);
    CHECK(out.head_dim == 4 && out.keys[1][1].cols == 4);
    CHECK(out.positions.size() == c.positions.size());
    CHECK(out.keys[0][0](2, 1) == c.keys[0][0](2, 2));
    CHECK(out.keys[1][0](1, 2) == 0.1234567891234);
    bool exact = true;
    for (int l = 0; l < 2; ++l)
        for (int h = 0; h < 2; ++h)
            for (size_t i = 0; i < 4; ++i)
                for (size_t j = 0; j < 4; ++j)
                    exact &= out.values[l][h](i, j) == c.values[l][h](i, mask.kept[j]);
    CHECK(exact);
    ChannelMask wrong;
    wrong.head_dim = 5;
    wrong.kept = {0, 1};
    CHECK_THROWS_WITH(prune_cache(c, wrong), "mask dim");
}

static void test_segment_attention_and_merge() {
    // cache_merge_test.cpp:147-200 at the B200 head dims
    const int d = 64;
    Matrix k = rand_matrix(9, 1, 40, d), v = rand_matrix(9, 2, 40, d);
    Vec q(d);
    {
        Matrix qq = rand_matrix(9, 3, 1, d, 0.3);
        q.assign(qq.data.begin(), qq.data.end());
    }
    Matrix kc(25, d), vc(25, d), ku(15, d), vu(15, d);
    std::copy(k.data.begin(), k.data.begin() + 25 * d, kc.data.begin());
    std::copy(v.data.begin(), v.data.begin() + 25 * d, vc.data.begin());
    std::copy(k.data.begin() + 25 * d, k.data.end(), ku.data.begin());
    std::copy(v.data.begin() + 25 * d, v.data.end(), vu.data.begin());
    MergedAttention m = merge_attention(segment_attention(q, kc, vc), segment_attention(q, ku, vu));
    std::vector<double> want(d);
    double s, sh;
    ekvo_segment_attention(q.data(), k.data.data(), v.data.data(), 40, d, d, want.data(), &s, &sh);
    CHECK(normwise(m.o, want) <= 1e-3);
    CHECK(std::abs(m.weights.alpha_ctx + m.weights.alpha_user - 1.0) < 1e-12);
    SegmentAttention one = segment_attention(q, kc, vc);
    double so, sho;
    std::vector<double> wc(d);
    ekvo_segment_attention(q.data(), kc.data.data(), vc.data.data(), 25, d, d, wc.data(), &so, &sho);
    CHECK(std::abs(one.sigma_raw() - so * std::exp(sho)) / (so * std::exp(sho)) < 1e-4);
    Matrix empty(0, d);
    CHECK_THROWS_WITH(segment_attention(q, empty, empty), "empty segment");
    SegmentAttention a, b;
    a.o = {1.0, 2.0};
    a.sigma = 0.0;
    b.o = {1.0, 2.0};
    b.sigma = 1.0;
    CHECK_THROWS_WITH(merge_attention(a, b), "non-positive or non-finite sigma");
}

// matrix_test.cpp:21-27: the reference's own triple loop (no FMA at -O2 x86-64)
static Matrix naive_matmul(const Matrix& a, const Matrix& b) {
    Matrix out(a.rows, b.cols);
    for (size_t i = 0; i < a.rows; ++i)
        for (size_t j = 0; j < b.cols; ++j) {
            double acc = 0.0;
            for (size_t k = 0; k < a.cols; ++k) acc += a(i, k) * b(k, j);
            out(i, j) = acc;
        }
    return out;
}

static void test_project_qkv_bit_exact() {
    // transformer.cpp:133-152 on the device in fp64: identical bits, any input values
    Model m = make_model(2, 4, 32, 16, 5);
    Matrix x(37, 128);
    ekvo_generate_embeddings(77, 37, 128, x.data.data());  // full fp64, not bf16-representable
    QkvRows r = project_qkv(m, x, 1, 2);
    const HeadWeights& w = m.layers[1].heads[2];
    CHECK(r.q.data == naive_matmul(x, w.wq).data);
    CHECK(r.k.data == naive_matmul(x, w.wk).data);
    CHECK(r.v.data == naive_matmul(x, w.wv).data);
    CHECK_THROWS_WITH(project_qkv(m, x, 2, 0), "layer 2 out of range");
    CHECK_THROWS_WITH(project_qkv(m, x, 0, 4), "head 4 out of range");
    CHECK_THROWS_WITH(project_qkv(m, Matrix(3, 5), 0, 0), "expected hidden_size 128");
}

static void test_segment_attention_fp64_pair() {
    // the reference's (o, sigma, shift) triple in fp64 (cache_merge.cpp:12-38)
    const int d = 48, n = 300;
    Matrix k(n, d), v(n, d);
    ekvo_generate_embeddings(91, n, d, k.data.data());
    ekvo_generate_embeddings(92, n, d, v.data.data());
    Vec q(d);
    ekvo_generate_embeddings(93, 1, d, q.data());
    for (double& x : q) x *= 3.0;  // hot logits: the max shift matters
    SegmentAttention a = segment_attention(q, k, v);
    std::vector<double> o(d);
    double sg, sh;
    ekvo_segment_attention(q.data(), k.data.data(), v.data.data(), n, d, d, o.data(), &sg, &sh);
    CHECK(a.shift == sh);  // the max logit: bit-identical
    CHECK(std::abs(a.sigma - sg) <= 1e-13 * sg);
    CHECK(normwise(a.o, o) <= 1e-13);
}

static void test_select_channels_fp64_inputs() {
    // full-precision Q/K (not bf16-representable) with a small but clear cut: the
    // fp64 device norms give the reference's mask
    const int d = 32, rows = 400;
    Matrix q(rows, d), k(rows, d);
    ekvo_generate_embeddings(101, rows, d, q.data.data());
    ekvo_generate_embeddings(102, rows, d, k.data.data());
    for (int i = 0; i < rows; ++i)
        for (int c = 0; c < d; ++c) q(i, c) *= 1.0 + 1e-4 * c;  // ~1e-4 score steps
    const PruneSpec spec = PruneSpec::from_lambda(0.5, d);
    std::vector<int> want(spec.retained);
    ekvo_select_channels(q.data.data(), rows, k.data.data(), rows, d, spec.retained, want.data(), nullptr);
    CHECK(select_channels(q, k, spec).kept == want);
}

static void test_prefill_and_forward_rows() {
    // forward_rows / prefill on the device vs the oracle (KV rows stored as bf16)
    const int L = 3, H = 8, d = 32, h = H * d, n = 12, mp = 64;
    Model m = make_model(L, H, d, mp, 31);
    for (int c = 0; c < h; ++c) {
        m.layers[0].gamma[c] = 1.0 + 0.01 * (c % 7);
        m.layers[0].bias[c] = 0.02 * ((c % 5) - 2);
    }
    Matrix emb(n, h);
    ekvo_generate_embeddings(33, n, h, emb.data.data());
    for (double& x : emb.data) x = (double)(float)x;
    FlopCounts fc;
    PrefillResult pr = prefill(m, emb, &fc);
    CHECK((int)pr.layer_outputs.size() == L && pr.cache.size() == n);
    CHECK((int)pr.cache.keys[2][3].rows == n);
    std::vector<double> w, wo, g, b, lo((size_t)L * n * h), ko((size_t)L * H * n * d), vo(ko.size());
    b200_layout(m, w, wo, g, b);
    ekvo_prefill_ex(L, H, d, mp, w.data(), wo.data(), g.data(), b.data(), m.pos_embedding.data.data(),
                    emb.data.data(), n, 1, lo.data(), ko.data(), vo.data());
    double worst = 0;
    for (int l = 0; l < L; ++l)
        for (int i = 0; i < n; ++i)
            worst = std::max(worst, normwise(pr.layer_outputs[l].row(i), lo, ((size_t)l * n + i) * h));
    std::printf("  prefill normwise error vs oracle: %.3e\n", worst);
    CHECK(worst <= 1e-3);
    // flop counts: the reference's closed form (transformer_test.cpp:251-281)
    CHECK(fc.proj == 3ll * n * h + (int64_t)L * n * H * 3 * d * (2ll * h - 1));
    CHECK(fc.out_proj == (int64_t)L * n * h * (2ll * h - 1));
    // incremental == monolithic: 8 rows, then 4 more on top of the cache
    Matrix a(8, h), c(4, h);
    std::copy(emb.data.begin(), emb.data.begin() + 8 * h, a.data.begin());
    std::copy(emb.data.begin() + 8 * h, emb.data.end(), c.data.begin());
    PrefillResult inc = prefill(m, a);
    std::vector<Matrix> more = forward_rows(m, inc.cache, c, PositionKind::user, nullptr);
    CHECK(inc.cache.size() == n && inc.cache.positions.back().kind == PositionKind::user);
    double dev = 0;
    for (int l = 0; l < L; ++l)
        for (int i = 0; i < 4; ++i)
            dev = std::max(dev, normwise(more[l].row(i), pr.layer_outputs[l].data, (size_t)(8 + i) * h));
    std::printf("  incremental vs monolithic prefill: %.3e\n", dev);
    CHECK(dev <= 1e-4);
    Vec last = decode_step(m, inc.cache, emb.row(0));
    CHECK((int)last.size() == h && inc.cache.size() == n + 1);
    CHECK_THROWS_WITH(decode_step(m, inc.cache, Vec(3)), "embedding size 3");
    KVCache wrong = KVCache::empty_for(L, H, d + 1);
    CHECK_THROWS_WITH(forward_rows(m, wrong, emb, PositionKind::context, nullptr), "cache shape");
    Matrix big(mp + 1, h);
    CHECK_THROWS_WITH(prefill(m, big), "position overflow");
}

static void test_build_deep_kv_on_tensor_cores() {
    // Artifacts::build_deep_kv (sim.cpp:217-265) with K1: the mask equals the
    // reference rule on the (bf16) inputs the tensor cores consumed; deep_kv is the
    // exact pruned cloud KV
    const int L = 4, H = 4, d = 64, h = H * d, S = 128, mp = 160;
    Model cloud = make_model(L, H, d, mp, 41);
    for (int l = 0; l < L; ++l)  // heterogeneous channel importance: a decidable cut
        for (int hd = 0; hd < H; ++hd)
            for (int r = 0; r < h; ++r)
                for (int c = 0; c < d; ++c) cloud.layers[l].heads[hd].wq(r, c) *= std::exp(0.03 * ((c * 37) % d) - 1.0);
    Matrix emb(S, h);
    ekvo_generate_embeddings(43, S, h, emb.data.data());
    PrefillResult pre = prefill(cloud, emb);
    const std::map<int, int> match = {{2, 0}, {3, 3}};
    const PruneSpec spec = PruneSpec::from_lambda(0.5, d);
    b200::DeepKV dk = b200::build_deep_kv(cloud, pre, emb, match, spec);
    CHECK((int)dk.mask.kept.size() == spec.retained && dk.cut_margin > 1e-6);
    // the reference rule on the same bf16-rounded X, W_Q and K
    auto r16 = [](double x) {
        float f = (float)x;
        uint32_t u;
        std::memcpy(&u, &f, 4);
        u += 0x7FFFu + ((u >> 16) & 1u);
        u &= 0xFFFF0000u;
        std::memcpy(&f, &u, 4);
        return (double)f;
    };
    std::vector<double> qs, ks;
    for (int lc : {0, 3}) {
        Matrix x(S, h);
        for (int r = 0; r < S; ++r)
            for (int c = 0; c < h; ++c)
                x(r, c) = r16(lc == 0 ? cloud.layers[0].gamma[c] * (emb(r, c) + cloud.pos_embedding(r, c)) +
                                            cloud.layers[0].bias[c]
                                      : pre.layer_outputs[lc - 1](r, c));
        for (int hd = 0; hd < H; ++hd) {
            Matrix wq = cloud.layers[lc].heads[hd].wq;
            for (double& v : wq.data) v = r16(v);
            Matrix q = naive_matmul(x, wq);
            qs.insert(qs.end(), q.data.begin(), q.data.end());
            for (double v : pre.cache.keys[lc][hd].data) ks.push_back(r16(v));
        }
    }
    std::vector<int> want(spec.retained);
    ekvo_select_channels(qs.data(), (int64_t)qs.size() / d, ks.data(), (int64_t)ks.size() / d, d,
                         spec.retained, want.data(), nullptr);
    CHECK(dk.mask.kept == want);
    bool exact = dk.deep_kv.size() == 2;
    for (const auto& [le, lc] : match)
        for (int hd = 0; hd < H; ++hd)
            for (int r = 0; r < S; ++r)
                for (int j = 0; j < spec.retained; ++j) {
                    exact &= dk.deep_kv.at(le).keys[hd](r, j) == pre.cache.keys[lc][hd](r, want[j]);
                    exact &= dk.deep_kv.at(le).values[hd](r, j) == pre.cache.values[lc][hd](r, want[j]);
                }
    CHECK(exact);
    b200::DeepKV full = b200::build_deep_kv(cloud, pre, emb, match, PruneSpec::from_lambda(0.0, d));
    CHECK((int)full.mask.kept.size() == d);
}

static void test_assemble_context_errors() {
    // cache_merge_test.cpp:224-271
    auto lkv = [](int S, int d) {
        LayerKV kv;
        for (int h = 0; h < 2; ++h) {
            kv.keys.push_back(Matrix(S, d));
            kv.values.push_back(Matrix(S, d));
        }
        return kv;
    };
    std::map<int, LayerKV> local, shared;
    for (int l : {0, 1, 2}) local[l] = lkv(5, 3);
    CHECK_THROWS_WITH(assemble_context(shared, local, {}, 4), "missing layer 3");
    local[3] = lkv(5, 3);
    shared[2] = lkv(5, 3);
    CHECK_THROWS_WITH(assemble_context(shared, local), "duplicate layer 2");
    shared.clear();
    local[1].keys[0] = Matrix(5, 2);
    CHECK_THROWS_WITH(assemble_context(shared, local), "layer 1");
    local[1] = lkv(5, 3);
    for (int l : {2, 3}) {
        shared[l] = local[l];
        local.erase(l);
    }
    AssembledContext ctx = assemble_context(shared, local);
    CHECK(ctx.provenance[0] == CacheOrigin::local && ctx.provenance[3] == CacheOrigin::cloud);
    CHECK(ctx.cache.size() == 5);
}

static void test_collaborative_decode_matches_oracle() {
    const int L = 3, H = 4, d = 64, h = H * d, S = 256, U = 5, T = 4, mp = 512;
    Model m = make_model(L, H, d, mp, 21);
    std::map<int, LayerKV> local, shared;
    std::vector<double> ck((size_t)L * H * S * d), cv(ck.size());
    for (int l = 0; l < L; ++l) {
        LayerKV kv;
        for (int hd = 0; hd < H; ++hd) {
            kv.keys.push_back(rand_matrix(50 + l, hd, S, d));
            kv.values.push_back(rand_matrix(60 + l, hd, S, d));
            std::copy(kv.keys.back().data.begin(), kv.keys.back().data.end(),
                      ck.begin() + ((size_t)l * H + hd) * S * d);
            std::copy(kv.values.back().data.begin(), kv.values.back().data.end(),
                      cv.begin() + ((size_t)l * H + hd) * S * d);
        }
        (l < 2 ? local : shared)[l] = kv;
    }
    AssembledContext ctx = assemble_context(shared, local, {}, L);
    Matrix user(U, h);
    ekvo_generate_embeddings(43, U, h, user.data.data());
    for (double& x : user.data) x = (double)(float)x;  // what crosses the ABI
    CollaborativeResult r = collaborative_decode(m, ctx, user, T);
    CHECK((int)r.prefill_outputs.size() == U && (int)r.step_outputs.size() == T);
    std::vector<double> w, wo, g, b, teacher((size_t)T * h), pre((size_t)U * h), st((size_t)T * h),
        pos(m.pos_embedding.data);
    b200_layout(m, w, wo, g, b);
    for (int i = 0; i < h; ++i) teacher[i] = r.prefill_outputs.back()[i];
    for (int t = 1; t < T; ++t)
        for (int i = 0; i < h; ++i) teacher[(size_t)t * h + i] = r.step_outputs[t - 1][i];
    ekvo_collaborative_decode(L, H, d, mp, w.data(), wo.data(), g.data(), b.data(), pos.data(), S,
                              ck.data(), cv.data(), user.data.data(), U, T, teacher.data(), 1,
                              pre.data(), st.data());
    double worst = 0;
    for (int i = 0; i < U; ++i) worst = std::max(worst, normwise(r.prefill_outputs[i], pre, (size_t)i * h));
    for (int t = 0; t < T; ++t) worst = std::max(worst, normwise(r.step_outputs[t], st, (size_t)t * h));
    std::printf("  collaborative_decode normwise error vs oracle: %.3e\n", worst);
    CHECK(worst <= 1e-3);
    // two consumers of one context agree exactly (cache_merge_test.cpp:328-348)
    CollaborativeResult r2 = collaborative_decode(m, ctx, user, T);
    CHECK(r2.step_outputs == r.step_outputs);
    // errors (cache_merge_test.cpp:350-368, transformer "position overflow")
    CHECK_THROWS_WITH(collaborative_decode(m, ctx, user, 0), "steps must be >= 1");
    Model small = make_model(L, H, d, S + 2, 7);
    CHECK_THROWS_WITH(collaborative_decode(small, ctx, user, T), "position overflow");
    AssembledContext wrong;
    wrong.cache = KVCache::empty_for(L, H, 32);
    wrong.cache.positions.push_back(PositionTag{PositionKind::context, 0});
    CHECK_THROWS_WITH(collaborative_decode(m, wrong, user, 1), "align with head pruning");
}

static void test_compress_round_trip() {
    KVCache c = KVCache::empty_for(1, 2, 128);
    for (int h = 0; h < 2; ++h) {
        c.keys[0][h] = rand_matrix(70, h, 64, 128, 2.0);
        c.values[0][h] = rand_matrix(71, h, 64, 128, 2.0);
    }
    for (int p = 0; p < 64; ++p) c.positions.push_back(PositionTag{PositionKind::context, p});
    ChannelMask mask;
    mask.head_dim = 128;
    for (int i = 0; i < 128; i += 2) mask.kept.push_back(i);
    for (int bits : {8, 4}) {
        auto q = b200::compress_cache(c, mask, bits);
        LayerKV back = b200::dequantize(q[0], 2);
        double worst = 0;
        for (int h = 0; h < 2; ++h)
            for (int i = 0; i < 64; ++i)
                for (int j = 0; j < 64; ++j) {
                    const double s = q[0].k_scales[((size_t)h * 64 + i) * (64 / q[0].group) + j / q[0].group];
                    worst = std::max(worst, std::abs(back.keys[h](i, j) - c.keys[0][h](i, mask.kept[j])) / s);
                }
        CHECK(worst <= 0.5 + 128 * std::ldexp(1.0, -23));
    }
}

static void test_layer_match_and_scheduler() {
    // layer_match_test.cpp:249-272 (self match is the identity map), cost_model_test.cpp:92-114
    std::vector<Matrix> outs;
    for (int l = 0; l < 4; ++l) outs.push_back(rand_matrix(80, l, 24, 16));
    SimilarityConfig cfg;
    cfg.theta_cka = 0.5;
    cfg.theta_rsa = 0.0;
    cfg.num_probe_samples = 24;
    LayerMatchReport r = match_layers(outs, outs, cfg);
    bool diag = r.matches.size() == 4;
    for (int l = 0; l < 4; ++l) diag &= r.best[l].has_value() && *r.best[l] == l && std::abs(r.cka(l, l) - 1) < 1e-12;
    CHECK(diag);
    CHECK(cache_source(5, 0.1, 99.0, 4, 6) == CacheSource::cloud);
    CHECK(cache_source(2, 3.0, 2.0, 4, 6) == CacheSource::peer);
    CHECK(cache_source(1, 2.0, 2.0, 4, 6) == CacheSource::local);
    CHECK_THROWS_WITH(cache_source(0, 1, 1, 4, 6), "outside 1..6");
    ScheduleTrace t = pipeline_schedule({{2, 3}, {1, 2}, {4, 5}});
    CHECK(t.layers[1].t_pip == 3.0 && t.pipelined_total == 14.0 && t.sequential_total == 17.0);
}

int main() {
    std::vector<std::pair<const char*, std::function<void()>>> tests = {
        {"prune spec and tie break", test_prune_spec_and_tie_break},
        {"select_channels == reference rule", test_select_channels_matches_reference_rule},
        {"prune_cache exact slice", test_prune_cache_is_an_exact_slice},
        {"segment attention + Eq. 5 merge", test_segment_attention_and_merge},
        {"assemble_context errors", test_assemble_context_errors},
        {"collaborative_decode vs oracle", test_collaborative_decode_matches_oracle},
        {"compress round trip", test_compress_round_trip},
        {"layer match + scheduler", test_layer_match_and_scheduler},
        {"project_qkv bit-exact", test_project_qkv_bit_exact},
        {"segment_attention fp64 (o, sigma, shift)", test_segment_attention_fp64_pair},
        {"select_channels fp64 inputs", test_select_channels_fp64_inputs},
        {"prefill / forward_rows / decode_step", test_prefill_and_forward_rows},
        {"b200::build_deep_kv (K1)", test_build_deep_kv_on_tensor_cores},
    };
    for (auto& [name, fn] : tests) {
        const int before = g_fail;
        try {
            fn();
        } catch (const std::exception& e) {
            ++g_fail;
            std::printf("FAIL %s: exception %s\n", name, e.what());
        }
        std::printf("%s  %s\n", g_fail == before ? "PASS" : "FAIL", name);
    }
    std::printf("%d checks, %d failures\n", g_checks, g_fail);
    return g_fail ? 1 : 0;
}
