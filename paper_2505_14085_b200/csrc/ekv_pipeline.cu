// C-ABI entry points of stage 1+2 as whole reference operations (include/ekv_capi.h):
//
//   ekv_prefill        prefill / forward_rows on the device (transformer.cpp:175-251):
//                      per-layer outputs and the KV cache of n rows;
//   ekv_deep_match     Artifacts::deep_match (sim.cpp:100-122): probe prefill of both
//                      models + K7 layer map + the deep-layer map and its error;
//   ekv_match_layers   match_layers (layer_match.cpp:166-228) from host buffers, on K7;
//   ekv_build_deep_kv  Artifacts::build_deep_kv (sim.cpp:217-265): K1 (tcgen05 Q
//                      projection of every distinct matched cloud layer with the K
//                      column norms fused) -> device ranking -> one batched K3 launch
//                      straight into the assembled context's deep layers.  One
//                      stream, no host round trip between the stages.
#include <algorithm>
#include <cmath>
#include <memory>
#include <numeric>
#include <random>
#include <string>
#include <vector>

#include "ekv_objects.h"

using namespace ekv;

namespace {

// ctx-owned scratch (grown on demand, synchronising only when it grows)
void* ctx_scratch(ekv_ctx_s* c, size_t bytes) {
    if (bytes > c->scratch_n) {
        EKV_CUDA(cudaStreamSynchronize(c->stream));
        if (c->scratch) cudaFree(c->scratch);
        c->scratch = nullptr;
        c->scratch_n = 0;
        c->scratch = dalloc<uint8_t>(bytes);
        c->scratch_n = bytes;
    }
    return c->scratch;
}

void rethrow(int rc) {
    if (rc != EKV_OK) throw Error(rc, g_err);
}

// device buffer of one call, stream-ordered on the context stream (pooled)
struct DevMem {
    void* p = nullptr;
    cudaStream_t st;
    DevMem(size_t bytes, cudaStream_t s) : st(s) { p = dalloc_on<uint8_t>(bytes, s); }
    ~DevMem() { cudaFreeAsync(p, st); }
    template <class T>
    T* as() const { return (T*)p; }
};

// forward_rows: n new rows on top of the cached rows of `cached` (null = an empty
// cache, i.e. prefill) through a transient session: the new rows attend to every
// cached row and causally to each other -- the same algebra as the reference's
// single softmax over [cache | new rows] (Eq. 5 merge, cache_merge.cpp:59-80).
void device_prefill(ekv_model_s* m, const float* emb, int n, float* layer_out, float* x0, void* k_out,
                    void* v_out, ekv_kvctx_s* cached = nullptr) {
    ekv_ctx_s* c = m->ctx;
    cudaStream_t st = c->stream;
    const int L = m->cfg.num_layers, h = m->h;
    ekv_kvctx_t kv = cached;
    std::unique_ptr<ekv_kvctx_s, int (*)(ekv_kvctx_t)> kvg(nullptr, ekv_kvctx_destroy);
    if (!kv) {
        std::vector<int> fmt(L, EKV_KV_BF16);
        rethrow(ekv_kvctx_create(m, 0, fmt.data(), m->cfg.head_dim, &kv));
        kvg.reset(kv);
    }
    ekv_session_t s = nullptr;
    rethrow(ekv_session_create(m, kv, n, &s));
    std::unique_ptr<ekv_session_s, int (*)(ekv_session_t)> sg(s, ekv_session_destroy);
    check_overflow(s, n);
    DevMem scratch(sizeof(float) * 2 * (size_t)n * h, st);
    if (x0) launch_input_transform(emb, m->gamma, m->bias, m->pos, kv->S, n, h, x0, st);
    forward_layer_major(s, emb, n, 0, st, nullptr, scratch.as<float>(), nullptr, layer_out);
    const size_t kv_bytes = sizeof(uint16_t) * (size_t)L * s->ukv_layer();  // cap == n
    if (k_out) EKV_CUDA(cudaMemcpyAsync(k_out, s->uk, kv_bytes, cudaMemcpyDeviceToDevice, st));
    if (v_out) EKV_CUDA(cudaMemcpyAsync(v_out, s->uv, kv_bytes, cudaMemcpyDeviceToDevice, st));
    EKV_CUDA(cudaStreamSynchronize(st));
}

// select_channels over the stacked Q/K rows of the matched cloud layers
// (sim.cpp:236-256): K1 (tcgen05 Q projection, column sums folded over heads and
// layers; the cached-K column sums fused) -> the reference ranking on the device.
// kept (device, ctx scratch) holds `retained` channels, margin the cut margin.
void align_select(ekv_ctx_s* c, const ekv_cloud_kv& cl, int retained, int** kept_out,
                  double** margin_out) {
    const int d_c = cl.d_c, S = cl.S, h_c = cl.H * cl.d_c;
    cudaStream_t st = c->stream;
    uint8_t* sc = (uint8_t*)ctx_scratch(c, sizeof(double) * (2 * d_c + 1) + sizeof(int) * d_c);
    double* qsq = (double*)sc;
    double* ksq = qsq + d_c;
    double* margin = ksq + d_c;
    int* kept = (int*)(margin + 1);
    *kept_out = kept;
    *margin_out = margin;
    if (retained == d_c) {  // ChannelMask::full (sim.cpp:255-256)
        std::vector<int> all(d_c);
        std::iota(all.begin(), all.end(), 0);
        const double inf = INFINITY;
        EKV_CUDA(cudaMemcpyAsync(kept, all.data(), sizeof(int) * d_c, cudaMemcpyHostToDevice, st));
        EKV_CUDA(cudaMemcpyAsync(margin, &inf, sizeof(double), cudaMemcpyHostToDevice, st));
        EKV_CUDA(cudaStreamSynchronize(st));  // pageable sources
        return;
    }
    require(retained >= 1, "select_channels: lambda prunes every channel");
    EKV_CUDA(cudaMemsetAsync(qsq, 0, sizeof(double) * 2 * d_c, st));
    AlignLaunch p{};
    p.X = cl.x;
    p.x_stride = cl.x_stride;
    p.x_index = cl.x_index;
    p.WqT = cl.wq;
    p.w_stride = cl.wq_stride;
    p.w_index = cl.wq_index;
    p.m = cl.m;
    p.S = S;
    p.h_c = h_c;
    p.n_cols = h_c;
    p.fold = d_c;
    p.colsq = qsq;
    p.kcolsq = ksq;
    p.k = cl.k;
    p.k_layers = cl.m;
    p.k_rows = (int64_t)cl.H * S;
    p.d_c = d_c;
    launch_align(p, st);
    launch_rank_channels(qsq, ksq, d_c, retained, kept, margin, st);
}

void fetch_mask(ekv_ctx_s* c, int retained, const int* kept, const double* margin, int* kept_host,
                double* margin_host) {
    std::vector<int> kv(retained);
    double mg = INFINITY;
    EKV_CUDA(cudaMemcpyAsync(kv.data(), kept, sizeof(int) * retained, cudaMemcpyDeviceToHost, c->stream));
    EKV_CUDA(cudaMemcpyAsync(&mg, margin, sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    EKV_CUDA(cudaStreamSynchronize(c->stream));
    if (kept_host) std::copy(kv.begin(), kv.end(), kept_host);
    if (margin_host) *margin_host = mg;
}

}  // namespace

extern "C" {

int ekv_prefill(ekv_model_t m, const float* emb_dev, int n, float* layer_out_dev, float* x0_dev,
                void* k_dev, void* v_dev) {
    return guard([&] {
        require(m && emb_dev, "ekv_prefill: null argument");
        require(n >= 1, "ekv_prefill: n must be >= 1");
        set_dev(m->ctx);
        device_prefill(m, emb_dev, n, layer_out_dev, x0_dev, k_dev, v_dev);
    });
}

int ekv_forward_rows(ekv_model_t m, ekv_kvctx_t cached, const float* emb_dev, int n, float* layer_out_dev,
                     float* x0_dev, void* k_dev, void* v_dev) {
    return guard([&] {
        require(m && emb_dev, "ekv_forward_rows: null argument");
        require(n >= 1, "ekv_forward_rows: n must be >= 1");
        set_dev(m->ctx);
        device_prefill(m, emb_dev, n, layer_out_dev, x0_dev, k_dev, v_dev, cached);
    });
}

int ekv_matmul_f64(ekv_ctx_t c, const double* a, const double* b, int n, int k, int m, double* out) {
    return guard([&] {
        require(c && a && b && out, "ekv_matmul_f64: null argument");
        require(n >= 0 && k >= 0 && m >= 0, "matmul: dimension mismatch");
        set_dev(c);
        launch_matmul_f64(a, b, n, k, m, out, c->stream);
    });
}

int ekv_segment_attention_f64(ekv_ctx_t c, const double* q, const double* k, const double* v, int n,
                              int d, int vd, double* o, double* sigma, double* shift) {
    return guard([&] {
        require(c && q && k && v && o && sigma && shift, "ekv_segment_attention_f64: null argument");
        require(n >= 1, "segment_attention: empty segment");
        require(d >= 1 && vd >= 1, "segment_attention: empty head");
        set_dev(c);
        double* sc = (double*)ctx_scratch(c, sizeof(double) * ((size_t)n + 2));
        launch_segment_attention_f64(q, k, v, n, d, vd, sc + 2, o, sc, c->stream);
        double st2[2];
        EKV_CUDA(cudaMemcpyAsync(st2, sc, sizeof(st2), cudaMemcpyDeviceToHost, c->stream));
        EKV_CUDA(cudaStreamSynchronize(c->stream));
        *sigma = st2[0];
        *shift = st2[1];
    });
}

int ekv_match_layers(ekv_ctx_t c, const double* edge_outs, int me, int ce, const double* cloud_outs,
                     int nc, int cc, int n, double theta_cka, double theta_rsa, double* cka,
                     double* rsa, int* best) {
    return guard([&] {
        require(c && edge_outs && cloud_outs && cka && rsa && best, "null argument");
        require(me >= 1 && nc >= 1, "match_layers: empty layer output list");
        require(n >= 1 && ce >= 1 && cc >= 1, "match_layers: bad layer width");
        set_dev(c);
        const size_t ne = (size_t)me * n * ce, ncl = (size_t)nc * n * cc;
        DevMem d(sizeof(double) * (ne + ncl), c->stream);
        EKV_CUDA(cudaMemcpyAsync(d.as<double>(), edge_outs, sizeof(double) * ne, cudaMemcpyHostToDevice,
                                 c->stream));
        EKV_CUDA(cudaMemcpyAsync(d.as<double>() + ne, cloud_outs, sizeof(double) * ncl,
                                 cudaMemcpyHostToDevice, c->stream));
        rethrow(ekv_match_layers_dev(c, d.as<double>(), me, ce, d.as<double>() + ne, nc, cc, n,
                                     theta_cka, theta_rsa, cka, rsa, best));
    });
}

int ekv_deep_match(ekv_model_t edge, ekv_model_t cloud, const float* edge_probe, const float* cloud_probe,
                   int n, int deep_layers, double theta_cka, double theta_rsa, int* deep_map,
                   double* cka, double* rsa, int* best) {
    return guard([&] {
        require(edge && cloud && edge_probe && cloud_probe && deep_map, "ekv_deep_match: null argument");
        require(edge->ctx == cloud->ctx, "ekv_deep_match: the models live on different contexts");
        const int M = edge->cfg.num_layers, N = cloud->cfg.num_layers;
        require(deep_layers >= 0 && deep_layers <= M,
                "ce_lslm: deep_layers " + std::to_string(deep_layers) + " outside [0, " +
                    std::to_string(M) + "]");
        require(n >= 2, "SimilarityConfig: num_probe_samples must be >= 2");
        ekv_ctx_s* c = edge->ctx;
        set_dev(c);
        const int he = edge->h, hc = cloud->h;
        const size_t ne = (size_t)M * n * he, ncl = (size_t)N * n * hc;
        // probe prefill of both models; per-layer outputs fp32 -> fp64 for K7
        DevMem f32(sizeof(float) * std::max(ne, ncl), c->stream);
        DevMem f64(sizeof(double) * (ne + ncl), c->stream);
        device_prefill(edge, edge_probe, n, f32.as<float>(), nullptr, nullptr, nullptr);
        launch_f32_to_f64(f32.as<float>(), f64.as<double>(), (int64_t)ne, c->stream);
        device_prefill(cloud, cloud_probe, n, f32.as<float>(), nullptr, nullptr, nullptr);
        launch_f32_to_f64(f32.as<float>(), f64.as<double>() + ne, (int64_t)ncl, c->stream);
        std::vector<double> ck((size_t)M * N), rs((size_t)M * N);
        std::vector<int> bst(M);
        rethrow(ekv_match_layers_dev(c, f64.as<double>(), M, he, f64.as<double>() + ne, N, hc, n,
                                     theta_cka, theta_rsa, ck.data(), rs.data(), bst.data()));
        if (cka) std::copy(ck.begin(), ck.end(), cka);
        if (rsa) std::copy(rs.begin(), rs.end(), rsa);
        if (best) std::copy(bst.begin(), bst.end(), best);
        const int boundary = M - deep_layers;
        for (int l = boundary; l < M; ++l) {
            require(bst[l] >= 0, "ce_lslm: edge layer " + std::to_string(l) +
                                     " has no matched cloud layer under the configured thresholds");
            deep_map[l - boundary] = bst[l];
        }
    });
}

int ekv_build_deep_kv(ekv_ctx_t c, const ekv_cloud_kv* cloud, double lambda, ekv_kvctx_t dst,
                      int n_deep, const int* edge_layers, const int* cloud_src, int* kept_host,
                      double* cut_margin_host) {
    return guard([&] {
        require(c && cloud && dst && (n_deep == 0 || (edge_layers && cloud_src)),
                "ekv_build_deep_kv: null argument");
        const ekv_cloud_kv& cl = *cloud;
        require(cl.m >= 1 && cl.m <= kMaxAlignLayers,
                "ekv_build_deep_kv: 1.." + std::to_string(kMaxAlignLayers) + " distinct cloud layers",
                EKV_EUNSUPPORTED);
        require(cl.x && cl.wq && cl.k && cl.v, "ekv_build_deep_kv: null cloud tensor");
        const int H = cl.H, d_c = cl.d_c, S = cl.S;
        ekv_model_s* em = dst->model;
        // the reference pairs heads one to one (scenario.cpp:224-234) and assembles
        // exactly the edge geometry (cache_merge.cpp:122-141)
        require(H == em->cfg.num_heads,
                "assemble_context: head count mismatch (cloud " + std::to_string(H) + ", edge " +
                    std::to_string(em->cfg.num_heads) + ")");
        int retained = 0;
        rethrow(ekv_prune_retained(lambda, d_c, &retained));
        const int d_e = em->cfg.head_dim;
        require(retained == d_e, "assemble_context: dim mismatch (cloud head_dim " + std::to_string(d_c) +
                                     " pruned to " + std::to_string(retained) + ", edge head_dim " +
                                     std::to_string(d_e) + "); align with head pruning");
        require(S == dst->S, "assemble_context: dim mismatch (cloud context " + std::to_string(S) +
                                 " rows, assembled context " + std::to_string(dst->S) + ")");
        int fmt = 0, group = 0;
        for (int i = 0; i < n_deep; ++i) {
            const int le = edge_layers[i];
            require(le >= 0 && le < em->cfg.num_layers,
                    "assemble_context: layer " + std::to_string(le) + " outside 0.." +
                        std::to_string(em->cfg.num_layers - 1));
            require(cloud_src[i] >= 0 && cloud_src[i] < cl.m,
                    "ekv_build_deep_kv: cloud source index out of range");
            const ekv_segment& sg = dst->seg[le];
            require(sg.format == EKV_KV_INT8 || sg.format == EKV_KV_INT4,
                    "ekv_build_deep_kv: deep layer " + std::to_string(le) +
                        " is not a quantised (cloud) layer of the context");
            require(i == 0 || (sg.format == fmt && sg.group == group),
                    "ekv_build_deep_kv: deep layers must share one code format");
            fmt = sg.format;
            group = sg.group;
        }
        set_dev(c);
        cudaStream_t st = c->stream;
        int* kept = nullptr;
        double* margin = nullptr;
        align_select(c, cl, retained, &kept, &margin);
        if (n_deep > 0) {
            require(2 * n_deep <= kMaxCompressJobs, "ekv_build_deep_kv: too many deep layers");
            std::vector<CompressJob> jobs(2 * n_deep);
            for (int i = 0; i < n_deep; ++i) {
                const ekv_segment& sg = dst->seg[edge_layers[i]];
                jobs[2 * i] = CompressJob{cl.k[cloud_src[i]], (void*)sg.k, (float*)sg.k_scales};
                jobs[2 * i + 1] = CompressJob{cl.v[cloud_src[i]], (void*)sg.v, (float*)sg.v_scales};
            }
            launch_kv_compress_jobs(jobs.data(), 2 * n_deep, (int64_t)H * S, d_c, kept, d_e, fmt, group,
                                    st);
        }
        fetch_mask(c, retained, kept, margin, kept_host, cut_margin_host);
    });
}

int ekv_align_select(ekv_ctx_t c, const ekv_cloud_kv* cloud, double lambda, int* kept_host,
                     double* cut_margin_host) {
    return guard([&] {
        require(c && cloud, "ekv_align_select: null argument");
        require(cloud->m >= 1 && cloud->m <= kMaxAlignLayers,
                "ekv_align_select: 1.." + std::to_string(kMaxAlignLayers) + " distinct cloud layers",
                EKV_EUNSUPPORTED);
        require(cloud->x && cloud->wq && cloud->k, "ekv_align_select: null cloud tensor");
        int retained = 0;
        rethrow(ekv_prune_retained(lambda, cloud->d_c, &retained));
        set_dev(c);
        int* kept = nullptr;
        double* margin = nullptr;
        align_select(c, *cloud, retained, &kept, &margin);
        fetch_mask(c, retained, kept, margin, kept_host, cut_margin_host);
    });
}

int ekv_prompt_context(ekv_model_t edge, ekv_model_t cloud, const float* emb_edge, const float* emb_cloud,
                       int n_deep, const int* deep_map, double lambda, ekv_kvctx_t dst, int* kept_host,
                       double* cut_margin_host) {
    return guard([&] {
        require(edge && cloud && dst && emb_edge && (n_deep == 0 || (deep_map && emb_cloud)),
                "ekv_prompt_context: null argument");
        require(edge->ctx == cloud->ctx, "ekv_prompt_context: the models live on different contexts");
        require(dst->model == edge, "ekv_prompt_context: the context belongs to another model");
        const int M = edge->cfg.num_layers, S = dst->S;
        require(n_deep >= 0 && n_deep <= M, "ce_lslm: deep_layers outside [0, num_layers]");
        ekv_ctx_s* c = edge->ctx;
        set_dev(c);
        cudaStream_t st = c->stream;
        if (S == 0) return;
        const int boundary = M - n_deep;
        const int He = edge->cfg.num_heads, de = edge->cfg.head_dim;
        // edge prefill of the context rows -> local layers [0, boundary) (sim.cpp:133, 192-205)
        if (boundary > 0) {
            const size_t lkv = (size_t)He * S * de;
            DevMem ek(sizeof(uint16_t) * M * lkv, st), ev(sizeof(uint16_t) * M * lkv, st);
            device_prefill(edge, emb_edge, S, nullptr, nullptr, ek.p, ev.p);
            for (int l = 0; l < boundary; ++l) {
                const ekv_segment& sg = dst->seg[l];
                require(sg.format == EKV_KV_BF16,
                        "ekv_prompt_context: local layer " + std::to_string(l) + " must be bf16");
                EKV_CUDA(cudaMemcpyAsync((void*)sg.k, ek.as<uint16_t>() + l * lkv, sizeof(uint16_t) * lkv,
                                         cudaMemcpyDeviceToDevice, st));
                EKV_CUDA(cudaMemcpyAsync((void*)sg.v, ev.as<uint16_t>() + l * lkv, sizeof(uint16_t) * lkv,
                                         cudaMemcpyDeviceToDevice, st));
            }
            EKV_CUDA(cudaStreamSynchronize(st));
        }
        if (n_deep == 0) return;
        // cloud prefill of the context rows: the hidden state entering every matched
        // layer and its KV cache (sim.cpp:134, 222-253)
        const int Lc = cloud->cfg.num_layers, Hc = cloud->cfg.num_heads, dc = cloud->cfg.head_dim;
        const int hc = cloud->h;
        std::vector<int> lcs(deep_map, deep_map + n_deep);
        for (int lc : lcs)
            require(lc >= 0 && lc < Lc, "ekv_prompt_context: matched cloud layer " + std::to_string(lc) +
                                            " outside 0.." + std::to_string(Lc - 1));
        std::sort(lcs.begin(), lcs.end());
        lcs.erase(std::unique(lcs.begin(), lcs.end()), lcs.end());  // std::set order (sim.cpp:219-221)
        const int m = (int)lcs.size();
        const size_t ckv = (size_t)Hc * S * dc;
        DevMem lo(sizeof(float) * (size_t)Lc * S * hc, st), x0(sizeof(float) * (size_t)S * hc, st);
        DevMem ck(sizeof(uint16_t) * Lc * ckv, st), cv(sizeof(uint16_t) * Lc * ckv, st);
        device_prefill(cloud, emb_cloud, S, lo.as<float>(), x0.as<float>(), ck.p, cv.p);
        DevMem xb(sizeof(uint16_t) * (size_t)m * S * hc, st);
        std::vector<const void*> kp(m), vp(m);
        std::vector<int> wq_index(m);
        for (int i = 0; i < m; ++i) {
            const int lc = lcs[i];
            const float* in = lc == 0 ? x0.as<float>() : lo.as<float>() + (size_t)(lc - 1) * S * hc;
            launch_f32_to_bf16(in, xb.as<uint16_t>() + (size_t)i * S * hc, (int64_t)S * hc, st);
            kp[i] = ck.as<uint16_t>() + (size_t)lc * ckv;
            vp[i] = cv.as<uint16_t>() + (size_t)lc * ckv;
            wq_index[i] = lc;
        }
        ekv_cloud_kv cl{};
        cl.m = m;
        cl.S = S;
        cl.H = Hc;
        cl.d_c = dc;
        cl.x = xb.p;
        cl.wq = cloud->weights;  // wqkvT(lc) rows [0, h_c) = W_Q^T of layer lc
        cl.wq_stride = (int64_t)cloud->layer_elems();
        cl.wq_index = wq_index.data();
        cl.k = kp.data();
        cl.v = vp.data();
        std::vector<int> le(n_deep), src(n_deep);
        for (int i = 0; i < n_deep; ++i) {
            le[i] = boundary + i;
            src[i] = (int)(std::lower_bound(lcs.begin(), lcs.end(), deep_map[i]) - lcs.begin());
        }
        rethrow(ekv_build_deep_kv(c, &cl, lambda, dst, n_deep, le.data(), src.data(), kept_host,
                                  cut_margin_host));
    });
}

int ekv_generate_embeddings(uint64_t seed, int n, int h, double* out) {
    return guard([&] {
        require(out || n == 0 || h == 0, "ekv_generate_embeddings: null output");
        require(n >= 0 && h >= 0, "ekv_generate_embeddings: negative shape");
        for (int i = 0; i < n; ++i) {
            // row i: its own mt19937_64 stream seeded with Rng::mix(seed, i) (rng.hpp:32-40)
            std::mt19937_64 eng(mix64(seed, (uint64_t)i));
            double* row = out + (size_t)i * h;
            for (int c = 0; c < h; ++c)
                row[c] = -1.0 + 2.0 * ((double)(eng() >> 11) * 0x1.0p-53);
        }
    });
}

int ekv_convert_f32_bf16(ekv_ctx_t c, const float* src, void* dst, int64_t n) {
    return guard([&] {
        require(c && src && dst, "ekv_convert_f32_bf16: null argument");
        set_dev(c);
        launch_f32_to_bf16(src, (uint16_t*)dst, n, c->stream);
    });
}

int ekv_colsq_f64(ekv_ctx_t c, const double* m_dev, int64_t rows, int d, double* colsq_dev) {
    return guard([&] {
        require(c && m_dev && colsq_dev, "ekv_colsq_f64: null argument");
        require(rows >= 0 && d >= 1, "ekv_colsq_f64: bad shape");
        set_dev(c);
        launch_colsq_f64(m_dev, rows, d, colsq_dev, c->stream);
    });
}

int ekv_kv_dequant_f64(ekv_ctx_t c, const void* codes, const float* scales, int64_t rows, int d_e,
                       int bits, int group, double* dst) {
    return guard([&] {
        require(c && codes && scales && dst, "ekv_kv_dequant_f64: null argument");
        require(bits == 8 || bits == 4, "kv_dequant: bits must be 8 or 4");
        require(group >= 1 && d_e % group == 0 && d_e * bits % 8 == 0, "kv_dequant: bad group");
        set_dev(c);
        launch_kv_dequant_f64(codes, scales, rows, d_e, bits, group, dst, c->stream);
    });
}

}  // extern "C"
