// The C-ABI (include/ekv_capi.h): argument validation with the reference's
// error texts, object lifetimes, and the collaborative-decode engine that
// strings K4/K5 together per layer and replays one captured CUDA graph per
// decode step.
#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstring>
#include <map>
#include <mutex>
#include <numeric>
#include <tuple>
#include <string>
#include <thread>
#include <vector>

#include "ekv_common.cuh"
#include "ekv_kernels.h"
#include "ekv_mega.h"
#include "ekv_batch.h"
#include "ekv_objects.h"

namespace ekv {

static std::atomic<int64_t> g_launches{0};
void count_launches(int64_t n) { g_launches += n; }

namespace {
std::mutex g_attr_mu;
std::map<std::pair<int, const void*>, int> g_smem_attr;          // (device, kernel) -> bytes set
std::map<std::tuple<int, const void*, int, int>, int> g_occ;     // (device, kernel, thr, smem)
std::map<int, int> g_sms;                                        // device -> SM count
int current_device() {
    int dev = 0;
    EKV_CUDA(cudaGetDevice(&dev));
    return dev;
}
}  // namespace

void ensure_smem_attr(const void* fn, int bytes) {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_attr_mu);
    int& have = g_smem_attr[{dev, fn}];
    if (have >= bytes) return;
    EKV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, bytes));
    have = bytes;
}

int device_sm_count() {
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto it = g_sms.find(dev);
    if (it != g_sms.end()) return it->second;
    int sms = 0;
    EKV_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
    g_sms[dev] = sms;
    return sms;
}

int blocks_per_sm(const void* fn, int threads, int smem) {
    ensure_smem_attr(fn, smem);
    const int dev = current_device();
    std::lock_guard<std::mutex> lk(g_attr_mu);
    auto key = std::make_tuple(dev, fn, threads, smem);
    auto it = g_occ.find(key);
    if (it != g_occ.end()) return it->second;
    int occ = 0;
    EKV_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, threads, smem));
    if (occ < 1) occ = 1;
    g_occ[key] = occ;
    return occ;
}

void launch_align_qnorm_batched(const void* X, const void* WqT, int m_layers, int S, int h_c,
                                int n_cols, double* colsq, int num_sms, cudaStream_t st);

}  // namespace ekv

using namespace ekv;

namespace ekv {
thread_local std::string g_err;

void release_ctx(ekv_ctx_s* c) {
    if (--c->refs > 0) return;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    if (c->own_stream) cudaStreamDestroy(c->stream);
    cudaStreamDestroy(c->capture);
    if (c->copy) cudaStreamDestroy(c->copy);
    if (c->aux) cudaStreamDestroy(c->aux);
    if (c->attn_ws) cudaFree(c->attn_ws);
    if (c->attn_ctr) cudaFree(c->attn_ctr);
    if (c->scratch) cudaFree(c->scratch);
    delete c;
}

void release_model(ekv_model_s* m) {
    if (--m->refs > 0) return;
    ekv_ctx_s* c = m->ctx;
    cudaSetDevice(c->device);
    cudaStreamSynchronize(c->stream);
    cudaFree(m->weights);
    cudaFree(m->gamma);
    cudaFree(m->bias);
    cudaFree(m->pos);
    delete m;
    release_ctx(c);
}

void release_kvctx(ekv_kvctx_s* kc) {
    if (--kc->refs > 0) return;
    ekv_model_s* m = kc->model;
    cudaSetDevice(m->ctx->device);
    cudaStreamSynchronize(m->ctx->copy);
    cudaStreamSynchronize(m->ctx->stream);
    for (void* p : kc->allocs) cudaFreeAsync(p, m->ctx->stream);
    delete kc;
    release_model(m);
}
}  // namespace ekv

namespace {

void check_device(int device, int* sms) {
    int n = 0;
    cudaError_t e = cudaGetDeviceCount(&n);
    if (e != cudaSuccess || n == 0) {
        (void)cudaGetLastError();
        throw Error(EKV_ENODEV, "no CUDA device (the B200 path has no CPU fallback)");
    }
    require(device >= 0 && device < n, "device " + std::to_string(device) + " out of range",
            EKV_ENODEV);
    cudaDeviceProp p;
    EKV_CUDA(cudaGetDeviceProperties(&p, device));
    require(p.major == 10, std::string("device ") + p.name + " is not sm_100 (B200)", EKV_ENODEV);
    *sms = p.multiProcessorCount;
}


// Tensor-core projections of R >= 2 rows of one session (K9 + split-K finish):
// QKV of layer l from `in` (fp32 [R][h]; layer 0 gets the input transform at
// positions S + user_len + row0 + r) -> q to s->q, k/v appended to the user
// cache at rows user_len + row0 + r; and the output projection x (fp32 [R][h])
// -> y (fp32 [R][h]) (+ y_hist[user_len + row0 + r] if non-null).
void tc_qkv_rows(ekv_session_s* s, int l, const float* in, int R, int row0, const CUtensorMap& pmap_x,
                 cudaStream_t st) {
    ekv_model_s* m = s->model;
    const int h = m->h;
    BatchXprep xp{};
    xp.B = R;
    xp.h = h;
    xp.state = s->state;
    xp.xhl = s->pxhl;
    xp.row0 = row0;
    if (l == 0) {
        xp.mode = 0;
        xp.xin = const_cast<float*>(in);
        xp.gamma = m->gamma;
        xp.bias = m->bias;
        xp.pos = m->pos;
        xp.pos_offset = s->kv->S;
        xp.pos_per_row = 1;
    } else {
        xp.mode = 1;
        xp.KS = 1;
        xp.part = in;
    }
    launch_batch_xprep(xp, st);
    const int ks = R <= 8 ? s->pKSq : batch_proj_splits(3 * h, h, R, m->ctx->num_sms);
    launch_batch_proj(s->pmap_w, l * 4 * h, 3 * h, h, pmap_x, R, ks, s->ppart, st);
    PrefillFinish f{};
    f.mode = 0;
    f.R = R;
    f.N = 3 * h;
    f.KS = ks;
    f.H = m->cfg.num_heads;
    f.d = m->cfg.head_dim;
    f.cap = s->cap;
    f.row0 = row0;
    f.part = s->ppart;
    f.q_out = s->q;
    f.uk = s->uk + (size_t)l * s->ukv_layer();
    f.uv = s->uv + (size_t)l * s->ukv_layer();
    f.state = s->state;
    launch_prefill_finish(f, st);
}

void tc_out_rows(ekv_session_s* s, int l, const float* x, float* y, float* y_hist, int R, int row0,
                 const CUtensorMap& pmap_x, cudaStream_t st, bool operand_ready = false) {
    const int h = s->model->h;
    if (!operand_ready) {  // else the attention already wrote the bf16 hi / lo operand
        BatchXprep xp{};
        xp.mode = 1;
        xp.B = R;
        xp.h = h;
        xp.KS = 1;
        xp.part = x;
        xp.state = s->state;
        xp.xhl = s->pxhl;
        launch_batch_xprep(xp, st);
    }
    const int ks = R <= 8 ? s->pKSo : batch_proj_splits(h, h, R, s->model->ctx->num_sms);
    launch_batch_proj(s->pmap_w, l * 4 * h + 3 * h, h, h, pmap_x, R, ks, s->ppart, st);
    PrefillFinish f{};
    f.mode = 1;
    f.R = R;
    f.N = h;
    f.KS = ks;
    f.row0 = row0;
    f.part = s->ppart;
    f.y = y;
    f.y_hist = y_hist;
    f.state = s->state;
    launch_prefill_finish(f, st);
}

CUtensorMap tc_operand_map(ekv_session_s* s, int R) {
    return make_map_3d_bf16(s->pxhl, (uint64_t)s->model->h, (uint64_t)R, 2, 64, (uint32_t)batch_proj_bn(R),
                            CU_TENSOR_MAP_SWIZZLE_128B);
}

// Tensor maps of context layer l for K10; false when K10 cannot read the layer
// (head_dim != 64, int4, or int8 with more than one scale group per row).
bool layer_ctx_maps(const ekv_kvctx_s* kv, int l, int H, int D, BatchCtxMaps& mp) {
    const ekv_segment& sg = kv->seg[l];
    mp.fmt = sg.format;
    if (sg.S == 0) return true;
    if (!batch_ctx_supported(D, sg.format, sg.group)) return false;
    const uint64_t rows = (uint64_t)H * sg.S;
    if (sg.format == EKV_KV_BF16) {
        mp.k = make_map_2d(sg.k, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)D, rows, (uint32_t)D, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B);
        mp.v = make_map_2d(sg.v, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)D, rows, (uint32_t)D, 128,
                           CU_TENSOR_MAP_SWIZZLE_128B);
    } else {
        mp.k = make_map_2d(sg.k, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)D, rows, (uint32_t)D, 128,
                           CU_TENSOR_MAP_SWIZZLE_NONE);
        mp.v = make_map_2d(sg.v, CU_TENSOR_MAP_DATA_TYPE_UINT8, 1, (uint64_t)D, rows, (uint32_t)D, 128,
                           CU_TENSOR_MAP_SWIZZLE_NONE);
        mp.ks = make_map_1d(sg.k_scales, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rows, 128);
        mp.vs = make_map_1d(sg.v_scales, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, rows, 128);
    }
    return true;
}

// Attention of R >= 2 prefill rows of one session on the tensor cores: K10 over
// the context (the rows play K10's sessions: every row attends the same S
// context rows, read once for all R rows instead of once per row), then K11 in
// prefill mode for the causal user segment + the Eq. 5 merge, writing the
// output projection's bf16 hi / lo operand.  q comes from the QKV finish
// (s->q), k / v are already in the user cache.  False: the layer needs K4.
bool tc_attn_rows(ekv_session_s* s, int l, int R, int row0, cudaStream_t st) {
    ekv_model_s* m = s->model;
    const int H = m->cfg.num_heads, D = d_of(m), h = m->h;
    const ekv_segment& sg = s->kv->seg[l];
    BatchCtxMaps mp{};
    if (!s->pctx && sg.S > 0) return false;
    if (!layer_ctx_maps(s->kv, l, H, D, mp)) return false;
    const int ns = sg.S > 0 ? batch_ctx_splits(sg.S, H, R, m->ctx->num_sms) : 0;
    if (ns > 0) {
        BatchCtxAttn a{};
        a.B = R;
        a.H = H;
        a.D = D;
        a.S = sg.S;
        a.nsplit = ns;
        a.KS = 1;
        a.n_qkv = h;  // q rows of s->q: row stride h, head hd at column hd * D
        a.qkv = s->q;
        a.part = s->pctx;
        a.state = s->state;
        launch_batch_ctx_attn(mp, a, st);
    }
    BatchUserMerge u{};
    u.B = R;
    u.H = H;
    u.D = D;
    u.L = 1;
    u.layer = 0;
    u.cap = s->cap;
    u.KS = 1;
    u.n_qkv = h;
    u.nsplit = ns;
    u.qkv = s->q;
    u.qfin = s->q;
    u.part = s->pctx;
    u.uk = s->uk + (size_t)l * s->ukv_layer();
    u.uv = s->uv + (size_t)l * s->ukv_layer();
    u.state = s->state;
    u.xhl = s->pxhl;
    u.prefill = 1;
    u.row0 = row0;
    launch_batch_user_merge(u, st);
    return true;
}

// One forward chunk of R <= 8 rows through every layer (merged_forward,
// cache_merge.cpp:156-226).  `in` holds the R input rows (fp32 [R][h]);
// `out_hist`/`hist_row_dev` receive the final-layer rows.
void forward_chunk(ekv_session_s* s, const float* in, int R, float* out_hist,
                   const int* hist_row_dev, cudaStream_t st, cudaEvent_t* ev = nullptr,
                   const cudaEvent_t* ready = nullptr) {
    ekv_model_s* m = s->model;
    const int L = m->cfg.num_layers, H = m->cfg.num_heads, d = d_of(m), h = m->h;
    int ei = 0;
    auto mark = [&] {
        if (ev) EKV_CUDA(cudaEventRecord(ev[ei++], st));
    };
    const bool tc = s->tc_prefill && R >= 2 && !ev;
    CUtensorMap pmap_x{};
    if (tc) pmap_x = tc_operand_map(s, R);
    for (int l = 0; l < L; ++l) {
        mark();
        if (tc) tc_qkv_rows(s, l, l == 0 ? in : s->xa, R, 0, pmap_x, st);
        GemvArgs g{};
        g.N = 3 * h;
        g.K = h;
        g.R = R;
        g.W = m->wqkvT(l);
        g.x = (l == 0) ? in : s->xa;
        if (l == 0) {
            g.gamma = m->gamma;
            g.bias = m->bias;
            g.pos = m->pos;
            g.pos_offset = s->kv->S;
            g.pos_base_dev = &s->state->user_len;
        }
        g.mode = 1;
        g.qkv_d = d;
        g.qkv_H = H;
        g.q_out = s->q;
        g.uk = s->uk + (size_t)l * s->ukv_layer();
        g.uv = s->uv + (size_t)l * s->ukv_layer();
        g.ucap = s->cap;
        g.user_base_dev = &s->state->user_len;
        if (!tc) launch_gemv(g, st);
        mark();
        // pipelined prefill: this layer's context must have arrived (Eq. 20: the
        // upload of layer l overlaps the compute of layers < l)
        if (ready && ready[l]) EKV_CUDA(cudaStreamWaitEvent(st, ready[l], 0));

        AttnArgs a{};
        a.R = R;
        a.H = H;
        a.D = d;
        a.q = s->q;
        const ekv_segment& sg = s->kv->seg[l];
        a.fmt = sg.format;
        a.S = sg.S;
        a.group = sg.group;
        a.ck = sg.k;
        a.cv = sg.v;
        a.cks = sg.k_scales;
        a.cvs = sg.v_scales;
        a.uk = g.uk;
        a.uv = g.uv;
        a.ucap = s->cap;
        a.user_base_dev = &s->state->user_len;
        a.out = s->xb;
        a.lse = nullptr;
        a.ws = s->ws;
        a.counters = s->counters;
        launch_decode_attention(a, st);
        mark();

        GemvArgs o{};
        o.N = h;
        o.K = h;
        o.R = R;
        o.W = m->woT(l);
        o.x = s->xb;
        o.mode = 0;
        o.y = s->xa;
        if (l == L - 1 && out_hist) {
            o.y_hist = out_hist;
            o.hist_row_dev = hist_row_dev;
        }
        if (tc) {
            // the prefill's final rows land in pre_out[user_len + r] (hist_row_dev is
            // &state->user_len for the prefill, the only caller with R >= 2)
            require(!(l == L - 1 && out_hist) || hist_row_dev == &s->state->user_len,
                    "tensor-core prefill: unexpected history row");
            tc_out_rows(s, l, s->xb, s->xa, (l == L - 1) ? out_hist : nullptr, R, 0, pmap_x, st);
        } else {
            launch_gemv(o, st);
        }
    }
    mark();
    launch_advance(s->state, R, st);
    mark();
}

// merged_forward of n user rows in LAYER-major order (every row through layer l
// before any row enters layer l+1), rows in chunks of <= 8; positions and user
// rows from host-side bases (base0 = user rows before the first new row).  Used by
// the Eq. 20 pipelined prefill, where layer l may only start once its context
// has arrived (ready[l]).  scratch: 2*n*h floats.  lev (optional): L+1 events
// around the layers.  Results are identical to forward_chunk's.
}  // namespace

namespace ekv {
void forward_layer_major(ekv_session_s* s, const float* emb, int n, int base0, cudaStream_t st,
                         const cudaEvent_t* ready, float* scratch, cudaEvent_t* lev, float* layer_out) {
    ekv_model_s* m = s->model;
    const int L = m->cfg.num_layers, H = m->cfg.num_heads, d = d_of(m), h = m->h;
    float* X = scratch;               // layer outputs [n][h]
    float* Y = scratch + (size_t)n * h;  // attention outputs [n][h]
    const int step = s->tc_prefill ? s->pchunk : 8;
    // context attention of the prefill rows on the tensor cores (K10 + K11) where the
    // layer's format allows; EKV_PREFILL_K4=1 keeps the split-KV kernel (experiments)
    const bool prefill_k10 = !getenv("EKV_PREFILL_K4");
    for (int l = 0; l < L; ++l) {
        if (lev) EKV_CUDA(cudaEventRecord(lev[l], st));
        for (int r0 = 0; r0 < n; r0 += step) {
            const int R = std::min(step, n - r0);
            const bool tc = s->tc_prefill && R >= 2;
            CUtensorMap pmap_x{};
            if (tc) pmap_x = tc_operand_map(s, R);
            if (tc) tc_qkv_rows(s, l, (l == 0) ? emb + (size_t)r0 * h : X + (size_t)r0 * h, R, base0 + r0 - s->user_len,
                                pmap_x, st);
            GemvArgs g{};
            g.N = 3 * h;
            g.K = h;
            g.R = R;
            g.W = m->wqkvT(l);
            g.x = (l == 0) ? emb + (size_t)r0 * h : X + (size_t)r0 * h;
            if (l == 0) {
                g.gamma = m->gamma;
                g.bias = m->bias;
                g.pos = m->pos;
                g.pos_offset = s->kv->S;
                g.pos_base = base0 + r0;
            }
            g.mode = 1;
            g.qkv_d = d;
            g.qkv_H = H;
            g.q_out = s->q;
            g.uk = s->uk + (size_t)l * s->ukv_layer();
            g.uv = s->uv + (size_t)l * s->ukv_layer();
            g.ucap = s->cap;
            g.user_base = base0 + r0;
            if (!tc) launch_gemv(g, st);
            if (r0 == 0 && ready && ready[l]) EKV_CUDA(cudaStreamWaitEvent(st, ready[l], 0));
            const bool k10 = tc && prefill_k10 && tc_attn_rows(s, l, R, base0 + r0 - s->user_len, st);
            AttnArgs a{};
            a.R = R;
            a.H = H;
            a.D = d;
            a.q = s->q;
            const ekv_segment& sg = s->kv->seg[l];
            a.fmt = sg.format;
            a.S = sg.S;
            a.group = sg.group;
            a.ck = sg.k;
            a.cv = sg.v;
            a.cks = sg.k_scales;
            a.cvs = sg.v_scales;
            a.uk = g.uk;
            a.uv = g.uv;
            a.ucap = s->cap;
            a.user_base = base0 + r0;
            a.out = Y + (size_t)r0 * h;
            a.ws = s->ws;
            a.counters = s->counters;
            if (!k10) launch_decode_attention(a, st);
            GemvArgs o{};
            o.N = h;
            o.K = h;
            o.R = R;
            o.W = m->woT(l);
            o.x = Y + (size_t)r0 * h;
            o.mode = 0;
            o.y = X + (size_t)r0 * h;
            if (l == L - 1) o.y_hist = s->pre_out + (size_t)(base0 + r0) * h;
            if (tc)
                tc_out_rows(s, l, Y + (size_t)r0 * h, X + (size_t)r0 * h,
                            (l == L - 1) ? s->pre_out : nullptr, R, base0 + r0 - s->user_len, pmap_x, st, k10);
            else
                launch_gemv(o, st);
        }
        if (layer_out)
            EKV_CUDA(cudaMemcpyAsync(layer_out + (size_t)l * n * h, X, sizeof(float) * n * h,
                                     cudaMemcpyDeviceToDevice, st));
    }
    if (lev) EKV_CUDA(cudaEventRecord(lev[L], st));
}

}  // namespace ekv

namespace {

size_t attn_ws_floats(int R, int H, int S, int d, int ucap) {
    int rpi = 0;
    const int items = attn_items(R, H, S, &rpi) + attn_user_items(ucap);
    return (size_t)R * H * items * (d + 2);
}

void session_alloc(ekv_session_s* s) {
    ekv_model_s* m = s->model;
    cudaStream_t ast = m->ctx->stream;
    const int L = m->cfg.num_layers, h = m->h;
    s->uk = dalloc_on<uint16_t>((size_t)L * s->ukv_layer(), ast);
    s->uv = dalloc_on<uint16_t>((size_t)L * s->ukv_layer(), ast);
    // the layer-major forward (prefill over many rows) runs the tensor-core projections
    // on chunks of up to 256 rows: the weights are read once per chunk, not per 8 rows
    const bool tc = m->h % 128 == 0 && !getenv("EKV_NO_TC_PREFILL");
    s->pchunk = tc ? std::max(8, std::min(s->cap, 256)) : 8;
    s->xa = dalloc_on<float>((size_t)8 * h, ast);
    s->xb = dalloc_on<float>((size_t)8 * h, ast);
    s->q = dalloc_on<float>((size_t)s->pchunk * h, ast);
    s->emb = dalloc_on<float>((size_t)s->cap * h, ast);
    s->pre_out = dalloc_on<float>((size_t)s->cap * h, ast);
    s->hist = dalloc_on<float>((size_t)s->cap * h, ast);
    s->state = dalloc_on<DevState>(1, ast);
    size_t ws = 0;
    for (int R : {1, 2, 3, 4, 5, 6, 7, 8, s->pchunk})
        ws = std::max(ws, attn_ws_floats(R, m->cfg.num_heads, s->kv->S, m->cfg.head_dim, s->cap));
    s->ws = dalloc_on<float>(ws, ast);
    s->counters = dalloc_on<unsigned>((size_t)s->pchunk * m->cfg.num_heads, ast);
    if (tc) {
        const int G = m->ctx->num_sms, h = m->h;
        s->tc_prefill = true;
        s->pKSq = batch_proj_splits(3 * h, h, 8, G);
        s->pKSo = batch_proj_splits(h, h, 8, G);
        s->pxhl = dalloc_on<uint16_t>((size_t)2 * s->pchunk * h, ast);
        size_t part = 0;
        for (int R : {8, s->pchunk})
            part = std::max(part, std::max((size_t)batch_proj_splits(3 * h, h, R, G) * 3 * h,
                                           (size_t)batch_proj_splits(h, h, R, G) * h) * R);
        s->ppart = dalloc_on<float>(part, ast);
        if (s->kv->S > 0 && m->cfg.head_dim == 64) {
            const int H = m->cfg.num_heads, ns = batch_ctx_splits(s->kv->S, H, 2, G);
            s->pctx = dalloc_on<float>((size_t)s->pchunk * H * ns * (64 + 4), ast);
        }
        s->pmap_w = make_map_2d(m->weights, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)h,
                                (uint64_t)m->cfg.num_layers * 4 * h, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
        // the operand map is re-encoded per chunk size R (rows >= R read as zeros)
    }
    {
        const int L = m->cfg.num_layers, H = m->cfg.num_heads, D = m->cfg.head_dim;
        const char* env = getenv("EKV_DECODE_PATH");
        if (env && std::string(env) == "graph") s->path = 1;
        {
            const int G = m->ctx->num_sms;
            s->mega_ok = mega_supported(L, H, D, s->kv->S, m->h) && m->h >= G &&
                         H * ((m->h + G - 1) / G) <= 1024;
        }
        if (s->mega_ok) {
            const int G = m->ctx->num_sms;
            const int h = m->h;
            const size_t words = (size_t)h + (size_t)H * h + 3 * (size_t)h + (size_t)G * 2 * (D + 2);
            s->mega_ll = dalloc_on<uint64_t>(words, ast);
            EKV_CUDA(cudaMemsetAsync(s->mega_ll, 0, sizeof(uint64_t) * words, ast));
            s->mega_sync = dalloc_on<unsigned>(8, ast);
            EKV_CUDA(cudaMemsetAsync(s->mega_sync, 0, sizeof(unsigned) * 8, ast));
            MegaArgs& a = s->mega;
            a.L = L;
            a.H = H;
            a.D = D;
            a.S = s->kv->S;
            a.cap = s->cap;
            a.gamma = m->gamma;
            a.bias = m->bias;
            a.pos = m->pos;
            a.state = s->state;
            a.x = s->xa;
            a.hist = s->hist;
            a.ll_x = s->mega_ll;
            a.ll_xpart = a.ll_x + h;
            a.ll_qkv = a.ll_xpart + (size_t)H * h;
            a.ll_part = a.ll_qkv + 3 * (size_t)h;
            a.sync = s->mega_sync;
            a.trace = nullptr;
            // W_o of layer l = rows [l*4h + 3h, l*4h + 4h) of the weight buffer
            a.wo_map = make_map_2d_bf16(m->weights, (uint64_t)h, (uint64_t)L * 4 * h, (uint32_t)D,
                                        (uint32_t)mega_wo_box_rows(D));
            a.wo_row0 = 3 * h;
            a.wo_layer_rows = 4 * h;
            a.prefetch_stages = 0;
            a.prefetch_ctx = 1;
            for (int l = 0; l < L; ++l) {
                const ekv_segment& sg = s->kv->seg[l];
                MegaLayer& ly = a.layer[l];
                ly.wqkv = m->wqkvT(l);
                ly.fmt = sg.S > 0 ? sg.format : EKV_KV_BF16;
                ly.group = sg.group > 0 ? sg.group : D;
                ly.ck = (const uint8_t*)sg.k;
                ly.cv = (const uint8_t*)sg.v;
                ly.cks = sg.k_scales;
                ly.cvs = sg.v_scales;
                ly.uk = s->uk + (size_t)l * s->ukv_layer();
                ly.uv = s->uv + (size_t)l * s->ukv_layer();
            }
            // L2 prefetch warp 16 stages (~192 KB per CTA) ahead of the ring while a CTA's
            // context share per layer is small: the phases then leave HBM idle between
            // them (C2: 3439 -> 3617 tok/s; S = 8192 +3%), but once the context stream
            // dominates, the early requests only compete with the demand loads (S = 16384
            // -7%, C4 -16%): profiles/r02_megakernel_experiments.txt
            {
                const int grid = mega_grid(a, m->ctx->num_sms);
                const double per = std::ceil((double)a.S * H / grid);  // context rows per CTA
                double most = 0.0;
                for (int l = 0; l < L; ++l) {
                    const MegaLayer& ly = a.layer[l];
                    const double rb = ly.fmt == 16 ? 2.0 * D : D * ly.fmt / 8.0 + 4.0 * D / ly.group;  // + scales
                    most = std::max(most, per * 2.0 * rb);
                }
                a.prefetch_stages = most <= 640.0 * 1024.0 ? 16 : 0;
            }
            if (const char* e = getenv("EKV_MEGA_PREFETCH")) a.prefetch_stages = atoi(e);
            if (const char* e = getenv("EKV_MEGA_PREFETCH_CTX")) a.prefetch_ctx = atoi(e);
            if (a.prefetch_stages > 0 && a.prefetch_stages < 4) a.prefetch_stages = 4;
        }
    }
    EKV_CUDA(cudaMemsetAsync(s->counters, 0, sizeof(unsigned) * s->pchunk * m->cfg.num_heads, ast));
    EKV_CUDA(cudaMemsetAsync(s->state, 0, sizeof(DevState), ast));
    EKV_CUDA(cudaMemsetAsync(s->uk, 0, sizeof(uint16_t) * L * s->ukv_layer(), ast));
    EKV_CUDA(cudaMemsetAsync(s->uv, 0, sizeof(uint16_t) * L * s->ukv_layer(), ast));
    EKV_CUDA(cudaStreamSynchronize(ast));
}

}  // namespace

namespace ekv {
void session_reset(ekv_session_s* s, cudaStream_t st) {
    EKV_CUDA(cudaMemsetAsync(s->state, 0, sizeof(DevState), st));
    s->user_len = 0;
    s->steps = 0;
}

void check_overflow(ekv_session_s* s, int n) {
    const int total = s->kv->S + s->user_len + n;
    require(total <= s->model->cfg.max_positions,
            "position overflow: " + std::to_string(total) + " > max_positions " +
                std::to_string(s->model->cfg.max_positions));
    require(s->user_len + n <= s->cap,
            "session full: " + std::to_string(s->user_len + n) + " user rows > capacity " +
                std::to_string(s->cap));
}

}  // namespace ekv

namespace {

// rows [0, n) of emb_dev through merged_forward in chunks of <= 8 rows;
// final-layer rows land in s->pre_out[user_row].
void session_forward(ekv_session_s* s, const float* emb_dev, int n, cudaStream_t st,
                     const cudaEvent_t* ready = nullptr) {
    check_overflow(s, n);
    if (s->tc_prefill && n >= 2 && !ready) {
        // many rows: layer-major, every layer's weights read once per chunk of <= 256
        // rows by the tensor-core projections (the user prefill of collaborative_decode)
        streamed_forward(s, emb_dev, n, nullptr, nullptr, nullptr, nullptr, nullptr);
        return;
    }
    for (int r0 = 0; r0 < n; r0 += 8) {
        const int R = std::min(8, n - r0);
        forward_chunk(s, emb_dev + (size_t)r0 * s->model->h, R, s->pre_out,
                      &s->state->user_len, st, nullptr, r0 == 0 ? ready : nullptr);
        s->user_len += R;
    }
    // decode feeds back the last row: place it in xa[0]; steps count from 0
    const int last = (n - 1) % 8;
    if (last > 0)
        EKV_CUDA(cudaMemcpyAsync(s->xa, s->xa + (size_t)last * s->model->h,
                                 sizeof(float) * s->model->h, cudaMemcpyDeviceToDevice, st));
    EKV_CUDA(cudaMemsetAsync(&s->state->step, 0, sizeof(int), st));
    s->steps = 0;
}

void ensure_step_graph(ekv_session_s* s) {
    if (s->step_graph) return;
    ekv_ctx_s* c = s->model->ctx;
    const int64_t before = g_launches.load();
    EKV_CUDA(cudaStreamBeginCapture(c->capture, cudaStreamCaptureModeThreadLocal));
    try {
        forward_chunk(s, s->xa, 1, s->hist, &s->state->step, c->capture);
    } catch (...) {
        cudaGraph_t g;
        cudaStreamEndCapture(c->capture, &g);
        if (g) cudaGraphDestroy(g);
        throw;
    }
    cudaGraph_t g = nullptr;
    EKV_CUDA(cudaStreamEndCapture(c->capture, &g));
    EKV_CUDA(cudaGraphInstantiate(&s->step_graph, g, 0));
    EKV_CUDA(cudaGraphDestroy(g));
    s->graph_kernels = g_launches.load() - before;
    g_launches -= s->graph_kernels;  // capture launched nothing; replays are counted
}

bool use_mega(const ekv_session_s* s) { return s->mega_ok && s->path == 0; }

void session_decode(ekv_session_s* s, int steps, cudaStream_t st) {
    require(steps >= 1, "collaborative_decode: steps must be >= 1");
    check_overflow(s, steps);
    require(s->steps + steps <= s->cap, "decode history full");
    if (use_mega(s)) {
        for (int t = 0; t < steps; ++t) launch_decode_mega(s->mega, s->model->ctx->num_sms, st);
        s->user_len += steps;
        s->steps += steps;
        return;
    }
    ensure_step_graph(s);
    for (int t = 0; t < steps; ++t) EKV_CUDA(cudaGraphLaunch(s->step_graph, st));
    count_launches(s->graph_kernels * steps);
    s->user_len += steps;
    s->steps += steps;
}

void ctx_storage(ekv_kvctx_s* c) {
    ekv_model_s* m = c->model;
    cudaStream_t ast = m->ctx->stream;
    const int L = m->cfg.num_layers, H = m->cfg.num_heads, d = d_of(m);
    c->seg.assign(L, ekv_segment{});
    for (int l = 0; l < L; ++l) {
        ekv_segment& s = c->seg[l];
        s.format = c->fmt[l];
        s.S = c->S;
        s.group = c->fmt[l] == EKV_KV_BF16 ? d : c->group;
        if (c->S == 0) continue;
        const size_t rows = (size_t)H * c->S;
        if (s.format == EKV_KV_BF16) {
            void* k = dalloc_on<uint16_t>(rows * d, ast);
            void* v = dalloc_on<uint16_t>(rows * d, ast);
            c->allocs.push_back(k);
            c->allocs.push_back(v);
            s.k = k;
            s.v = v;
        } else {
            const size_t bytes = rows * d * s.format / 8;
            void* k = dalloc_on<uint8_t>(bytes, ast);
            void* v = dalloc_on<uint8_t>(bytes, ast);
            float* ks = dalloc_on<float>(rows * (d / s.group), ast);
            float* vs = dalloc_on<float>(rows * (d / s.group), ast);
            for (void* p : {k, v, (void*)ks, (void*)vs}) c->allocs.push_back(p);
            s.k = k;
            s.v = v;
            s.k_scales = ks;
            s.v_scales = vs;
        }
    }
}

}  // namespace

// ===========================================================================
// Batched sessions (k_batch.cu): B sessions over one shared context, one
// forward row of every session per replay of one captured CUDA graph.
// ===========================================================================
struct ekv_batch_s {
    ekv_model_s* model = nullptr;
    ekv_kvctx_s* kv = nullptr;
    int B = 0, cap = 0;
    int KSq = 1, KSo = 1, nsplit = 0;
    uint16_t* uk = nullptr;   // [B][L][H][cap][D]
    uint16_t* uv = nullptr;
    float* xin = nullptr;     // [B][h] step input / last output
    float* hist = nullptr;    // [cap][B][h] output rows
    float* emb = nullptr;     // [B][cap][h] staged user embeddings
    uint16_t* xhl = nullptr;  // [2][B][h]
    float* qkv = nullptr;     // [KSq][B][3h]
    float* xpart = nullptr;   // [KSo][B][h]
    float* part = nullptr;    // [B][H][nsplit][D+4]: m, l, -, -, o[D]
    float* qfin = nullptr;    // [B][h] this row's q (finalised by the context kernel)
    bool use_qfin = true;     // K10 finalises q/k/v (worth it while the QKV projection is split)
    DevState* state = nullptr;
    CUtensorMap map_w{}, map_x{};
    std::vector<BatchCtxMaps> maps;   // per context layer
    cudaGraphExec_t graph = nullptr;
    int64_t graph_kernels = 0;
    int user_len = 0, rows = 0;
};

namespace {

// one forward row of every session; ev (optional) gets 1 + 5L + 2 events:
// [xprep0 | per layer: qkv, ctx, user, out, xprep | advance]
void batch_row(ekv_batch_s* b, cudaStream_t st, cudaEvent_t* ev = nullptr) {
    int ei = 0;
    auto mark = [&] {
        if (ev) EKV_CUDA(cudaEventRecord(ev[ei++], st));
    };
    mark();
    ekv_model_s* m = b->model;
    const int L = m->cfg.num_layers, H = m->cfg.num_heads, D = d_of(m), h = m->h, B = b->B;
    BatchXprep x0{};
    x0.mode = 0;
    x0.B = B;
    x0.h = h;
    x0.xin = b->xin;
    x0.gamma = m->gamma;
    x0.bias = m->bias;
    x0.pos = m->pos;
    x0.pos_offset = b->kv->S;
    x0.state = b->state;
    x0.xhl = b->xhl;
    launch_batch_xprep(x0, st);
    mark();
    for (int l = 0; l < L; ++l) {
        launch_batch_proj(b->map_w, l * 4 * h, 3 * h, h, b->map_x, B, b->KSq, b->qkv, st);
        mark();
        const ekv_segment& sg = b->kv->seg[l];
        const int ns = sg.S > 0 ? b->nsplit : 0;
        if (ns > 0) {
            BatchCtxAttn a{};
            a.B = B;
            a.H = H;
            a.D = D;
            a.S = sg.S;
            a.nsplit = ns;
            a.KS = b->KSq;
            a.n_qkv = 3 * h;
            a.qkv = b->qkv;
            a.part = b->part;
            a.qfin = b->use_qfin ? b->qfin : nullptr;
            a.uk = b->uk;
            a.uv = b->uv;
            a.L = L;
            a.layer = l;
            a.cap = b->cap;
            a.state = b->state;
            launch_batch_ctx_attn(b->maps[l], a, st);
        }
        mark();
        BatchUserMerge u{};
        u.B = B;
        u.H = H;
        u.D = D;
        u.L = L;
        u.layer = l;
        u.cap = b->cap;
        u.KS = b->KSq;
        u.n_qkv = 3 * h;
        u.nsplit = ns;
        u.qkv = b->qkv;
        u.qfin = (ns > 0 && b->use_qfin) ? b->qfin : nullptr;
        u.part = b->part;
        u.uk = b->uk;
        u.uv = b->uv;
        u.state = b->state;
        u.xhl = b->xhl;
        launch_batch_user_merge(u, st);
        mark();
        launch_batch_proj(b->map_w, l * 4 * h + 3 * h, h, h, b->map_x, B, b->KSo, b->xpart, st);
        mark();
        BatchXprep xp{};
        xp.mode = (l == L - 1) ? 2 : 1;
        xp.B = B;
        xp.h = h;
        xp.KS = b->KSo;
        xp.part = b->xpart;
        xp.xin = b->xin;
        xp.hist = b->hist;
        xp.state = b->state;
        xp.xhl = b->xhl;
        launch_batch_xprep(xp, st);
        mark();
    }
    launch_advance(b->state, 1, st);
    mark();
}

void batch_free(ekv_batch_s* b) {
    for (void* p : {(void*)b->uk, (void*)b->uv, (void*)b->xin, (void*)b->hist, (void*)b->emb,
                    (void*)b->xhl, (void*)b->qkv, (void*)b->xpart, (void*)b->part, (void*)b->qfin,
                    (void*)b->state})
        if (p) cudaFree(p);
}

void batch_alloc(ekv_batch_s* b) {
    ekv_model_s* m = b->model;
    const int L = m->cfg.num_layers, H = m->cfg.num_heads, D = d_of(m), h = m->h, B = b->B;
    const int G = m->ctx->num_sms;
    b->KSq = batch_proj_splits(3 * h, h, B, G);
    b->KSo = batch_proj_splits(h, h, B, G);
    if (const char* e = getenv("EKV_BATCH_KSQ")) b->KSq = std::max(1, std::min(8, atoi(e)));  // experiments
    if (const char* e = getenv("EKV_BATCH_KSO")) b->KSo = std::max(1, std::min(16, atoi(e)));
    b->nsplit = batch_ctx_splits(b->kv->S, H, B, G);
    const size_t ukv = (size_t)B * L * H * b->cap * D;
    b->uk = dalloc<uint16_t>(ukv);
    b->uv = dalloc<uint16_t>(ukv);
    b->xin = dalloc<float>((size_t)B * h);
    b->hist = dalloc<float>((size_t)b->cap * B * h);
    b->emb = dalloc<float>((size_t)B * b->cap * h);
    b->xhl = dalloc<uint16_t>((size_t)2 * B * h);
    b->qkv = dalloc<float>((size_t)b->KSq * B * 3 * h);
    b->xpart = dalloc<float>((size_t)b->KSo * B * h);
    b->part = dalloc<float>((size_t)B * H * std::max(b->nsplit, 1) * (D + 4));
    b->qfin = dalloc<float>((size_t)B * h);
    b->use_qfin = b->KSq > 1;
    if (const char* e = getenv("EKV_BATCH_QFIN")) b->use_qfin = atoi(e) != 0;  // experiments
    b->state = dalloc<DevState>(1);
    EKV_CUDA(cudaMemset(b->uk, 0, sizeof(uint16_t) * ukv));
    EKV_CUDA(cudaMemset(b->uv, 0, sizeof(uint16_t) * ukv));
    EKV_CUDA(cudaMemset(b->xin, 0, sizeof(float) * B * h));
    EKV_CUDA(cudaMemset(b->state, 0, sizeof(DevState)));
    b->map_w = make_map_2d(m->weights, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, (uint64_t)h,
                           (uint64_t)L * 4 * h, 64, 128, CU_TENSOR_MAP_SWIZZLE_128B);
    b->map_x = make_map_3d_bf16(b->xhl, (uint64_t)h, (uint64_t)B, 2, 64, (uint32_t)batch_proj_bn(B),
                                CU_TENSOR_MAP_SWIZZLE_128B);
    b->maps.resize(L);
    for (int l = 0; l < L; ++l) layer_ctx_maps(b->kv, l, H, D, b->maps[l]);
}

void batch_check(ekv_batch_s* b, int n) {
    const int total = b->kv->S + b->user_len + n;
    require(total <= b->model->cfg.max_positions,
            "position overflow: " + std::to_string(total) + " > max_positions " +
                std::to_string(b->model->cfg.max_positions));
    require(b->rows + n <= b->cap, "session full: " + std::to_string(b->rows + n) +
                                       " rows > capacity " + std::to_string(b->cap));
}

void batch_replay(ekv_batch_s* b, cudaStream_t st) {
    if (!b->graph) {
        ekv_ctx_s* c = b->model->ctx;
        const int64_t before = g_launches.load();
        EKV_CUDA(cudaStreamBeginCapture(c->capture, cudaStreamCaptureModeThreadLocal));
        try {
            batch_row(b, c->capture);
        } catch (...) {
            cudaGraph_t g = nullptr;
            cudaStreamEndCapture(c->capture, &g);
            if (g) cudaGraphDestroy(g);
            throw;
        }
        cudaGraph_t g = nullptr;
        EKV_CUDA(cudaStreamEndCapture(c->capture, &g));
        EKV_CUDA(cudaGraphInstantiate(&b->graph, g, 0));
        EKV_CUDA(cudaGraphDestroy(g));
        b->graph_kernels = g_launches.load() - before;
        g_launches -= b->graph_kernels;
    }
    EKV_CUDA(cudaGraphLaunch(b->graph, st));
    count_launches(b->graph_kernels);
}

// rows [0, n) of emb (device, fp32 [B][n][h], row stride `ld` rows) as user rows
void batch_forward(ekv_batch_s* b, const float* emb, int n, int ld, cudaStream_t st) {
    batch_check(b, n);
    const size_t h = b->model->h;
    for (int r = 0; r < n; ++r) {
        EKV_CUDA(cudaMemcpy2DAsync(b->xin, sizeof(float) * h, emb + (size_t)r * h, sizeof(float) * h * ld,
                                   sizeof(float) * h, b->B, cudaMemcpyDeviceToDevice, st));
        batch_replay(b, st);
    }
    b->user_len += n;
    b->rows += n;
}

void batch_decode(ekv_batch_s* b, int steps, cudaStream_t st) {
    require(steps >= 1, "collaborative_decode: steps must be >= 1");
    batch_check(b, steps);
    for (int t = 0; t < steps; ++t) batch_replay(b, st);
    b->user_len += steps;
    b->rows += steps;
}

void batch_reset(ekv_batch_s* b, cudaStream_t st) {
    EKV_CUDA(cudaMemsetAsync(b->state, 0, sizeof(DevState), st));
    EKV_CUDA(cudaMemsetAsync(b->xin, 0, sizeof(float) * b->B * b->model->h, st));
    b->user_len = 0;
    b->rows = 0;
}

}  // namespace

// ===========================================================================
extern "C" {

int ekv_abi_version(void) { return EKV_ABI_VERSION; }
const char* ekv_last_error(void) { return g_err.c_str(); }

int ekv_ctx_create(int device, void* stream, ekv_ctx_t* out) {
    return guard([&] {
        require(out != nullptr, "ekv_ctx_create: null output");
        int sms = 0;
        check_device(device, &sms);
        auto* c = new ekv_ctx_s();
        c->device = device;
        c->num_sms = sms;
        EKV_CUDA(cudaSetDevice(device));
        if (stream) {
            c->stream = (cudaStream_t)stream;
        } else {
            EKV_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
            c->own_stream = true;
        }
        EKV_CUDA(cudaStreamCreateWithFlags(&c->capture, cudaStreamNonBlocking));
        EKV_CUDA(cudaStreamCreateWithFlags(&c->copy, cudaStreamNonBlocking));
        EKV_CUDA(cudaStreamCreateWithFlags(&c->aux, cudaStreamNonBlocking));
        // keep freed stream-ordered allocations in the pool (per-request objects)
        cudaMemPool_t pool;
        EKV_CUDA(cudaDeviceGetDefaultMemPool(&pool, device));
        uint64_t keep = UINT64_MAX;
        EKV_CUDA(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep));
        *out = c;
    });
}

int ekv_ctx_destroy(ekv_ctx_t c) {
    return guard([&] {
        if (c) release_ctx(c);
    });
}

int ekv_ctx_stream(ekv_ctx_t c, void** stream) {
    return guard([&] {
        require(c && stream, "ekv_ctx_stream: null argument");
        *stream = (void*)c->stream;
    });
}

int ekv_ctx_synchronize(ekv_ctx_t c) {
    return guard([&] {
        require(c != nullptr, "null context");
        set_dev(c);
        EKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int ekv_ctx_kernel_launches(ekv_ctx_t c, int64_t* count) {
    return guard([&] {
        require(c && count, "null argument");
        *count = g_launches.load();
    });
}

int ekv_device_alloc(ekv_ctx_t c, size_t bytes, void** out) {
    return guard([&] {
        require(c && out, "ekv_device_alloc: null argument");
        set_dev(c);
        // from the device's pooled stream-ordered allocator: the C++ mirror allocates per
        // call, and the pool makes that free of cudaMalloc / cudaFree device syncs
        *out = dalloc_on<uint8_t>(bytes, c->stream);
        EKV_CUDA(cudaStreamSynchronize(c->stream));  // usable from any stream on return
    });
}

int ekv_device_free(ekv_ctx_t c, void* p) {
    return guard([&] {
        require(c != nullptr, "null context");
        set_dev(c);
        if (p) EKV_CUDA(cudaFreeAsync(p, c->stream));  // after the stream's queued work
    });
}

int ekv_memset(ekv_ctx_t c, void* dst, int value, size_t bytes) {
    return guard([&] {
        require(c && (dst || bytes == 0), "ekv_memset: null argument");
        set_dev(c);
        EKV_CUDA(cudaMemsetAsync(dst, value, bytes, c->stream));
        EKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int ekv_copy(ekv_ctx_t c, void* dst, const void* src, size_t bytes, int kind) {
    return guard([&] {
        require(c && ((dst && src) || bytes == 0), "ekv_copy: null argument");
        require(kind >= 0 && kind <= 2, "ekv_copy: kind must be 0, 1 or 2");
        set_dev(c);
        const cudaMemcpyKind k = kind == 0 ? cudaMemcpyHostToDevice
                                           : (kind == 1 ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice);
        EKV_CUDA(cudaMemcpyAsync(dst, src, bytes, k, c->stream));
        EKV_CUDA(cudaStreamSynchronize(c->stream));
    });
}

int ekv_fill_uniform_bf16(ekv_ctx_t c, void* dst, int64_t n, uint64_t seed, uint64_t stream_id,
                          double lo, double hi) {
    return guard([&] {
        require(c && (dst || n == 0), "ekv_fill_uniform_bf16: null argument");
        set_dev(c);
        launch_fill_uniform_bf16(dst, n, seed, stream_id, lo, hi, c->stream);
    });
}

// ---------------------------------------------------------------- stage 1
int ekv_prune_retained(double lambda, int head_dim, int* retained) {
    return guard([&] {
        require(retained != nullptr, "null argument");
        require(lambda >= 0.0 && lambda <= 1.0, "PruneSpec: lambda outside [0,1]");
        require(head_dim >= 1, "PruneSpec: head_dim must be >= 1");
        *retained = (int)std::floor((1.0 - lambda) * head_dim + 1e-9);
    });
}

int ekv_align_qnorm(ekv_ctx_t c, const void* X, const void* WqT, int m, int S, int h_c,
                    int n_cols, double* colsq) {
    return guard([&] {
        require(c && X && WqT && colsq, "ekv_align_qnorm: null argument");
        require(m >= 1 && S >= 1 && h_c >= 1 && n_cols >= 1, "ekv_align_qnorm: empty shape");
        set_dev(c);
        launch_align_qnorm_batched(X, WqT, m, S, h_c, n_cols, colsq, c->num_sms, c->stream);
    });
}

int ekv_kv_colnorm(ekv_ctx_t c, const void* K, int64_t rows, int d_c, double* colsq) {
    return guard([&] {
        require(c && K && colsq, "ekv_kv_colnorm: null argument");
        require(rows >= 0 && d_c >= 1, "ekv_kv_colnorm: bad shape");
        set_dev(c);
        launch_kv_colnorm(K, rows, d_c, colsq, c->stream);
    });
}

int ekv_rank_channels(const double* q_colsq, const double* k_colsq, int d_c, int retained,
                      int* kept, double* cut_margin) {
    return guard([&] {
        require(q_colsq && k_colsq && (kept || retained == 0), "ekv_rank_channels: null argument");
        require(d_c >= 1 && retained >= 0 && retained <= d_c,
                "PruneSpec: retained " + std::to_string(retained) + " outside [0," +
                    std::to_string(d_c) + "]");
        std::vector<double> score(d_c);
        for (int i = 0; i < d_c; ++i) score[i] = std::sqrt(q_colsq[i]) * std::sqrt(k_colsq[i]);
        std::vector<int> order(d_c);
        std::iota(order.begin(), order.end(), 0);
        std::stable_sort(order.begin(), order.end(),
                         [&](int a, int b) { return score[a] > score[b]; });
        std::vector<int> k(order.begin(), order.begin() + retained);
        std::sort(k.begin(), k.end());
        std::copy(k.begin(), k.end(), kept);
        if (cut_margin) {
            double mg = INFINITY;
            if (retained > 0 && retained < d_c) {
                const double a = score[order[retained - 1]], b = score[order[retained]];
                mg = a > 0 ? (a - b) / a : 0.0;
            }
            *cut_margin = mg;
        }
    });
}

int ekv_match_layers_dev(ekv_ctx_t c, const double* edge_outs, int me, int ce, const double* cloud_outs,
                         int nc, int cc, int n, double theta_cka, double theta_rsa, double* cka_out,
                         double* rsa_out, int* best) {
    return guard([&] {
        require(c && edge_outs && cloud_outs && cka_out && rsa_out && best, "null argument");
        require(me >= 1 && nc >= 1, "match_layers: empty layer output list");
        require(theta_cka >= 0.0, "SimilarityConfig: theta_cka must be >= 0");
        require(theta_rsa >= -1.0, "SimilarityConfig: theta_rsa must be >= -1");
        require(n >= 3, "rsa: need N >= 3 samples");
        require(n <= 256, "match_layers_dev: at most 256 probe rows", EKV_EUNSUPPORTED);
        require(ce >= 1 && cc >= 1, "match_layers: bad layer width");
        set_dev(c);
        const int L = me + nc;
        const size_t m = (size_t)n * (n - 1) / 2, P = (size_t)me * nc;
        // one work allocation: doubles then ints
        const size_t nd = L + 2 * (size_t)L * n * n + L + (size_t)L * m + 2 * P;
        const size_t ni = L + P;
        char* w = nullptr;
        EKV_CUDA(cudaMallocAsync((void**)&w, nd * sizeof(double) + ni * sizeof(int), c->stream));
        double* d = (double*)w;
        double* scale = d;
        double* gram = scale + L;
        double* centred = gram + (size_t)L * n * n;
        double* self_h = centred + (size_t)L * n * n;
        double* cosflat = self_h + L;
        double* hsic = cosflat + (size_t)L * m;
        double* corr = hsic + P;
        int* zero_row = (int*)(corr + P);
        int* zero_var = zero_row + L;
        launch_layer_match(edge_outs, me, ce, cloud_outs, nc, cc, n, scale, gram, centred, self_h, cosflat,
                           zero_row, hsic, corr, zero_var, c->stream);
        std::vector<double> hself(L), hh(P), hc(P);
        std::vector<int> hz(L), hv(P);
        EKV_CUDA(cudaMemcpyAsync(hself.data(), self_h, sizeof(double) * L, cudaMemcpyDeviceToHost, c->stream));
        EKV_CUDA(cudaMemcpyAsync(hh.data(), hsic, sizeof(double) * P, cudaMemcpyDeviceToHost, c->stream));
        EKV_CUDA(cudaMemcpyAsync(hc.data(), corr, sizeof(double) * P, cudaMemcpyDeviceToHost, c->stream));
        EKV_CUDA(cudaMemcpyAsync(hz.data(), zero_row, sizeof(int) * L, cudaMemcpyDeviceToHost, c->stream));
        EKV_CUDA(cudaMemcpyAsync(hv.data(), zero_var, sizeof(int) * P, cudaMemcpyDeviceToHost, c->stream));
        EKV_CUDA(cudaFreeAsync(w, c->stream));
        EKV_CUDA(cudaStreamSynchronize(c->stream));
        // the reference's argmax and its error order (cka, then rsa, per (le, lc))
        for (int le = 0; le < me; ++le) {
            int bl = -1;
            double bc = 0.0;
            for (int lc = 0; lc < nc; ++lc) {
                const size_t p = (size_t)le * nc + lc;
                require(hself[le] >= 1e-15 && hself[me + lc] >= 1e-15, "cka: degenerate representation");
                require(hz[le] < 0, "rsa: zero-norm row " + std::to_string(hz[le]));
                require(hz[me + lc] < 0, "rsa: zero-norm row " + std::to_string(hz[me + lc]));
                require(!hv[p], "pearson_corr: zero variance");
                const double ck = hh[p] / std::sqrt(hself[le] * hself[me + lc]);
                cka_out[p] = ck;
                rsa_out[p] = hc[p];
                if (ck >= theta_cka && hc[p] >= theta_rsa && (bl < 0 || ck > bc)) {
                    bl = lc;
                    bc = ck;
                }
            }
            best[le] = bl;
        }
    });
}

// ---------------------------------------------------------------- stage 2
static void check_rows_args(ekv_ctx_t c, const void* a, const void* b, int64_t rows, int d_c,
                            const int* kept, int d_e, const char* fn) {
    require(c && a && b && kept, std::string(fn) + ": null argument");
    require(rows >= 0 && d_c >= 1 && d_e >= 1 && d_e <= d_c,
            std::string(fn) + ": need 1 <= d_e <= d_c");
}

int ekv_kv_gather(ekv_ctx_t c, const void* src, int64_t rows, int d_c, const int* kept, int d_e,
                  void* dst) {
    return guard([&] {
        check_rows_args(c, src, dst, rows, d_c, kept, d_e, "ekv_kv_gather");
        set_dev(c);
        launch_kv_gather(src, rows, d_c, kept, d_e, dst, c->stream);
    });
}

int ekv_gather_columns(ekv_ctx_t c, const void* src, int64_t rows, int d_c, const int* kept,
                       int d_e, int elem_bytes, void* dst) {
    return guard([&] {
        check_rows_args(c, src, dst, rows, d_c, kept, d_e, "ekv_gather_columns");
        set_dev(c);
        launch_gather_columns(src, rows, d_c, kept, d_e, elem_bytes, dst, c->stream);
    });
}

int ekv_kv_compress(ekv_ctx_t c, const void* src, int64_t rows, int d_c, const int* kept, int d_e,
                    int bits, int group, void* codes, float* scales) {
    return guard([&] {
        check_rows_args(c, src, codes, rows, d_c, kept, d_e, "ekv_kv_compress");
        require(scales != nullptr, "ekv_kv_compress: null scales");
        require(bits == 8 || bits == 4, "ekv_kv_compress: bits must be 8 or 4");
        require(group >= 1 && d_e % group == 0, "ekv_kv_compress: group must divide d_e");
        require(bits == 8 || (group % 2 == 0 && d_e % 2 == 0),
                "ekv_kv_compress: int4 needs an even group");
        set_dev(c);
        launch_kv_compress(src, rows, d_c, kept, d_e, bits, group, codes, scales, c->stream);
    });
}

int ekv_kv_compress_batched(ekv_ctx_t c, int n, const void* const* src, int64_t rows, int d_c,
                            const int* kept, int d_e, int bits, int group, void* const* codes,
                            float* const* scales) {
    return guard([&] {
        require(c && src && codes && scales && kept, "ekv_kv_compress_batched: null argument");
        require(n >= 0 && n <= kMaxCompressJobs, "ekv_kv_compress_batched: 0.." +
                                                     std::to_string(kMaxCompressJobs) + " jobs");
        require(rows >= 0 && d_c >= 1 && d_e >= 1 && d_e <= d_c,
                "ekv_kv_compress_batched: need 1 <= d_e <= d_c");
        require(bits == 8 || bits == 4, "ekv_kv_compress: bits must be 8 or 4");
        require(group >= 1 && d_e % group == 0, "ekv_kv_compress: group must divide d_e");
        require(bits == 8 || group % 2 == 0, "ekv_kv_compress: int4 needs an even group");
        std::vector<CompressJob> jobs(n);
        for (int i = 0; i < n; ++i) {
            require(src[i] && codes[i] && scales[i], "ekv_kv_compress_batched: null job pointer");
            jobs[i] = CompressJob{src[i], codes[i], scales[i]};
        }
        set_dev(c);
        launch_kv_compress_jobs(jobs.data(), n, rows, d_c, kept, d_e, bits, group, c->stream);
    });
}

int ekv_kv_dequant(ekv_ctx_t c, const void* codes, const float* scales, int64_t rows, int d_e,
                   int bits, int group, void* dst) {
    return guard([&] {
        require(c && codes && scales && dst, "ekv_kv_dequant: null argument");
        require(bits == 8 || bits == 4, "ekv_kv_dequant: bits must be 8 or 4");
        require(group >= 1 && d_e % group == 0, "ekv_kv_dequant: group must divide d_e");
        set_dev(c);
        launch_kv_dequant(codes, scales, rows, d_e, bits, group, dst, c->stream);
    });
}

// ---------------------------------------------------------------- stage 3
static void check_segment(const ekv_segment& s, int d) {
    require(s.S >= 0, "decode_attention: negative context length");
    if (s.S == 0) return;
    require(s.k && s.v, "decode_attention: null context K/V");
    require(s.format == EKV_KV_BF16 || s.format == EKV_KV_INT8 || s.format == EKV_KV_INT4,
            "decode_attention: unknown context format");
    if (s.format != EKV_KV_BF16) {
        require(s.k_scales && s.v_scales, "decode_attention: null scales");
        const int epl = s.format == EKV_KV_INT8 ? 16 : 32;
        require(s.group >= epl && s.group % epl == 0 && d % s.group == 0,
                "decode_attention: group must be a multiple of " + std::to_string(epl) +
                    " dividing head_dim",
                EKV_EUNSUPPORTED);
    }
}

int ekv_decode_attention(ekv_ctx_t c, int R, int H, int d, const float* q,
                         const ekv_segment* ctx_seg, const void* uk, const void* uv, int user_cap,
                         int user_base, float* out, float* lse) {
    return guard([&] {
        require(c && q && ctx_seg && uk && uv && out, "ekv_decode_attention: null argument");
        require(R >= 1 && H >= 1, "ekv_decode_attention: empty shape");
        require(d == 32 || d == 64 || d == 128, "ekv_decode_attention: head_dim must be 32, 64 or 128",
                EKV_EUNSUPPORTED);
        require(user_base >= 0 && user_base + R <= user_cap,
                "segment_attention: empty segment (user rows exceed the cache)");
        check_segment(*ctx_seg, d);
        set_dev(c);
        // the scratch belongs to this context (its device and stream): grown on demand
        const size_t need = attn_ws_floats(R, H, ctx_seg->S, d, user_cap);
        if (need > c->attn_ws_n) {
            EKV_CUDA(cudaStreamSynchronize(c->stream));
            if (c->attn_ws) cudaFree(c->attn_ws);
            c->attn_ws = nullptr;
            c->attn_ws = dalloc<float>(need);
            c->attn_ws_n = need;
        }
        if ((size_t)R * H > c->attn_ctr_n) {
            EKV_CUDA(cudaStreamSynchronize(c->stream));
            if (c->attn_ctr) cudaFree(c->attn_ctr);
            c->attn_ctr = nullptr;
            c->attn_ctr = dalloc<unsigned>((size_t)R * H);
            EKV_CUDA(cudaMemset(c->attn_ctr, 0, sizeof(unsigned) * R * H));
            c->attn_ctr_n = (size_t)R * H;
        }
        float* ws = c->attn_ws;
        unsigned* ctr = c->attn_ctr;
        AttnArgs a{};
        a.R = R;
        a.H = H;
        a.D = d;
        a.q = q;
        a.fmt = ctx_seg->S > 0 ? ctx_seg->format : EKV_KV_BF16;
        a.S = ctx_seg->S;
        a.group = ctx_seg->group;
        a.ck = ctx_seg->k;
        a.cv = ctx_seg->v;
        a.cks = ctx_seg->k_scales;
        a.cvs = ctx_seg->v_scales;
        a.uk = (const uint16_t*)uk;
        a.uv = (const uint16_t*)uv;
        a.ucap = user_cap;
        a.user_base = user_base;
        a.out = out;
        a.lse = lse;
        a.ws = ws;
        a.counters = ctr;
        launch_decode_attention(a, c->stream);
    });
}

// ---------------------------------------------------------------- model
int ekv_model_create(ekv_ctx_t c, const ekv_model_config* cfg, ekv_model_t* out) {
    return guard([&] {
        require(c && cfg && out, "ekv_model_create: null argument");
        require(cfg->num_layers >= 1, "ModelConfig: num_layers must be >= 1");
        require(cfg->head_dim >= 1, "ModelConfig: head_dim must be >= 1");
        require(cfg->num_heads >= 1, "ModelConfig: num_heads must be >= 1");
        require(cfg->max_positions >= 1, "ModelConfig: max_positions must be >= 1");
        const int h = cfg->num_heads * cfg->head_dim;
        require(h % 256 == 0 && h <= 4096,
                "ModelConfig: hidden_size must be a multiple of 256 (<= 4096) for the B200 "
                "projection kernels",
                EKV_EUNSUPPORTED);
        require(cfg->head_dim == 32 || cfg->head_dim == 64 || cfg->head_dim == 128,
                "ModelConfig: head_dim must be 32, 64 or 128", EKV_EUNSUPPORTED);
        set_dev(c);
        auto* m = new ekv_model_s();
        m->ctx = c;
        m->cfg = *cfg;
        m->h = h;
        try {
            m->weights = dalloc<uint16_t>((size_t)cfg->num_layers * m->layer_elems());
            m->gamma = dalloc<float>(h);
            m->bias = dalloc<float>(h);
            m->pos = dalloc<uint16_t>((size_t)cfg->max_positions * h);
        } catch (...) {
            cudaFree(m->weights);
            cudaFree(m->gamma);
            cudaFree(m->bias);
            cudaFree(m->pos);
            delete m;
            throw;
        }
        c->refs++;
        *out = m;
    });
}

int ekv_model_destroy(ekv_model_t m) {
    return guard([&] {
        if (m) release_model(m);
    });
}

int ekv_model_set_layer(ekv_model_t m, int layer, const uint16_t* wqkvT, const uint16_t* woT) {
    return guard([&] {
        require(m && wqkvT && woT, "ekv_model_set_layer: null argument");
        require(layer >= 0 && layer < m->cfg.num_layers,
                "project_qkv: layer " + std::to_string(layer) + " out of range");
        set_dev(m->ctx);
        const size_t h = m->h;
        EKV_CUDA(cudaMemcpyAsync(m->wqkvT(layer), wqkvT, 3 * h * h * 2, cudaMemcpyHostToDevice,
                                 m->ctx->stream));
        EKV_CUDA(cudaMemcpyAsync(m->woT(layer), woT, h * h * 2, cudaMemcpyHostToDevice,
                                 m->ctx->stream));
        EKV_CUDA(cudaStreamSynchronize(m->ctx->stream));
    });
}

int ekv_model_set_io(ekv_model_t m, const float* gamma, const float* bias, const uint16_t* pos) {
    return guard([&] {
        require(m && gamma && bias && pos, "ekv_model_set_io: null argument");
        set_dev(m->ctx);
        const size_t h = m->h;
        EKV_CUDA(cudaMemcpyAsync(m->gamma, gamma, h * 4, cudaMemcpyHostToDevice, m->ctx->stream));
        EKV_CUDA(cudaMemcpyAsync(m->bias, bias, h * 4, cudaMemcpyHostToDevice, m->ctx->stream));
        EKV_CUDA(cudaMemcpyAsync(m->pos, pos, (size_t)m->cfg.max_positions * h * 2,
                                 cudaMemcpyHostToDevice, m->ctx->stream));
        EKV_CUDA(cudaStreamSynchronize(m->ctx->stream));
    });
}

int ekv_model_synthesize(ekv_model_t m, uint64_t seed, double w_scale, double pos_scale) {
    return guard([&] {
        require(m != nullptr, "null model");
        set_dev(m->ctx);
        cudaStream_t st = m->ctx->stream;
        const int L = m->cfg.num_layers, h = m->h;
        const double qs = w_scale / std::sqrt((double)m->cfg.head_dim);  // 1/sqrt(d) folded into W_Q
        for (int l = 0; l < L; ++l) {
            launch_fill_uniform_bf16(m->wqkvT(l), (int64_t)h * h, seed, 4 * l + 0, -qs, qs, st);
            launch_fill_uniform_bf16(m->wqkvT(l) + (size_t)h * h, (int64_t)2 * h * h, seed,
                                     4 * l + 1, -w_scale, w_scale, st);
            launch_fill_uniform_bf16(m->woT(l), (int64_t)h * h, seed, 4 * l + 2, -w_scale,
                                     w_scale, st);
        }
        launch_fill_uniform_bf16(m->pos, (int64_t)m->cfg.max_positions * h, seed, 0x706F73,
                                 -pos_scale, pos_scale, st);
        std::vector<float> ones(h, 1.0f), zeros(h, 0.0f);
        EKV_CUDA(cudaMemcpyAsync(m->gamma, ones.data(), h * 4, cudaMemcpyHostToDevice, st));
        EKV_CUDA(cudaMemcpyAsync(m->bias, zeros.data(), h * 4, cudaMemcpyHostToDevice, st));
        EKV_CUDA(cudaStreamSynchronize(st));
    });
}

int ekv_model_weights(ekv_model_t m, int layer, void** wqkvT, void** woT) {
    return guard([&] {
        require(m && wqkvT && woT, "null argument");
        require(layer >= 0 && layer < m->cfg.num_layers, "layer out of range");
        *wqkvT = m->wqkvT(layer);
        *woT = m->woT(layer);
    });
}

int ekv_model_io(ekv_model_t m, float** gamma, float** bias, void** pos) {
    return guard([&] {
        require(m && gamma && bias && pos, "null argument");
        *gamma = m->gamma;
        *bias = m->bias;
        *pos = m->pos;
    });
}

// ---------------------------------------------------------------- context
int ekv_kvctx_create(ekv_model_t m, int S, const int* layer_format, int group, ekv_kvctx_t* out) {
    return guard([&] {
        require(m && layer_format && out, "ekv_kvctx_create: null argument");
        require(S >= 0, "assemble_context: negative context length");
        const int L = m->cfg.num_layers, d = m->cfg.head_dim;
        auto* c = new ekv_kvctx_s();
        c->model = m;
        c->S = S;
        c->group = group;
        c->fmt.assign(layer_format, layer_format + L);
        try {
            for (int l = 0; l < L; ++l) {
                const int f = c->fmt[l];
                require(f == EKV_KV_BF16 || f == EKV_KV_INT8 || f == EKV_KV_INT4,
                        "assemble_context: layer " + std::to_string(l) + " has an unknown format");
                if (f != EKV_KV_BF16) {
                    const int epl = f == EKV_KV_INT8 ? 16 : 32;
                    require(group >= epl && group % epl == 0 && d % group == 0,
                            "assemble_context: layer " + std::to_string(l) +
                                " dim mismatch (group " + std::to_string(group) +
                                " incompatible with head_dim " + std::to_string(d) + ")",
                            EKV_EUNSUPPORTED);
                }
            }
            set_dev(m->ctx);
            ctx_storage(c);
        } catch (...) {
            for (void* p : c->allocs) cudaFreeAsync(p, m->ctx->stream);
            cudaStreamSynchronize(m->ctx->stream);
            delete c;
            throw;
        }
        EKV_CUDA(cudaStreamSynchronize(m->ctx->stream));  // storage usable from any stream
        m->refs++;
        *out = c;
    });
}

int ekv_kvctx_destroy(ekv_kvctx_t c) {
    return guard([&] {
        if (c) release_kvctx(c);
    });
}

int ekv_kvctx_layer(ekv_kvctx_t c, int layer, ekv_segment* seg) {
    return guard([&] {
        require(c && seg, "null argument");
        require(layer >= 0 && layer < (int)c->seg.size(),
                "assemble_context: missing layer " + std::to_string(layer));
        *seg = c->seg[layer];
    });
}

int ekv_kvctx_upload_bf16(ekv_kvctx_t c, int layer, const uint16_t* k, const uint16_t* v) {
    return guard([&] {
        require(c && k && v, "null argument");
        require(layer >= 0 && layer < (int)c->seg.size(),
                "assemble_context: missing layer " + std::to_string(layer));
        const ekv_segment& s = c->seg[layer];
        require(s.format == EKV_KV_BF16,
                "assemble_context: layer " + std::to_string(layer) + " is not a bf16 layer");
        if (c->S == 0) return;
        set_dev(c->model->ctx);
        const size_t bytes = (size_t)c->model->cfg.num_heads * c->S * c->model->cfg.head_dim * 2;
        cudaStream_t st = c->model->ctx->stream;
        EKV_CUDA(cudaMemcpyAsync((void*)s.k, k, bytes, cudaMemcpyHostToDevice, st));
        EKV_CUDA(cudaMemcpyAsync((void*)s.v, v, bytes, cudaMemcpyHostToDevice, st));
        EKV_CUDA(cudaStreamSynchronize(st));
    });
}

int ekv_kvctx_set_layer(ekv_kvctx_t c, int layer, const void* k, const void* v, const float* ks,
                        const float* vs) {
    return guard([&] {
        require(c && k && v, "ekv_kvctx_set_layer: null argument");
        require(layer >= 0 && layer < (int)c->seg.size(),
                "assemble_context: missing layer " + std::to_string(layer));
        const ekv_segment& s = c->seg[layer];
        if (c->S == 0) return;
        ekv_model_s* m = c->model;
        set_dev(m->ctx);
        cudaStream_t st = m->ctx->stream;
        const size_t rows = (size_t)m->cfg.num_heads * c->S, d = m->cfg.head_dim;
        const size_t bytes = rows * d * s.format / 8;
        EKV_CUDA(cudaMemcpyAsync((void*)s.k, k, bytes, cudaMemcpyDeviceToDevice, st));
        EKV_CUDA(cudaMemcpyAsync((void*)s.v, v, bytes, cudaMemcpyDeviceToDevice, st));
        if (s.format != EKV_KV_BF16) {
            require(ks && vs, "ekv_kvctx_set_layer: quantised layer needs scales");
            const size_t sb = rows * (d / s.group) * sizeof(float);
            EKV_CUDA(cudaMemcpyAsync((void*)s.k_scales, ks, sb, cudaMemcpyDeviceToDevice, st));
            EKV_CUDA(cudaMemcpyAsync((void*)s.v_scales, vs, sb, cudaMemcpyDeviceToDevice, st));
        }
    });
}

int ekv_kvctx_copy_layers(ekv_kvctx_t dst, ekv_kvctx_t src, const int* layers, int n) {
    return guard([&] {
        require(dst && src && (layers || n == 0), "ekv_kvctx_copy_layers: null argument");
        ekv_model_s* dm = dst->model;
        ekv_model_s* sm = src->model;
        require(dm->cfg.num_heads == sm->cfg.num_heads && dm->cfg.head_dim == sm->cfg.head_dim &&
                    dst->S == src->S,
                "assemble_context: dim mismatch (peer context H=" + std::to_string(sm->cfg.num_heads) +
                    " S=" + std::to_string(src->S) + ", this context H=" + std::to_string(dm->cfg.num_heads) +
                    " S=" + std::to_string(dst->S) + ")");
        const int dd = dm->ctx->device, sd = sm->ctx->device;
        if (dd != sd) {  // NVLink peer access when the pair supports it (else staged by the driver)
            int ok = 0;
            EKV_CUDA(cudaDeviceCanAccessPeer(&ok, dd, sd));
            if (ok) {
                set_dev(dm->ctx);
                cudaError_t e = cudaDeviceEnablePeerAccess(sd, 0);
                if (e != cudaSuccess && e != cudaErrorPeerAccessAlreadyEnabled) EKV_CUDA(e);
                (void)cudaGetLastError();
            }
        }
        // the copy runs on the destination's stream after the source's queued work
        cudaEvent_t src_done = nullptr;
        set_dev(sm->ctx);
        EKV_CUDA(cudaEventCreateWithFlags(&src_done, cudaEventDisableTiming));
        EKV_CUDA(cudaEventRecord(src_done, sm->ctx->stream));
        set_dev(dm->ctx);
        cudaStream_t st = dm->ctx->stream;
        cudaError_t werr = cudaStreamWaitEvent(st, src_done, 0);
        cudaEventDestroy(src_done);
        EKV_CUDA(werr);
        const size_t rows = (size_t)dm->cfg.num_heads * dst->S, d = dm->cfg.head_dim;
        for (int i = 0; i < n; ++i) {
            const int l = layers[i];
            require(l >= 0 && l < (int)dst->seg.size() && l < (int)src->seg.size(),
                    "assemble_context: missing layer " + std::to_string(l));
            const ekv_segment& a = src->seg[l];
            const ekv_segment& b = dst->seg[l];
            require(a.format == b.format && a.group == b.group,
                    "assemble_context: layer " + std::to_string(l) + " format differs between the contexts");
            if (dst->S == 0) continue;
            const size_t cb = rows * d * b.format / 8, sb = rows * (d / std::max(b.group, 1)) * 4;
            EKV_CUDA(cudaMemcpyPeerAsync((void*)b.k, dd, a.k, sd, cb, st));
            EKV_CUDA(cudaMemcpyPeerAsync((void*)b.v, dd, a.v, sd, cb, st));
            if (b.format != EKV_KV_BF16) {
                EKV_CUDA(cudaMemcpyPeerAsync((void*)b.k_scales, dd, a.k_scales, sd, sb, st));
                EKV_CUDA(cudaMemcpyPeerAsync((void*)b.v_scales, dd, a.v_scales, sd, sb, st));
            }
        }
        EKV_CUDA(cudaStreamSynchronize(st));
    });
}

int ekv_kvctx_synthesize(ekv_kvctx_t c, uint64_t seed) {
    return guard([&] {
        require(c != nullptr, "null context");
        if (c->S == 0) return;
        ekv_model_s* m = c->model;
        set_dev(m->ctx);
        cudaStream_t st = m->ctx->stream;
        const int H = m->cfg.num_heads, d = m->cfg.head_dim;
        const int64_t rows = (int64_t)H * c->S;
        for (size_t l = 0; l < c->seg.size(); ++l) {
            const ekv_segment& s = c->seg[l];
            if (s.format == EKV_KV_BF16) {
                launch_fill_uniform_bf16((void*)s.k, rows * d, seed, 1000 + 2 * l, -1.0, 1.0, st);
                launch_fill_uniform_bf16((void*)s.v, rows * d, seed, 1001 + 2 * l, -1.0, 1.0, st);
            } else {
                // random bf16 staging rows, then the real compressor (kept = identity)
                uint16_t* tmp = dalloc<uint16_t>((size_t)rows * d);
                int* kept = dalloc<int>(d);
                std::vector<int> id(d);
                std::iota(id.begin(), id.end(), 0);
                EKV_CUDA(cudaMemcpyAsync(kept, id.data(), sizeof(int) * d, cudaMemcpyHostToDevice, st));
                for (int kv = 0; kv < 2; ++kv) {
                    launch_fill_uniform_bf16(tmp, rows * d, seed, 1000 + 2 * l + kv, -1.0, 1.0, st);
                    launch_kv_compress(tmp, rows, d, kept, d, s.format, s.group,
                                       (void*)(kv ? s.v : s.k),
                                       (float*)(kv ? s.v_scales : s.k_scales), st);
                }
                EKV_CUDA(cudaStreamSynchronize(st));
                cudaFree(tmp);
                cudaFree(kept);
            }
        }
        EKV_CUDA(cudaStreamSynchronize(st));
    });
}

// ---------------------------------------------------------------- sessions
int ekv_session_create(ekv_model_t m, ekv_kvctx_t c, int max_user_rows, ekv_session_t* out) {
    return guard([&] {
        require(m && c && out, "ekv_session_create: null argument");
        require(c->model == m || (c->model->cfg.num_heads == m->cfg.num_heads &&
                                  c->model->cfg.head_dim == m->cfg.head_dim),
                "collaborative_decode: context dims do not match model; align with head pruning "
                "first");
        require((int)c->seg.size() == m->cfg.num_layers,
                "collaborative_decode: context has " + std::to_string(c->seg.size()) +
                    " layers, model has " + std::to_string(m->cfg.num_layers));
        require(max_user_rows >= 1, "ekv_session_create: max_user_rows must be >= 1");
        set_dev(m->ctx);
        auto* s = new ekv_session_s();
        s->model = m;
        s->kv = c;
        s->cap = max_user_rows;
        try {
            session_alloc(s);
        } catch (...) {
            for (void* p : {(void*)s->uk, (void*)s->uv, (void*)s->xa, (void*)s->xb, (void*)s->q,
                            (void*)s->emb, (void*)s->pre_out, (void*)s->hist, (void*)s->state,
                            (void*)s->ws, (void*)s->counters, (void*)s->pxhl, (void*)s->ppart,
                            (void*)s->pctx, (void*)s->mega_ll, (void*)s->mega_sync})
                if (p) cudaFreeAsync(p, m->ctx->stream);
            cudaStreamSynchronize(m->ctx->stream);
            delete s;
            throw;
        }
        m->refs++;
        c->refs++;
        *out = s;
    });
}

int ekv_session_destroy(ekv_session_t s) {
    return guard([&] {
        if (!s) return;
        cudaSetDevice(s->model->ctx->device);
        cudaStream_t fst = s->model->ctx->stream;
        cudaStreamSynchronize(s->model->ctx->copy);
        cudaStreamSynchronize(fst);
        if (s->step_graph) cudaGraphExecDestroy(s->step_graph);
        for (void* p : {(void*)s->uk, (void*)s->uv, (void*)s->xa, (void*)s->xb, (void*)s->q,
                        (void*)s->emb, (void*)s->pre_out, (void*)s->hist, (void*)s->state,
                        (void*)s->ws, (void*)s->counters, (void*)s->mega_ll, (void*)s->mega_sync,
                        (void*)s->pxhl, (void*)s->ppart, (void*)s->pctx})
            if (p) cudaFreeAsync(p, fst);
        ekv_kvctx_s* kv = s->kv;
        ekv_model_s* m = s->model;
        delete s;
        release_kvctx(kv);
        release_model(m);
    });
}

int ekv_session_trace_step(ekv_session_t s, uint64_t* out, int capacity, int* n_out) {
    return guard([&] {
        require(s && out && n_out, "null argument");
        require(use_mega(s), "trace: the persistent decode kernel is not active");
        const int G = mega_grid(s->mega, s->model->ctx->num_sms);
        const int L = s->model->cfg.num_layers;
        const int n = 16 * (L + 1) * G;
        require(capacity >= n, "trace: need " + std::to_string(n) + " entries");
        check_overflow(s, 1);
        set_dev(s->model->ctx);
        cudaStream_t st = s->model->ctx->stream;
        unsigned long long* d = dalloc<unsigned long long>(n);
        EKV_CUDA(cudaMemsetAsync(d, 0, sizeof(unsigned long long) * n, st));
        MegaArgs a = s->mega;
        a.trace = d;
        launch_decode_mega(a, G, st);
        EKV_CUDA(cudaMemcpyAsync(out, d, sizeof(uint64_t) * n, cudaMemcpyDeviceToHost, st));
        EKV_CUDA(cudaStreamSynchronize(st));
        cudaFree(d);
        s->user_len += 1;
        s->steps += 1;
        *n_out = n;
    });
}

int ekv_session_set_decode_path(ekv_session_t s, int path, int* active) {
    return guard([&] {
        require(s != nullptr, "null session");
        require(path == 0 || path == 1, "decode path must be 0 (persistent kernel) or 1 (graph)");
        s->path = path;
        if (active) *active = use_mega(s) ? 0 : 1;
    });
}

int ekv_session_reset(ekv_session_t s) {
    return guard([&] {
        require(s != nullptr, "null session");
        set_dev(s->model->ctx);
        session_reset(s, s->model->ctx->stream);
    });
}

int ekv_session_length(ekv_session_t s, int* rows) {
    return guard([&] {
        require(s && rows, "null argument");
        *rows = s->user_len;
    });
}

int ekv_session_forward(ekv_session_t s, const float* emb, int n, float* out) {
    return guard([&] {
        require(s && emb && out, "ekv_session_forward: null argument");
        require(n >= 1, "ekv_session_forward: n must be >= 1");
        set_dev(s->model->ctx);
        cudaStream_t st = s->model->ctx->stream;
        const int first = s->user_len;
        session_forward(s, emb, n, st);
        EKV_CUDA(cudaMemcpyAsync(out, s->pre_out + (size_t)first * s->model->h,
                                 sizeof(float) * n * s->model->h, cudaMemcpyDeviceToDevice, st));
    });
}

int ekv_session_decode(ekv_session_t s, int steps, float* out) {
    return guard([&] {
        require(s && out, "ekv_session_decode: null argument");
        set_dev(s->model->ctx);
        cudaStream_t st = s->model->ctx->stream;
        if (s->user_len == 0 && s->steps == 0)  // no prefill: the first input row is zeros
            EKV_CUDA(cudaMemsetAsync(s->xa, 0, sizeof(float) * s->model->h, st));
        const int first = s->steps;
        session_decode(s, steps, st);
        EKV_CUDA(cudaMemcpyAsync(out, s->hist + (size_t)first * s->model->h,
                                 sizeof(float) * steps * s->model->h, cudaMemcpyDeviceToDevice, st));
    });
}

int ekv_session_profile_step(ekv_session_t s, float* kernel_ms, int capacity, int* n_kernels) {
    return guard([&] {
        require(s && kernel_ms && n_kernels, "ekv_session_profile_step: null argument");
        const int n = use_mega(s) ? 1 : 3 * s->model->cfg.num_layers + 1;
        require(capacity >= n, "ekv_session_profile_step: need room for " + std::to_string(n) +
                                   " kernel times");
        check_overflow(s, 1);
        require(s->steps + 1 <= s->cap, "decode history full");
        set_dev(s->model->ctx);
        cudaStream_t st = s->model->ctx->stream;
        if (s->user_len == 0 && s->steps == 0)
            EKV_CUDA(cudaMemsetAsync(s->xa, 0, sizeof(float) * s->model->h, st));
        if (use_mega(s)) {
            cudaEvent_t e0, e1;
            EKV_CUDA(cudaEventCreate(&e0));
            EKV_CUDA(cudaEventCreate(&e1));
            EKV_CUDA(cudaEventRecord(e0, st));
            launch_decode_mega(s->mega, s->model->ctx->num_sms, st);
            EKV_CUDA(cudaEventRecord(e1, st));
            EKV_CUDA(cudaEventSynchronize(e1));
            EKV_CUDA(cudaEventElapsedTime(&kernel_ms[0], e0, e1));
            cudaEventDestroy(e0);
            cudaEventDestroy(e1);
            s->user_len += 1;
            s->steps += 1;
            *n_kernels = 1;
            return;
        }
        std::vector<cudaEvent_t> ev(n + 1);
        for (auto& e : ev) EKV_CUDA(cudaEventCreate(&e));
        try {
            forward_chunk(s, s->xa, 1, s->hist, &s->state->step, st, ev.data());
            EKV_CUDA(cudaStreamSynchronize(st));
            for (int i = 0; i < n; ++i) EKV_CUDA(cudaEventElapsedTime(&kernel_ms[i], ev[i], ev[i + 1]));
        } catch (...) {
            for (auto& e : ev) cudaEventDestroy(e);
            throw;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        s->user_len += 1;
        s->steps += 1;
        *n_kernels = n;
    });
}

int ekv_session_user_kv(ekv_session_t s, int layer, void** k, void** v, int* cap) {
    return guard([&] {
        require(s && k && v && cap, "null argument");
        require(layer >= 0 && layer < s->model->cfg.num_layers, "layer out of range");
        *k = s->uk + (size_t)layer * s->ukv_layer();
        *v = s->uv + (size_t)layer * s->ukv_layer();
        *cap = s->cap;
    });
}

int ekv_collaborative_decode(ekv_session_t s, const float* user_emb, int U, int steps,
                             float* prefill_out, float* step_out) {
    return guard([&] {
        require(s && step_out && (U == 0 || user_emb), "collaborative_decode: null argument");
        require(steps >= 1, "collaborative_decode: steps must be >= 1");
        require(U >= 0, "collaborative_decode: negative user rows");
        ekv_model_s* m = s->model;
        set_dev(m->ctx);
        cudaStream_t st = m->ctx->stream;
        const int total = s->kv->S + U + steps;
        require(total <= m->cfg.max_positions,
                "position overflow: " + std::to_string(total) + " > max_positions " +
                    std::to_string(m->cfg.max_positions));
        session_reset(s, st);
        const size_t h = m->h;
        if (U > 0) {
            check_overflow(s, U);
            EKV_CUDA(cudaMemcpyAsync(s->emb, user_emb, sizeof(float) * U * h,
                                     cudaMemcpyHostToDevice, st));
            session_forward(s, s->emb, U, st);
            if (prefill_out)
                EKV_CUDA(cudaMemcpyAsync(prefill_out, s->pre_out, sizeof(float) * U * h,
                                         cudaMemcpyDeviceToHost, st));
        } else {
            EKV_CUDA(cudaMemsetAsync(s->xa, 0, sizeof(float) * h, st));
        }
        session_decode(s, steps, st);
        EKV_CUDA(cudaMemcpyAsync(step_out, s->hist, sizeof(float) * steps * h,
                                 cudaMemcpyDeviceToHost, st));
        EKV_CUDA(cudaStreamSynchronize(st));
    });
}


// ---------------------------------------------------------------- batched sessions
int ekv_batch_create(ekv_model_t m, ekv_kvctx_t c, int sessions, int max_rows, ekv_batch_t* out) {
    return guard([&] {
        require(m && c && out, "ekv_batch_create: null argument");
        require(c->model == m || (c->model->cfg.num_heads == m->cfg.num_heads &&
                                  c->model->cfg.head_dim == m->cfg.head_dim),
                "collaborative_decode: context dims do not match model; align with head pruning "
                "first");
        require((int)c->seg.size() == m->cfg.num_layers,
                "collaborative_decode: context has " + std::to_string(c->seg.size()) +
                    " layers, model has " + std::to_string(m->cfg.num_layers));
        require(sessions >= 1, "ekv_batch_create: sessions must be >= 1");
        require(max_rows >= 1, "ekv_batch_create: max_rows must be >= 1");
        require(m->h % 128 == 0, "batched decode: hidden size must be a multiple of 128",
                EKV_EUNSUPPORTED);
        for (int l = 0; l < m->cfg.num_layers; ++l)
            require(c->seg[l].S == 0 || batch_ctx_supported(d_of(m), c->seg[l].format, c->seg[l].group),
                    "batched decode: context layer " + std::to_string(l) + " format " +
                        std::to_string(c->seg[l].format) + " with head_dim " +
                        std::to_string(d_of(m)) + " not supported",
                    EKV_EUNSUPPORTED);
        set_dev(m->ctx);
        auto* b = new ekv_batch_s();
        b->model = m;
        b->kv = c;
        b->B = sessions;
        b->cap = max_rows;
        try {
            batch_alloc(b);
        } catch (...) {
            batch_free(b);
            delete b;
            throw;
        }
        m->refs++;
        c->refs++;
        *out = b;
    });
}

int ekv_batch_destroy(ekv_batch_t b) {
    return guard([&] {
        if (!b) return;
        cudaSetDevice(b->model->ctx->device);
        cudaStreamSynchronize(b->model->ctx->stream);
        if (b->graph) cudaGraphExecDestroy(b->graph);
        batch_free(b);
        ekv_kvctx_s* kv = b->kv;
        ekv_model_s* m = b->model;
        delete b;
        release_kvctx(kv);
        release_model(m);
    });
}

int ekv_batch_reset(ekv_batch_t b) {
    return guard([&] {
        require(b != nullptr, "null batch");
        set_dev(b->model->ctx);
        batch_reset(b, b->model->ctx->stream);
    });
}

int ekv_batch_info(ekv_batch_t b, int* sessions, int* rows, int* splits) {
    return guard([&] {
        require(b != nullptr, "null batch");
        if (sessions) *sessions = b->B;
        if (rows) *rows = b->rows;
        if (splits) {
            splits[0] = b->KSq;
            splits[1] = b->KSo;
            splits[2] = b->nsplit;
        }
    });
}

int ekv_batch_forward(ekv_batch_t b, const float* emb_dev, int n, float* out_dev) {
    return guard([&] {
        require(b && (emb_dev || n == 0), "ekv_batch_forward: null argument");
        require(n >= 0, "ekv_batch_forward: negative row count");
        if (n == 0) return;
        set_dev(b->model->ctx);
        cudaStream_t st = b->model->ctx->stream;
        const int r0 = b->rows;
        batch_forward(b, emb_dev, n, n, st);
        if (out_dev)
            EKV_CUDA(cudaMemcpyAsync(out_dev, b->hist + (size_t)r0 * b->B * b->model->h,
                                     sizeof(float) * n * b->B * b->model->h, cudaMemcpyDeviceToDevice, st));
    });
}

int ekv_batch_decode(ekv_batch_t b, int steps, float* out_dev) {
    return guard([&] {
        require(b != nullptr, "null batch");
        set_dev(b->model->ctx);
        cudaStream_t st = b->model->ctx->stream;
        const int r0 = b->rows;
        batch_decode(b, steps, st);
        if (out_dev)
            EKV_CUDA(cudaMemcpyAsync(out_dev, b->hist + (size_t)r0 * b->B * b->model->h,
                                     sizeof(float) * steps * b->B * b->model->h, cudaMemcpyDeviceToDevice,
                                     st));
    });
}

int ekv_batch_profile_row(ekv_batch_t b, float* kernel_ms, int capacity, int* n_kernels) {
    return guard([&] {
        require(b && kernel_ms && n_kernels, "ekv_batch_profile_row: null argument");
        const int L = b->model->cfg.num_layers;
        const int n = 5 * L + 2;
        require(capacity >= n, "ekv_batch_profile_row: need room for " + std::to_string(n) + " kernel times");
        batch_check(b, 1);
        set_dev(b->model->ctx);
        cudaStream_t st = b->model->ctx->stream;
        std::vector<cudaEvent_t> ev(n + 1);
        for (auto& e : ev) EKV_CUDA(cudaEventCreate(&e));
        try {
            batch_row(b, st, ev.data());
            EKV_CUDA(cudaStreamSynchronize(st));
            for (int i = 0; i < n; ++i) EKV_CUDA(cudaEventElapsedTime(&kernel_ms[i], ev[i], ev[i + 1]));
        } catch (...) {
            for (auto& e : ev) cudaEventDestroy(e);
            throw;
        }
        for (auto& e : ev) cudaEventDestroy(e);
        b->user_len += 1;
        b->rows += 1;
        *n_kernels = n;
    });
}

int ekv_collaborative_decode_batch(ekv_batch_t b, const float* user_emb, int U, int steps,
                                   float* prefill_out, float* step_out) {
    return guard([&] {
        require(b && step_out && (U == 0 || user_emb), "collaborative_decode: null argument");
        require(steps >= 1, "collaborative_decode: steps must be >= 1");
        require(U >= 0, "collaborative_decode: negative user rows");
        ekv_model_s* m = b->model;
        set_dev(m->ctx);
        cudaStream_t st = m->ctx->stream;
        const int total = b->kv->S + U + steps;
        require(total <= m->cfg.max_positions,
                "position overflow: " + std::to_string(total) + " > max_positions " +
                    std::to_string(m->cfg.max_positions));
        require(U + steps <= b->cap, "session full: " + std::to_string(U + steps) +
                                         " rows > capacity " + std::to_string(b->cap));
        batch_reset(b, st);
        const size_t h = m->h, B = b->B;
        if (U > 0) {
            EKV_CUDA(cudaMemcpyAsync(b->emb, user_emb, sizeof(float) * B * U * h, cudaMemcpyHostToDevice, st));
            batch_forward(b, b->emb, U, U, st);
            if (prefill_out)
                EKV_CUDA(cudaMemcpyAsync(prefill_out, b->hist, sizeof(float) * U * B * h,
                                         cudaMemcpyDeviceToHost, st));
        }
        batch_decode(b, steps, st);
        EKV_CUDA(cudaMemcpyAsync(step_out, b->hist + (size_t)U * B * h, sizeof(float) * steps * B * h,
                                 cudaMemcpyDeviceToHost, st));
        EKV_CUDA(cudaStreamSynchronize(st));
    });
}


// ---------------------------------------------------------------- Eq. 20 pipelined prefill
}  // extern "C"

namespace ekv {
// Layer-major forward of n user rows where layer l's attention waits on ready[l] (null =
// the layer is resident), then the decode state is advanced past the rows.  Shared by the
// host-upload (Eq. 20 over pinned host memory) and the event-driven (NCCL receive) entry
// points.  t_comp_ms (optional): per-layer compute re-measured by a kernel-by-kernel re-run
// with the context resident (diagnostic: doubles the work, so only when asked for).
void streamed_forward(ekv_session_s* s, const float* emb_dev, int n, float* out_dev,
                      cudaEvent_t* ready, cudaEvent_t start_ev, cudaEvent_t end_ev,
                      float* t_comp_ms) {
    ekv_model_s* m = s->model;
    ekv_ctx_s* c = m->ctx;
    const int L = m->cfg.num_layers;
    cudaStream_t st = c->stream;
    const int prev_len = s->user_len;
    float* scratch = nullptr;
    std::vector<cudaEvent_t> lev;
    auto cleanup = [&] {
        if (scratch) cudaFreeAsync(scratch, st);
        for (auto& e : lev)
            if (e) cudaEventDestroy(e);
    };
    try {
        EKV_CUDA(cudaMallocAsync((void**)&scratch, sizeof(float) * 2 * n * m->h, st));
        if (start_ev) EKV_CUDA(cudaEventRecord(start_ev, st));
        forward_layer_major(s, emb_dev, n, prev_len, st, ready, scratch, nullptr);
        if (end_ev) EKV_CUDA(cudaEventRecord(end_ev, st));
        if (out_dev)
            EKV_CUDA(cudaMemcpyAsync(out_dev, s->pre_out + (size_t)prev_len * m->h,
                                     sizeof(float) * n * m->h, cudaMemcpyDeviceToDevice, st));
        if (t_comp_ms) {
            // the same rows again, layer by layer with the context resident (rewrites the
            // same user-cache rows and outputs with identical values)
            lev.assign(L + 1, nullptr);
            for (auto& e : lev) EKV_CUDA(cudaEventCreate(&e));
            forward_layer_major(s, emb_dev, n, prev_len, st, nullptr, scratch, lev.data());
            EKV_CUDA(cudaStreamSynchronize(st));
            for (int l = 0; l < L; ++l) EKV_CUDA(cudaEventElapsedTime(&t_comp_ms[l], lev[l], lev[l + 1]));
        }
        // state: n more user rows; decode continues from the last row (xa[0]), step 0
        launch_advance(s->state, n, st);
        EKV_CUDA(cudaMemsetAsync(&s->state->step, 0, sizeof(int), st));
        EKV_CUDA(cudaMemcpyAsync(s->xa, scratch + (size_t)(n - 1) * m->h, sizeof(float) * m->h,
                                 cudaMemcpyDeviceToDevice, st));
        s->user_len += n;
        s->steps = 0;
    } catch (...) {
        cleanup();
        throw;
    }
    cleanup();
}
}  // namespace ekv

extern "C" {

int ekv_session_forward_pipelined(ekv_session_t s, const float* emb_dev, int n, float* out_dev,
                                  const ekv_layer_upload* uploads, int overlap, float* t_comm_ms,
                                  float* t_comp_ms, float* total_ms) {
    return guard([&] {
        require(s && emb_dev && uploads, "ekv_session_forward_pipelined: null argument");
        require(n >= 1, "ekv_session_forward_pipelined: n must be >= 1");
        ekv_model_s* m = s->model;
        ekv_ctx_s* c = m->ctx;
        const int L = m->cfg.num_layers, H = m->cfg.num_heads, d = d_of(m);
        check_overflow(s, n);
        set_dev(c);
        cudaStream_t st = c->stream, cp = c->copy;
        std::vector<cudaEvent_t> up(L + 1, nullptr), ready(L, nullptr), cs(2, nullptr);
        auto cleanup = [&] {
            for (auto* v : {&up, &ready, &cs})
                for (auto& e : *v)
                    if (e) cudaEventDestroy(e);
        };
        try {
            for (auto& e : up) EKV_CUDA(cudaEventCreate(&e));
            for (auto& e : cs) EKV_CUDA(cudaEventCreate(&e));
            // start both streams from the same point
            EKV_CUDA(cudaEventRecord(up[0], st));
            EKV_CUDA(cudaStreamWaitEvent(cp, up[0], 0));
            EKV_CUDA(cudaEventRecord(up[0], cp));
            for (int l = 0; l < L; ++l) {
                const ekv_layer_upload& u = uploads[l];
                const ekv_segment& sg = s->kv->seg[l];
                if (u.k_host && sg.S > 0) {
                    const size_t rows = (size_t)H * sg.S;
                    const size_t row_b = sg.format == EKV_KV_BF16 ? (size_t)d * 2 : (size_t)d * sg.format / 8;
                    require(u.v_host != nullptr, "upload: layer " + std::to_string(l) + " has K but no V");
                    EKV_CUDA(cudaMemcpyAsync((void*)sg.k, u.k_host, rows * row_b, cudaMemcpyHostToDevice, cp));
                    EKV_CUDA(cudaMemcpyAsync((void*)sg.v, u.v_host, rows * row_b, cudaMemcpyHostToDevice, cp));
                    if (sg.format != EKV_KV_BF16) {
                        require(u.k_scales_host && u.v_scales_host,
                                "upload: quantised layer " + std::to_string(l) + " needs scales");
                        const size_t sb = rows * (d / sg.group) * sizeof(float);
                        EKV_CUDA(cudaMemcpyAsync((void*)sg.k_scales, u.k_scales_host, sb, cudaMemcpyHostToDevice, cp));
                        EKV_CUDA(cudaMemcpyAsync((void*)sg.v_scales, u.v_scales_host, sb, cudaMemcpyHostToDevice, cp));
                    }
                    EKV_CUDA(cudaEventCreateWithFlags(&ready[l], cudaEventDisableTiming));
                    EKV_CUDA(cudaEventRecord(ready[l], cp));
                }
                EKV_CUDA(cudaEventRecord(up[l + 1], cp));
            }
            if (!overlap) {  // sequential reference schedule: every upload before any compute
                EKV_CUDA(cudaStreamWaitEvent(st, up[L], 0));
            }
            streamed_forward(s, emb_dev, n, out_dev, overlap ? ready.data() : nullptr, cs[0], cs[1],
                             t_comp_ms);
            EKV_CUDA(cudaStreamSynchronize(cp));
            EKV_CUDA(cudaStreamSynchronize(st));
            if (t_comm_ms)
                for (int l = 0; l < L; ++l) EKV_CUDA(cudaEventElapsedTime(&t_comm_ms[l], up[l], up[l + 1]));
            if (total_ms) EKV_CUDA(cudaEventElapsedTime(total_ms, up[0], cs[1]));
        } catch (...) {
            cleanup();
            throw;
        }
        cleanup();
    });
}

int ekv_session_forward_streamed(ekv_session_t s, const float* emb_dev, int n, float* out_dev,
                                 void* const* layer_ready) {
    return guard([&] {
        require(s && emb_dev, "ekv_session_forward_streamed: null argument");
        require(n >= 1, "ekv_session_forward_streamed: n must be >= 1");
        ekv_model_s* m = s->model;
        check_overflow(s, n);
        set_dev(m->ctx);
        std::vector<cudaEvent_t> ready(m->cfg.num_layers, nullptr);
        if (layer_ready)
            for (int l = 0; l < m->cfg.num_layers; ++l) ready[l] = (cudaEvent_t)layer_ready[l];
        streamed_forward(s, emb_dev, n, out_dev, ready.data(), nullptr, nullptr, nullptr);
    });
}

// ---------------------------------------------------------------- scheduler
int ekv_cache_source(int layer, double cost_local, double cost_peer, int boundary, int m,
                     int* source) {
    return guard([&] {
        require(source != nullptr, "null argument");
        require(layer >= 1 && layer <= m, "cache_source: layer " + std::to_string(layer) +
                                              " outside 1.." + std::to_string(m));
        *source = layer > boundary ? 2 : (cost_local <= cost_peer ? 0 : 1);
    });
}

int ekv_pipeline_schedule(const double* t_comm, const double* t_comp, int n, double* t_pip,
                          double* sequential_total, double* pipelined_total) {
    return guard([&] {
        require(n >= 1, "pipeline_schedule: empty layer list");
        require(t_comm && t_comp && t_pip && sequential_total && pipelined_total,
                "pipeline_schedule: null argument");
        for (int l = 0; l < n; ++l)
            require(t_comm[l] >= 0.0 && t_comp[l] >= 0.0, "pipeline_schedule: negative time");
        double prev = 0.0, pip = 0.0, seq = 0.0;
        for (int l = 0; l < n; ++l) {
            t_pip[l] = std::max(t_comm[l], prev);
            pip += t_pip[l];
            prev = t_comp[l];
        }
        for (int l = 0; l < n; ++l) seq += t_comm[l] + t_comp[l];
        *pipelined_total = pip + t_comp[n - 1];
        *sequential_total = seq;
    });
}

}  // extern "C"
