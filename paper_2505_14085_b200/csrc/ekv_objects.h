// Internal object model of the C ABI (not installed): the structs behind the
// opaque handles of include/ekv_capi.h, the error guard every entry point runs
// in, and the session routines shared by the translation units that implement
// the ABI (ekv_capi.cu: context/model/session/batch; ekv_pipeline.cu: stage 1+2
// and the device prefill / layer map).
#pragma once

#include <cuda.h>

#include <atomic>
#include <string>
#include <vector>

#include "ekv_batch.h"
#include "ekv_common.cuh"
#include "ekv_kernels.h"
#include "ekv_mega.h"

namespace ekv {

extern thread_local std::string g_err;  // message of the last failure on this thread

// Run an entry point body; map exceptions to (status, ekv_last_error()).
template <class F>
int guard(F&& f) {
    try {
        f();
        return EKV_OK;
    } catch (const Error& e) {
        g_err = e.what();
        return e.status;
    } catch (const std::bad_alloc&) {
        g_err = "host allocation failed";
        return EKV_ENOMEM;
    } catch (const std::exception& e) {
        g_err = e.what();
        return EKV_EINVAL;
    }
}

template <class T>
T* dalloc(size_t count) {
    void* p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMalloc(&p, count * sizeof(T));
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        throw Error(EKV_ENOMEM, "cudaMalloc of " + std::to_string(count * sizeof(T)) +
                                    " bytes failed: " + cudaGetErrorString(e));
    }
    return (T*)p;
}


// Stream-ordered allocation from the device's default memory pool (kept cached:
// ekv_ctx_create raises the pool's release threshold), for the objects created
// per request -- sessions, assembled contexts, prefill scratch -- so creating and
// destroying them costs no device-wide synchronisation.
template <class T>
T* dalloc_on(size_t count, cudaStream_t st) {
    void* p = nullptr;
    if (count == 0) count = 1;
    cudaError_t e = cudaMallocAsync(&p, count * sizeof(T), st);
    if (e != cudaSuccess) {
        (void)cudaGetLastError();
        throw Error(EKV_ENOMEM, "cudaMallocAsync of " + std::to_string(count * sizeof(T)) +
                                    " bytes failed: " + cudaGetErrorString(e));
    }
    return (T*)p;
}

}  // namespace ekv

using ekv::DevState;
using ekv::MegaArgs;

// Lifetimes: every handle is reference counted.  The destroy call drops the
// caller's reference and each dependent object holds one on what it uses
// (model -> ctx, kvctx -> model, session / batch -> model + kvctx), so handles
// may be destroyed in any order (garbage-collected host wrappers do).
struct ekv_ctx_s {
    std::atomic<int> refs{1};
    int device = 0;
    int num_sms = 148;
    cudaStream_t stream = nullptr;
    cudaStream_t capture = nullptr;  // graphs are captured here, launched on `stream`
    cudaStream_t copy = nullptr;     // context uploads of the pipelined prefill (Eq. 20)
    cudaStream_t aux = nullptr;      // side work off the critical path (pack checksums)
    bool own_stream = false;
    // scratch of ekv_decode_attention (split-KV partials + merge counters), grown on demand
    float* attn_ws = nullptr;
    size_t attn_ws_n = 0;
    unsigned* attn_ctr = nullptr;
    size_t attn_ctr_n = 0;
    // general scratch of the stage 1+2 entry points (ekv_pipeline.cu), grown on demand
    void* scratch = nullptr;
    size_t scratch_n = 0;
};

struct ekv_model_s {
    std::atomic<int> refs{1};
    ekv_ctx_s* ctx = nullptr;
    ekv_model_config cfg{};
    int h = 0;
    uint16_t* weights = nullptr;  // per layer: [3h][h] wqkvT then [h][h] woT
    float* gamma = nullptr;
    float* bias = nullptr;
    uint16_t* pos = nullptr;
    size_t layer_elems() const { return (size_t)4 * h * h; }
    uint16_t* wqkvT(int l) const { return weights + (size_t)l * layer_elems(); }
    uint16_t* woT(int l) const { return wqkvT(l) + (size_t)3 * h * h; }
};

struct ekv_kvctx_s {
    std::atomic<int> refs{1};
    ekv_model_s* model = nullptr;
    int S = 0, group = 0;
    std::vector<int> fmt;
    std::vector<ekv_segment> seg;
    std::vector<void*> allocs;
};

struct ekv_session_s {
    ekv_model_s* model = nullptr;
    ekv_kvctx_s* kv = nullptr;
    int cap = 0;                   // user/generated rows
    uint16_t* uk = nullptr;        // [L][H][cap][d]
    uint16_t* uv = nullptr;
    float* xa = nullptr;           // [8][h]
    float* xb = nullptr;           // [8][h]
    float* q = nullptr;            // [8][h]
    float* emb = nullptr;          // [cap][h] staged user embeddings
    float* pre_out = nullptr;      // [cap][h] prefill outputs by user row
    float* hist = nullptr;         // [cap][h] decode-step outputs by step
    DevState* state = nullptr;
    float* ws = nullptr;
    unsigned* counters = nullptr;
    int user_len = 0;              // host mirror of state->user_len
    int steps = 0;                 // host mirror of state->step
    cudaGraphExec_t step_graph = nullptr;
    int64_t graph_kernels = 0;
    // persistent decode-step kernel (k_decode_mega.cu)
    int path = 0;                  // 0 = megakernel when supported, 1 = per-layer graph
    bool mega_ok = false;
    uint64_t* mega_ll = nullptr;     // tagged words of the dataflow (MegaArgs::ll_*)
    unsigned* mega_sync = nullptr;   // [0] launch epoch
    MegaArgs mega{};
    // tensor-core prefill projections (R >= 2 rows; h % 128 == 0)
    bool tc_prefill = false;
    uint16_t* pxhl = nullptr;      // [2][8][h] bf16 hi / lo operand
    float* ppart = nullptr;        // [max(KSq*3h, KSo*h)][8] split-K partials
    float* pctx = nullptr;         // [pchunk][H][splits][d+4] context partials of the prefill rows (K10)
    int pKSq = 1, pKSo = 1;
    int pchunk = 8;                // rows per tensor-core chunk of the layer-major forward
    CUtensorMap pmap_w{}, pmap_x{};
    size_t ukv_layer() const { return (size_t)model->cfg.num_heads * cap * model->cfg.head_dim; }
};


namespace ekv {

inline void set_dev(ekv_ctx_s* c) { EKV_CUDA(cudaSetDevice(c->device)); }
inline int d_of(const ekv_model_s* m) { return m->cfg.head_dim; }

// Layer-major forward of n rows of a session (all rows through layer l before
// l + 1); ready[l] (optional) gates layer l's attention; lev[l] (optional)
// timestamps layer l; layer_out (optional, fp32 [L][n][h]) receives every
// layer's output rows (the reference KVCache::layer_outputs of forward_rows).
void forward_layer_major(ekv_session_s* s, const float* emb, int n, int base0, cudaStream_t st,
                         const cudaEvent_t* ready, float* scratch, cudaEvent_t* lev,
                         float* layer_out = nullptr);
void session_reset(ekv_session_s* s, cudaStream_t st);
// forward_layer_major + state advance of n user rows; ready[l] gates layer l
// (null = resident); start/end events optional; t_comp_ms (optional) re-measures
// each layer's compute kernel by kernel (diagnostic, doubles the work).
void streamed_forward(ekv_session_s* s, const float* emb_dev, int n, float* out_dev, cudaEvent_t* ready,
                      cudaEvent_t start_ev, cudaEvent_t end_ev, float* t_comp_ms);
void release_ctx(ekv_ctx_s* c);
void release_model(ekv_model_s* m);
void release_kvctx(ekv_kvctx_s* c);
void check_overflow(ekv_session_s* s, int n);

}  // namespace ekv
