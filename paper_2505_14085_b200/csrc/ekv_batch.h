// Launch interface of the batched-session decode kernels (k_batch.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ekv_kernels.h"

namespace ekv {

struct BatchXprep {
    int mode;              // 0: layer-0 input transform of xin; 1: sum partials; 2: final output
    int B, h, KS;
    const float* part;     // [KS][B][h] split-K partials of the output projection
    float* xin;            // [B][h] step input (mode 0 reads, mode 2 writes)
    float* hist;           // [rows][B][h] output rows (mode 2), row = state->step
    const float* gamma;
    const float* bias;
    const uint16_t* pos;   // [max_pos][h]
    int pos_offset;        // S: position of user row u is S + u
    int pos_per_row;       // 1: row b sits at position S + user_len + row0 + b (prefill rows of one session)
    int row0;
    const DevState* state;
    uint16_t* xhl;         // [2][B][h] bf16 hi, lo (projection operand)
};

// Prefill projections on the tensor cores (R >= 2 rows of one session): the
// finish step of K9's split-K partials.  mode 0 (QKV, N = 3h): q -> q_out
// fp32 [R][h], k/v rounded to bf16 into the user cache rows user_len + r
// (layout [H][cap][d]); mode 1 (out-proj, N = h): y [R][h] and, if y_hist,
// y_hist[user_len + r].
struct PrefillFinish {
    int mode, R, N, KS, H, d, cap;
    int row0;              // rows of this chunk start at user_len + row0
    const float* part;     // [KS][R][N]
    float* q_out;
    uint16_t* uk;
    uint16_t* uv;
    float* y;
    float* y_hist;
    const DevState* state;
};
void launch_prefill_finish(const PrefillFinish& a, cudaStream_t st);

struct BatchCtxAttn {
    int B, H, D, S, nsplit, KS, n_qkv;
    const float* qkv;      // [KS][B][n_qkv] partials of the QKV projection (q at column 0)
    float* part;           // [B][H][nsplit][D + 4]  (m, l, -, -, o[D]) unnormalised
    // finalisation of this row's q / k / v (optional, qfin != null): q summed into
    // qfin [B][h]; k, v summed, rounded to bf16 and appended to the user caches
    float* qfin;
    uint16_t* uk;          // [B][L][H][cap][D]
    uint16_t* uv;
    int L, layer, cap;
    const DevState* state;
};

struct BatchUserMerge {
    int B, H, D, L, layer, cap, KS, n_qkv, nsplit;
    // prefill (R rows of ONE session, requires qfin): item b is row b of the chunk, whose
    // k / v sit at cache row user_len + row0 + b of the single cache at uk / uv (b-stride 0);
    // causal: row b attends to the cache rows before it and to itself
    int prefill, row0;
    const float* qkv;      // [KS][B][3h]
    const float* qfin;     // non-null: q from qfin [B][h], k / v already appended by K10
    const float* part;     // context partials (nsplit may be 0)
    uint16_t* uk;          // [B][L][H][cap][D]
    uint16_t* uv;
    const DevState* state;
    uint16_t* xhl;         // [2][B][h] attention output hi, lo
};

CUtensorMap make_map_2d(const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t inner,
                        uint64_t rows, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw);
CUtensorMap make_map_1d(const void* base, CUtensorMapDataType dt, uint64_t n, uint32_t box);
CUtensorMap make_map_3d_bf16(const void* base, uint64_t inner, uint64_t rows, uint64_t depth,
                             uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw);

int batch_proj_bn(int B);
int batch_proj_splits(int N_out, int K, int B, int num_sms);
void launch_batch_proj(const CUtensorMap& map_w, int w_row0, int N_out, int K, const CUtensorMap& map_x,
                       int B, int KS, float* out, cudaStream_t st);
void launch_batch_xprep(const BatchXprep& a, cudaStream_t st);
int batch_ctx_splits(int S, int H, int B, int num_sms);
// tensor maps of one context layer: bf16 -> k, v tiles [H*S][D] (SW128);
// int8 -> k, v codes [H*S][D] bytes and ks, vs row scales [H*S] fp32 (1-D)
struct BatchCtxMaps {
    int fmt;
    CUtensorMap k, v, ks, vs;
};
bool batch_ctx_supported(int D, int fmt, int group);
void launch_batch_ctx_attn(const BatchCtxMaps& maps, const BatchCtxAttn& a, cudaStream_t st);
void launch_batch_user_merge(const BatchUserMerge& a, cudaStream_t st);

}  // namespace ekv
