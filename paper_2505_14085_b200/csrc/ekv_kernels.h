// Internal launch interface of the sm_100a kernels (not part of the C ABI).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace ekv {

// Device-resident decode state of a session (read by the graph's kernels).
struct DevState {
    int user_len;  // rows in the user/generated cache before this forward
    int step;      // decode-step counter (history row)
};

void launch_fill_uniform_bf16(void* dst, int64_t n, uint64_t seed, uint64_t stream_id, double lo,
                              double hi, cudaStream_t st);
// Batched compression: one launch over up to kMaxCompressJobs (src, codes,
// scales) triples sharing rows / d_c / kept / d_e / bits / group.
struct CompressJob {
    const void* src;
    void* codes;
    float* scales;
};
constexpr int kMaxCompressJobs = 128;
struct CompressJobs {
    CompressJob job[kMaxCompressJobs];
};
void launch_kv_compress_jobs(const CompressJob* jobs, int n_jobs, int64_t rows, int d_c,
                             const int* kept, int d_e, int bits, int group, cudaStream_t st);
void launch_kv_compress(const void* src, int64_t rows, int d_c, const int* kept, int d_e, int bits,
                        int group, void* codes, float* scales, cudaStream_t st);
void launch_kv_gather(const void* src, int64_t rows, int d_c, const int* kept, int d_e, void* dst,
                      cudaStream_t st);
void launch_gather_columns(const void* src, int64_t rows, int d_c, const int* kept, int d_e,
                           int elem_bytes, void* dst, cudaStream_t st);
void launch_kv_dequant(const void* codes, const float* scales, int64_t rows, int d_e, int bits,
                       int group, void* dst, cudaStream_t st);
void launch_kv_colnorm(const void* K, int64_t rows, int d_c, double* colsq, cudaStream_t st);
void launch_layer_match(const double* edge_outs, int me, int ce, const double* cloud_outs, int nc, int cc,
                        int n, double* scale, double* gram, double* centred, double* self_hsic,
                        double* cosflat, int* zero_row, double* hsic, double* corr, int* zero_var,
                        cudaStream_t st);

// ---- K4 decode attention -------------------------------------------------
struct AttnArgs {
    int R, H, D;
    const float* q;  // [R][H][D]
    // context segment (head-major [H][S][...])
    int fmt, S, group;
    const void* ck;
    const void* cv;
    const float* cks;
    const float* cvs;
    // user segment bf16 [H][ucap][D]; visible rows of query r = base + r + 1,
    // base = *user_base_dev if non-null else user_base.
    const uint16_t* uk;
    const uint16_t* uv;
    int ucap;
    const int* user_base_dev;
    int user_base;
    // outputs
    float* out;  // [R][H][D]
    float* lse;  // [R][H] or null
    // workspace (from attn_workspace_bytes)
    float* ws;
    unsigned* counters;  // [R*H], zero on entry, zero on exit
};
// Context items per (row, head): chosen from S, H, R; user items cover ucap rows.
// Workspace = R*H*(ctx items + user items)*(D+2) floats.
int attn_items(int R, int H, int S, int* rows_per_item);
int attn_user_items(int ucap);
void launch_decode_attention(const AttnArgs& a, cudaStream_t st);

// ---- K5 projections (GEMV / skinny GEMM over R <= 8 rows) ---------------------
struct GemvArgs {
    int N, K, R;
    const uint16_t* W;  // [N][K] bf16 (out-feature major)
    const float* x;     // [R][K] fp32 input rows
    // optional input transform (layer 0): x' = gamma*(x + pos[p0 + r]) + bias
    const float* gamma;
    const float* bias;
    const uint16_t* pos;      // [max_pos][K] bf16
    int pos_offset;           // p0 = pos_offset + *pos_base_dev (or + pos_base)
    const int* pos_base_dev;
    int pos_base;
    // epilogue: mode 0 -> y[r][n]; mode 1 -> QKV split into q / user K / user V
    int mode;
    float* y;
    float* y_hist;            // mode 0 extra copy: y_hist[(*hist_row_dev + r)][n] if non-null
    const int* hist_row_dev;
    int qkv_d, qkv_H;         // mode 1: N = 3*H*d
    float* q_out;             // [R][H*d]
    uint16_t* uk;             // [H][ucap][d]
    uint16_t* uv;
    int ucap;
    const int* user_base_dev; // row written = base + r
    int user_base;
};
void launch_gemv(const GemvArgs& a, cudaStream_t st);

// advance the device decode state: user_len += n, step += 1
void launch_advance(DevState* s, int n, cudaStream_t st);

// ---- K1 alignment GEMM (tcgen05 / TMEM / TMA) --------------------------------
void launch_align_qnorm(const void* X, const void* WqT, int S, int h_c, int n_cols, double* colsq,
                        cudaStream_t st);

}  // namespace ekv
