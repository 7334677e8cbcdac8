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
constexpr int kMaxAlignLayers = 64;
// Kernel parameters of K1 (by value, __grid_constant__).
struct AlignArgs {
    int m_layers, S, h_c, n_cols;
    int fold;                        // 0: colsq [m][n_cols]; d_c: colsq [d_c] over heads and layers
    double* colsq;
    int x_index[kMaxAlignLayers];    // layer coordinate of group i in the X / W_Q tensor maps
    int w_index[kMaxAlignLayers];
    // fused K2 (warps 2-3): kcolsq[c] += sum over every row of every k[i] of K[row][c]^2
    double* kcolsq;
    int k_layers, d_c;
    int64_t k_rows;                  // rows (H*S) per layer
    const uint16_t* k[kMaxAlignLayers];
};
// Host description of one K1 launch.  X layers live at X + x_index[i]*x_stride
// ([S][h_c] each, stride 0 = S*h_c), W_Q^T layers at WqT + w_index[i]*w_stride
// ([n_cols][h_c], stride 0 = n_cols*h_c); null index tables mean 0..m-1.
struct AlignLaunch {
    const void* X = nullptr;
    int64_t x_stride = 0;
    const int* x_index = nullptr;
    const void* WqT = nullptr;
    int64_t w_stride = 0;
    const int* w_index = nullptr;
    int m = 0, S = 0, h_c = 0, n_cols = 0;
    int fold = 0;
    double* colsq = nullptr;
    double* kcolsq = nullptr;   // null: no fused K norms
    const void* const* k = nullptr;
    int k_layers = 0, d_c = 0;
    int64_t k_rows = 0;
};
void launch_align(const AlignLaunch& p, cudaStream_t st);

// ---- small device utilities (k_util.cu) ------------------------------------------
// Reference ranking (head_prune.cpp:98-107) on the device: score_c =
// sqrt(q[c])*sqrt(k[c]) in fp64, stable descending order, keep the first
// `retained`, listed ascending -> kept[retained]; margin = (s[r-1]-s[r])/s[r-1].
void launch_rank_channels(const double* q, const double* k, int d_c, int retained, int* kept,
                          double* margin, cudaStream_t st);
void launch_f32_to_bf16(const float* src, uint16_t* dst, int64_t n, cudaStream_t st);
void launch_f32_to_f64(const float* src, double* dst, int64_t n, cudaStream_t st);
// x0[r] = gamma * (emb[r] + pos[p0 + r]) + bias (the layer-0 input transform, fp32)
void launch_input_transform(const float* emb, const float* gamma, const float* bias,
                            const uint16_t* pos, int p0, int n, int h, float* x0, cudaStream_t st);
// fp64 column sums of squares of an fp64 matrix [rows][d] (accumulated)
void launch_colsq_f64(const double* m, int64_t rows, int d, double* colsq, cudaStream_t st);
// exact dequantisation to fp64: dst = code * (double)scale
void launch_kv_dequant_f64(const void* codes, const float* scales, int64_t rows, int d_e, int bits,
                           int group, double* dst, cudaStream_t st);
// reference-order fp64 matmul (bit-identical to matrix.cpp:19-36): out[n][m] = a[n][k] b[k][m]
void launch_matmul_f64(const double* a, const double* b, int n, int k, int m, double* out,
                       cudaStream_t st);
// segment_attention_prefix in fp64 (cache_merge.cpp:12-38); logits scratch [n];
// stats = {sigma, shift}
void launch_segment_attention_f64(const double* q, const double* k, const double* v, int n, int d,
                                  int vd, double* logits, double* o, double* stats, cudaStream_t st);

}  // namespace ekv
