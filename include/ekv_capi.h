/*
 * ekv_capi.h -- the C-ABI drop-in boundary of the B200 CE-LSLM KV-reuse path.
 *
 * The reference (/root/reference/proj) exposes this path as free C++
 * functions in namespace edgekv, compiled into the static library
 * edgekv_core (proj/src/CMakeLists.txt:1-13); it has no FFI or plugin
 * registry.  Each entry point below names the reference interface it
 * replaces (file:line under /root/reference/proj).  The C++ mirror of the
 * reference interface (include/edgekv_b200.hpp) and the Python host layer
 * (paper_2505_14085_b200/) sit on top of this ABI; INTEGRATION.md shows the
 * binding a reference maintainer would add.
 *
 * Conventions
 *  - Plain pointers and sizes only.  "dev" = device pointer (caller-owned,
 *    on the context's device), "host" = host pointer.  bf16 tensors are
 *    passed as void* / uint16_t* holding IEEE bfloat16 bits.
 *  - Every call returns EKV_OK (0) or a negative ekv_status; the message of
 *    the last failure on the calling thread is ekv_last_error().  Message
 *    substrings match the reference's std::invalid_argument texts where the
 *    reference has one (e.g. "empty segment", "missing layer 3",
 *    "align with head pruning", "position overflow").
 *  - Device work is asynchronous on the context's stream (ekv_ctx_create)
 *    unless the function says it synchronises.  No entry point allocates
 *    device memory on the hot path; buffers are sized at create time.
 *  - There is no CPU fallback: on a host without a B200 (sm_100) every
 *    compute entry point fails with EKV_ENODEV.
 */
#ifndef EKV_CAPI_H
#define EKV_CAPI_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif
#if defined(__GNUC__)
#pragma GCC visibility push(default)
#endif

#define EKV_ABI_VERSION 1

typedef enum {
    EKV_OK = 0,
    EKV_EINVAL = -1,      /* bad argument (std::invalid_argument in the reference) */
    EKV_ECUDA = -2,       /* CUDA runtime/driver failure */
    EKV_ENOMEM = -3,      /* device allocation failed */
    EKV_ENODEV = -4,      /* no sm_100 device */
    EKV_EUNSUPPORTED = -5 /* shape/format outside the compiled kernels */
} ekv_status;

/* KV storage formats of a context layer (AssembledContext provenance:
 * local layers are bf16, cloud layers arrive compressed). */
typedef enum { EKV_KV_BF16 = 16, EKV_KV_INT8 = 8, EKV_KV_INT4 = 4 } ekv_kv_format;

typedef struct ekv_ctx_s* ekv_ctx_t;         /* device, stream, workspace          */
typedef struct ekv_model_s* ekv_model_t;     /* edge model weights (Model)          */
typedef struct ekv_kvctx_s* ekv_kvctx_t;     /* assembled context (AssembledContext)*/
typedef struct ekv_session_s* ekv_session_t; /* user cache + decode state          */
typedef struct ekv_batch_s* ekv_batch_t;     /* B sessions over one shared context */

/* ------------------------------------------------------------------ */
/* Context, errors, utilities                                          */
/* ------------------------------------------------------------------ */
int ekv_abi_version(void);
const char* ekv_last_error(void);
/* stream: a cudaStream_t to run on, or NULL for a context-owned stream. */
int ekv_ctx_create(int device, void* stream, ekv_ctx_t* out);
int ekv_ctx_destroy(ekv_ctx_t ctx);
int ekv_ctx_stream(ekv_ctx_t ctx, void** stream);
int ekv_ctx_synchronize(ekv_ctx_t ctx);
/* Number of kernels this library has launched through ctx (graph replays
 * count every kernel node). */
int ekv_ctx_kernel_launches(ekv_ctx_t ctx, int64_t* count);

/* Device memory helpers for hosts that do not link the CUDA runtime (the C++
 * mirror): allocation on the context's device from the device's pooled
 * stream-ordered allocator (no device-wide synchronisation per allocation;
 * ekv_device_free releases after the context stream's queued work), and
 * synchronous copies on the context stream.  kind: 0 host->device,
 * 1 device->host, 2 device->device. */
int ekv_device_alloc(ekv_ctx_t ctx, size_t bytes, void** out);
int ekv_device_free(ekv_ctx_t ctx, void* p);
int ekv_memset(ekv_ctx_t ctx, void* dst_dev, int value, size_t bytes);
int ekv_copy(ekv_ctx_t ctx, void* dst, const void* src, size_t bytes, int kind);

/* Counter-hash synthetic data (bit-identical to oracle ekvo_fill_uniform_bf16):
 * dst[i] = bf16_rn(lo + (hi-lo) * ((mix(mix(seed,stream_id), i) >> 11) * 2^-53)),
 * mix = Rng::mix (rng.hpp:35-40). */
int ekv_fill_uniform_bf16(ekv_ctx_t ctx, void* dst_dev, int64_t n, uint64_t seed,
                          uint64_t stream_id, double lo, double hi);

/* ------------------------------------------------------------------ */
/* Stage 1: layer-alignment map and projection into edge head geometry */
/* ------------------------------------------------------------------ */

/* generate_embeddings (transformer.cpp:308-317; Rng rng.hpp:13-45), host: row i
 * is drawn from mt19937_64(Rng::mix(seed, i)), value = -1 + 2*((u >> 11) * 2^-53),
 * so row i at width h is a prefix of row i at any larger width.  out host fp64
 * [n][h].  The reference's probe / context / user inputs (sim.cpp:101-104,
 * 130-132, 163). */
int ekv_generate_embeddings(uint64_t seed, int n, int h, double* out);

/* PruneSpec::from_lambda (head_prune.cpp:14-22): retained = floor((1-l)*d + 1e-9). */
int ekv_prune_retained(double lambda, int head_dim, int* retained);

/* K1 (tcgen05/TMEM GEMM fed by TMA): Q = X * Wq for each of m matched cloud
 * layers (a grouped GEMM: the reference stacks every distinct matched layer,
 * sim.cpp:236-253), reduced in the epilogue to per-column sums of squares;
 * Q is never stored.  Replaces project_qkv (transformer.cpp:133-152) as
 * called from build_deep_kv (sim.cpp:240-253) plus the Q column-norm loop of
 * select_channels (head_prune.cpp:92-97).
 *   X    dev bf16 [m][S][h_c]        (cloud hidden state entering layer lc)
 *   WqT  dev bf16 [m][n_cols][h_c]   (n_cols = H*d_c; row hd*d_c+c = W_Q[lc][hd](:,c))
 *   colsq dev fp64 [m][n_cols]       ACCUMULATED (+=), fp32 per tile -> fp64.
 * Requires S % 128 == 0, n_cols % 256 == 0, h_c % 64 == 0. */
int ekv_align_qnorm(ekv_ctx_t ctx, const void* X_dev, const void* WqT_dev, int m, int S, int h_c,
                    int n_cols, double* colsq_dev);

/* K2: per-column sums of squares of cached cloud K (saves recomputing
 * K = X*W_K; K half of head_prune.cpp:92-97).  K dev bf16 [rows][d_c]
 * (rows = H*S of one layer), colsq dev fp64 [d_c] ACCUMULATED (+=). */
int ekv_kv_colnorm(ekv_ctx_t ctx, const void* K_dev, int64_t rows, int d_c, double* colsq_dev);

/* Host ranking with the reference rule (head_prune.cpp:98-107): score_c =
 * sqrt(q_colsq[c]) * sqrt(k_colsq[c]); stable descending sort; keep the
 * first `retained`; sort kept ascending.  cut_margin (optional) = relative
 * score gap across the cut, (s[r-1]-s[r]) / s[r-1], reported for near-tie
 * audits.  All pointers host. */
int ekv_rank_channels(const double* q_colsq, const double* k_colsq, int d_c, int retained,
                      int* kept, double* cut_margin);

/* Layer map (match_layers, layer_match.cpp:166-228) over probe outputs in HOST
 * memory [me][n][ce] / [nc][n][cc] (fp64): uploaded and computed by K7 on the
 * context's device (bit-identical to the reference).  best[le] = matched cloud
 * layer or -1; cka/rsa outputs [me][nc].  Synchronises. */
int ekv_match_layers(ekv_ctx_t ctx, const double* edge_outs, int me, int ce, const double* cloud_outs,
                     int nc, int cc, int n, double theta_cka, double theta_rsa, double* cka,
                     double* rsa, int* best);
/* K7: the same layer map on the device.  edge_outs / cloud_outs are DEVICE
 * buffers (the probe-prefill outputs, fp64); cka / rsa / best are host arrays.
 * Bit-identical to match_layers (layer_match.cpp:166-228): fp64 in the
 * reference's operation order.  Same errors and messages.  n <= 256.
 * Synchronises the context's stream. */
int ekv_match_layers_dev(ekv_ctx_t c, const double* edge_outs, int me, int ce,
                         const double* cloud_outs, int nc, int cc, int n, double theta_cka,
                         double theta_rsa, double* cka, double* rsa, int* best);

/* fp64 per-column sums of squares of an fp64 matrix (dev [rows][d] -> dev
 * colsq[d], ACCUMULATED): the column-norm loop of select_channels
 * (head_prune.cpp:92-97) for callers that hold Q / K in fp64 (the C++ mirror). */
int ekv_colsq_f64(ekv_ctx_t ctx, const double* m_dev, int64_t rows, int d, double* colsq_dev);

/* ------------------------------------------------------------------ */
/* Device prefill, layer map and deep-KV construction (whole ops)      */
/* ------------------------------------------------------------------ */

/* prefill (transformer.cpp:244-251) = forward_rows with PositionKind::context over
 * an empty KVCache (transformer.cpp:175-242), on the device: n rows at positions
 * 0..n-1 through every layer of the model.  Outputs (device, each may be NULL):
 *   layer_out fp32 [L][n][h]  the per-layer outputs (KVCache layer_outputs);
 *   x0        fp32 [n][h]     gamma*(emb+pos)+b, the hidden state entering layer 0
 *                             (build_deep_kv's input of cloud layer 0, sim.cpp:224-234);
 *   k, v      bf16 [L][H][n][d] the rows' KV cache (KVCache keys / values).
 * emb fp32 [n][h] on the device.  Synchronises. */
int ekv_prefill(ekv_model_t m, const float* emb_dev, int n, float* layer_out_dev, float* x0_dev,
                void* k_dev, void* v_dev);

/* forward_rows (transformer.cpp:175-242) on the device: n new rows on top of the
 * rows already cached in `cached` (an assembled context of this model's geometry;
 * NULL = an empty cache, i.e. ekv_prefill), positions S..S+n-1.  Outputs as
 * ekv_prefill (k / v receive the NEW rows' cache entries, [L][H][n][d]). */
int ekv_forward_rows(ekv_model_t m, ekv_kvctx_t cached, const float* emb_dev, int n,
                     float* layer_out_dev, float* x0_dev, void* k_dev, void* v_dev);

/* The reference's fp64 arithmetic on the device, for callers that need its bits
 * (the C++ mirror's project_qkv / segment_attention):
 *   ekv_matmul_f64: out[n][m] = a[n][k] * b[k][m] (dev fp64, row-major), every
 *     entry accumulated from 0.0 left to right with separate IEEE multiply and add
 *     -- bit-identical to matmul (matrix.cpp:19-36) built without FMA;
 *   ekv_segment_attention_f64: segment_attention (cache_merge.cpp:12-57) of one
 *     query q[d] over k[n][d], v[n][vd] (dev fp64): o[vd] (dev), sigma and shift
 *     (host) = the reference's (Sigma exp(l - max), max) pair; exp() is CUDA's
 *     (<= 1 ulp from libm), everything else in the reference's order.  Synchronises. */
int ekv_matmul_f64(ekv_ctx_t ctx, const double* a_dev, const double* b_dev, int n, int k, int m,
                   double* out_dev);
int ekv_segment_attention_f64(ekv_ctx_t ctx, const double* q_dev, const double* k_dev,
                              const double* v_dev, int n, int d, int vd, double* o_dev,
                              double* sigma, double* shift);

/* Artifacts::deep_match (sim.cpp:100-122) on the device: probe prefill of the edge
 * and the cloud model (n probe rows each, fp32 on the device: the reference's
 * generate_embeddings(Rng::mix(seed, 0x9B0BE), n, h)), K7 match_layers over the
 * per-layer outputs, then the map of the deep edge layers [M - deep_layers, M):
 * deep_map[i] = matched cloud layer of edge layer M - deep_layers + i (host int).
 * cka / rsa (host fp64 [M][N]) and best (host int [M], -1 = unmatched) may be NULL.
 * Error: "ce_lslm: edge layer N has no matched cloud layer under the configured
 * thresholds" (sim.cpp:113-115).  Both models on one context.  Synchronises. */
int ekv_deep_match(ekv_model_t edge, ekv_model_t cloud, const float* edge_probe_dev,
                   const float* cloud_probe_dev, int n, int deep_layers, double theta_cka,
                   double theta_rsa, int* deep_map, double* cka, double* rsa, int* best);

/* The cloud side of build_deep_kv: the m distinct matched cloud layers (sorted,
 * as the reference's std::set, sim.cpp:219-221), their input hidden states, W_Q
 * and cached K / V.  Layer i of X lives at x + x_index[i]*x_stride elements
 * ([S][h_c] bf16; stride 0 = S*h_c, x_index NULL = 0..m-1); its W_Q^T at
 * wq + wq_index[i]*wq_stride ([H*d_c][h_c] bf16, row hd*d_c+c = W_Q[lc][hd](:,c);
 * stride 0 = h_c*h_c -- an ekv_model's weights give wqkvT(0), 4*h_c*h_c, lc);
 * k[i] / v[i] dev bf16 [H][S][d_c] (the cloud KVCache of that layer). */
typedef struct {
    int m, S, H, d_c;
    const void* x;
    int64_t x_stride;
    const int* x_index;
    const void* wq;
    int64_t wq_stride;
    const int* wq_index;
    const void* const* k;
    const void* const* v;
} ekv_cloud_kv;

/* select_channels over the stacked Q / K rows of every matched cloud layer and
 * head (sim.cpp:236-256, head_prune.cpp:83-108), on the device: K1 (tcgen05 Q
 * projection, column sums folded over heads and layers) with the cached-K column
 * sums fused, then the reference ranking on the device.  kept (host int
 * [retained], ascending) and cut_margin may be NULL.  Synchronises. */
int ekv_align_select(ekv_ctx_t ctx, const ekv_cloud_kv* cloud, double lambda, int* kept,
                     double* cut_margin);

/* Artifacts::build_deep_kv (sim.cpp:217-265) on the device, one stream, no host
 * round trip: K1 (tcgen05: Q of every matched layer, column sums of squares
 * folded over heads and layers; the cached-K column sums fused into the same
 * launch) -> the reference ranking on the device (head_prune.cpp:94-107;
 * ChannelMask::full when nothing is pruned, sim.cpp:255-256) -> one batched K3
 * launch compressing K and V of every deep layer into the context:
 * deep_kv[edge_layers[i]] = prune(cloud layer cloud_src[i]) (sim.cpp:258-264).
 * The deep layers must be quantised layers of dst sharing one format.  kept
 * (host int [retained], ascending) and cut_margin (host, see
 * ekv_rank_channels) may be NULL.  Errors mirror assemble_context ("head count
 * mismatch", "dim mismatch ... align with head pruning").  Synchronises. */
int ekv_build_deep_kv(ekv_ctx_t ctx, const ekv_cloud_kv* cloud, double lambda, ekv_kvctx_t dst,
                      int n_deep, const int* edge_layers, const int* cloud_src, int* kept,
                      double* cut_margin);

/* Artifacts::prompt + build_deep_kv + assembled_context (sim.cpp:124-138,
 * 186-212, 217-265) on the device: the edge prefill of the context rows fills
 * the local layers [0, M - n_deep) of dst (bf16); the cloud prefill of the same
 * rows gives the hidden state entering each matched cloud layer and its KV cache;
 * ekv_build_deep_kv fills the deep layers [M - n_deep, M) (int8 / int4).
 *   emb_edge fp32 [S][h_e], emb_cloud fp32 [S][h_c] (device; the reference's
 *   generate_embeddings(Rng::mix(seed, 0xC7E20000 + pid), S, h)), S = dst's rows;
 *   deep_map[i] = cloud layer matched to edge layer M - n_deep + i (ekv_deep_match).
 * kept / cut_margin as ekv_build_deep_kv.  Synchronises. */
int ekv_prompt_context(ekv_model_t edge, ekv_model_t cloud, const float* emb_edge_dev,
                       const float* emb_cloud_dev, int n_deep, const int* deep_map, double lambda,
                       ekv_kvctx_t dst, int* kept, double* cut_margin);

/* bf16_rn of an fp32 device array (e.g. prefill hidden states -> K1 operands). */
int ekv_convert_f32_bf16(ekv_ctx_t ctx, const float* src_dev, void* dst_dev, int64_t n);

/* ------------------------------------------------------------------ */
/* Stage 2: representation compression (gather + quantise + pack)     */
/* ------------------------------------------------------------------ */

/* prune_cache column slice (head_prune.cpp:170-197): dst[i][c] = src[i][kept[c]].
 * src dev bf16 [rows][d_c], kept dev int32 [d_e], dst dev bf16 [rows][d_e]. */
int ekv_kv_gather(ekv_ctx_t ctx, const void* src_dev, int64_t rows, int d_c,
                  const int* kept_dev, int d_e, void* dst_dev);

/* The same column gather for 2-, 4- or 8-byte elements (e.g. fp64 caches of
 * the C++ mirror, where prune_cache must stay an exact copy). */
int ekv_gather_columns(ekv_ctx_t ctx, const void* src_dev, int64_t rows, int d_c,
                       const int* kept_dev, int d_e, int elem_bytes, void* dst_dev);

/* K3: gather kept channels, quantise, pack (no reference -- SPEC.md:281, 488;
 * contract in DESIGN.md section 3, restated in oracle/ekv_oracle.c):
 * per row and group of `group` gathered channels, scale = amax/Q (fp32),
 * code = clamp(rint(x/scale), -Q, Q), Q = 127 (bits 8) or 7 (bits 4).
 *   codes  dev [rows][d_e*bits/8] (int8, or int4 two's-complement nibbles,
 *          element 2j in the low nibble), scales dev fp32 [rows][d_e/group]. */
int ekv_kv_compress(ekv_ctx_t ctx, const void* src_dev, int64_t rows, int d_c,
                    const int* kept_dev, int d_e, int bits, int group, void* codes_dev,
                    float* scales_dev);

/* K3 over n (src, codes, scales) triples in ONE launch (e.g. K and V of every
 * deep layer of build_deep_kv, sim.cpp:258-264).  The three arrays are HOST
 * arrays of DEVICE pointers; all jobs share rows/d_c/kept/d_e/bits/group. */
int ekv_kv_compress_batched(ekv_ctx_t ctx, int n, const void* const* src_dev, int64_t rows,
                            int d_c, const int* kept_dev, int d_e, int bits, int group,
                            void* const* codes_dev, float* const* scales_dev);

/* K6: dst = bf16_rn(code * scale) (fp32 product), dev bf16 [rows][d_e]. */
int ekv_kv_dequant(ekv_ctx_t ctx, const void* codes_dev, const float* scales_dev, int64_t rows,
                   int d_e, int bits, int group, void* dst_dev);
/* K6, exact: dst = code * (double)scale, dev fp64 [rows][d_e] (the historical-cache
 * and C++-mirror paths that hand dequantised KV back as fp64). */
int ekv_kv_dequant_f64(ekv_ctx_t ctx, const void* codes_dev, const float* scales_dev, int64_t rows,
                       int d_e, int bits, int group, double* dst_dev);

/* ------------------------------------------------------------------ */
/* Stage 3: edge decode attention over the reused KV                   */
/* ------------------------------------------------------------------ */

/* One layer's context segment, head-major [H][S][...] like the reference
 * KVCache [layer][head] matrices (transformer.hpp:64-74). */
typedef struct {
    int format;             /* ekv_kv_format */
    int S;                  /* context rows (0 = no context: merge bypassed) */
    int group;              /* quantisation group (ignored for bf16) */
    const void* k;          /* bf16 [H][S][d] or codes [H][S][d*bits/8] */
    const void* v;
    const float* k_scales;  /* [H][S][d/group] (quantised formats) */
    const float* v_scales;
} ekv_segment;

/* K4: segment attention of every query row over the whole context segment
 * (segment_attention_prefix(q, ck, cv, s), cache_merge.cpp:12-38) and over
 * the causal user segment (visible = user_base + r + 1 rows,
 * cache_merge.cpp:206-207), merged exactly by the normaliser rule of Eq. 5
 * (merge_attention, cache_merge.cpp:59-80).  Logits are raw q.k (no scale).
 * Split-KV over the context; partial (max, sum, o) merged by the last CTA.
 *   q       dev fp32 [R][H][d]
 *   user_k  dev bf16 [H][user_cap][d], user_v likewise
 *   out     dev fp32 [R][H][d];  lse dev fp32 [R][H] (optional, natural log)
 * d must be 32, 64 or 128. */
int ekv_decode_attention(ekv_ctx_t ctx, int R, int H, int d, const float* q_dev,
                         const ekv_segment* ctx_seg, const void* user_k_dev,
                         const void* user_v_dev, int user_cap, int user_base, float* out_dev,
                         float* lse_dev);

/* ------------------------------------------------------------------ */
/* Edge model, assembled context, sessions (collaborative decode)      */
/* ------------------------------------------------------------------ */

/* Model / ModelConfig (transformer.hpp:11-20, 76-83) in the B200 layout:
 *   wqkvT[l] bf16 [3h][h]: row part*h + hd*d + c == W_{Q,K,V}[l][hd](:, c)
 *   woT[l]   bf16 [h][h]:  woT[j][i] == out_proj[l](i, j)
 *   gamma, bias fp32 [h] (input transform before layer 0), pos bf16 [max_pos][h]. */
typedef struct {
    int num_layers;
    int num_heads;
    int head_dim;
    int max_positions;
} ekv_model_config;

int ekv_model_create(ekv_ctx_t ctx, const ekv_model_config* cfg, ekv_model_t* out);
int ekv_model_destroy(ekv_model_t m);
/* Upload one layer from host bf16 arrays (sizes as above). */
int ekv_model_set_layer(ekv_model_t m, int layer, const uint16_t* wqkvT_host,
                        const uint16_t* woT_host);
int ekv_model_set_io(ekv_model_t m, const float* gamma_host, const float* bias_host,
                     const uint16_t* pos_host);
/* Device-side synthetic init (random-init weights of the architecture):
 * counter-hash U[-w_scale, w_scale] for weights (1/sqrt(d) folded into W_Q),
 * U[-pos_scale, pos_scale] for positions, gamma = 1, bias = 0. */
int ekv_model_synthesize(ekv_model_t m, uint64_t seed, double w_scale, double pos_scale);
/* Device pointers of the weights (for tests / tooling). */
int ekv_model_weights(ekv_model_t m, int layer, void** wqkvT_dev, void** woT_dev);
int ekv_model_io(ekv_model_t m, float** gamma_dev, float** bias_dev, void** pos_dev);

/* AssembledContext (cache_merge.hpp:48-51, assemble_context
 * cache_merge.cpp:82-150): S context rows; layer_format[l] gives each
 * layer's storage (EKV_KV_BF16 for local/peer layers, EKV_KV_INT8/INT4 for
 * cloud layers).  Storage is allocated here; producers write it through
 * ekv_kvctx_layer (e.g. with ekv_kv_compress) or ekv_kvctx_upload_bf16. */
int ekv_kvctx_create(ekv_model_t m, int S, const int* layer_format_host, int group,
                     ekv_kvctx_t* out);
int ekv_kvctx_destroy(ekv_kvctx_t c);
int ekv_kvctx_layer(ekv_kvctx_t c, int layer, ekv_segment* seg_out);
/* Host bf16 [H][S][d] upload into a bf16 layer. */
int ekv_kvctx_upload_bf16(ekv_kvctx_t c, int layer, const uint16_t* k_host,
                          const uint16_t* v_host);
/* Deliver one layer from caller device buffers (D2D on the context stream):
 * bf16 layers take k/v bf16 [H][S][d]; quantised layers take codes
 * [H][S][d*bits/8] and scales fp32 [H][S][d/group].  This is where the
 * cloud->edge transfer lands (sim.cpp:802-814, assembled_context
 * sim.cpp:186-212). */
int ekv_kvctx_set_layer(ekv_kvctx_t c, int layer, const void* k_dev, const void* v_dev,
                        const float* k_scales_dev, const float* v_scales_dev);
/* Peer sharing of context layers (the simulator's peer source, Eq. 19
 * cache_source -> peer, sim.cpp:705-719, 757-786): copy `layers` of `src` (a
 * context of the same geometry, possibly on another GPU of this process) into
 * `dst`, device to device over NVLink (cudaMemcpyPeerAsync, peer access enabled
 * when the pair supports it), ordered after src's queued work, on dst's stream.
 * Across processes the same transfer runs over NCCL (paper_2505_14085_b200.dist).
 * Synchronises dst's stream. */
int ekv_kvctx_copy_layers(ekv_kvctx_t dst, ekv_kvctx_t src, const int* layers, int n);
/* Fill every layer with counter-hash random data (synthetic context). */
int ekv_kvctx_synthesize(ekv_kvctx_t c, uint64_t seed);

/* A decode session: the user/generated KV cache (bf16 [L][H][cap][d]) plus
 * the device state of merged_forward (cache_merge.cpp:156-226).  Sessions
 * sharing one kvctx share its storage read-only. */
int ekv_session_create(ekv_model_t m, ekv_kvctx_t c, int max_user_rows, ekv_session_t* out);
int ekv_session_destroy(ekv_session_t s);
int ekv_session_reset(ekv_session_t s);
int ekv_session_length(ekv_session_t s, int* user_rows);
/* merged_forward over n new rows given on the device (fp32 [n][h]);
 * writes the final-layer rows to out_dev (fp32 [n][h]). */
int ekv_session_forward(ekv_session_t s, const float* emb_dev, int n, float* out_dev);
/* `steps` autoregressive steps, each feeding back the previous final-layer
 * row (collaborative_decode loop, cache_merge.cpp:256-271).  Outputs fp32
 * [steps][h] on the device.  Replays one captured CUDA graph per step. */
int ekv_session_decode(ekv_session_t s, int steps, float* out_dev);
/* Decode implementation: 0 = one persistent kernel per step (k_decode_mega.cu,
 * default when the shape allows: S % 16 == 0, h <= 2048, <= 64 layers),
 * 1 = the per-layer kernels (K5, K4, K5) replayed from a CUDA graph.
 * active (optional) receives the path that will actually run. */
int ekv_session_set_decode_path(ekv_session_t s, int path, int* active);
/* Diagnostics of the persistent path: one real decode step with %globaltimer
 * stamps (ns) of its phases: out[(l*G + g)*16 + k] = CTA g in layer l at k =
 * 0 layer start, 1 input ready, 2 QKV rows done, 3 q/k/v of its heads ready,
 * 4 attention partials published, 5 head merge done, 6 output-projection
 * partials published, 7 layer output reduced; k = 8..10: ring-wait cycles of
 * the consumer warps in the QKV, attention and output-projection phases.
 * out[(L*G + g)*16 + k]: 0 CTA start, 1/2 producer start/end (ns), 3 stages
 * issued, 4 producer cycles waiting for free ring slots, 5 producer cycles.
 * G = the persistent kernel's grid (the largest multiple of H <= the SM count);
 * n_out = 16*(L+1)*G.  Needs capacity >= 16*(L+1)*(SM count). */
int ekv_session_trace_step(ekv_session_t s, uint64_t* out, int capacity, int* n_out);
/* One decode step launched kernel by kernel with CUDA events between the
 * launches (diagnostics / roofline attribution; the step is real and advances
 * the session).  Graph path: kernel_ms[3l+0] = layer l QKV projection,
 * [3l+1] = decode attention, [3l+2] = output projection, [3L] = state advance.
 * Persistent path: kernel_ms[0] = the whole step (one kernel). */
int ekv_session_profile_step(ekv_session_t s, float* kernel_ms, int capacity, int* n_kernels);
/* Device pointer of the user cache of one layer (bf16 [H][cap][d]). */
int ekv_session_user_kv(ekv_session_t s, int layer, void** k_dev, void** v_dev, int* cap);

/* collaborative_decode (cache_merge.hpp:73-75, cache_merge.cpp:230-273) with
 * HOST buffers, synchronous: resets the session, copies user_emb (fp32
 * [U][h]) to the device, runs the user prefill and `steps` decode steps,
 * copies prefill outputs (fp32 [U][h], may be NULL) and step outputs
 * (fp32 [steps][h]) back.  Errors: "steps must be >= 1", "position overflow",
 * "align with head pruning" (context dims differ from the model). */
int ekv_collaborative_decode(ekv_session_t s, const float* user_emb_host, int U, int steps,
                             float* prefill_out_host, float* step_out_host);

/* Eq. 20 pipelined prefill (cost_model.cpp:73-100 pipeline_schedule; the
 * simulator's per-layer transfer/compute overlap, sim.cpp:652-683, 909-933):
 * the context layers listed in `uploads` arrive from HOST memory (pinned, the
 * emulated cloud->edge link) on the context's copy stream while the user rows
 * are forwarded on the compute stream; layer l's attention waits only for
 * layer l's upload, so upload l overlaps the compute of layers < l.
 * uploads[L]: per layer, host K/V in the layer's storage format (bf16 [H][S][d]
 * or codes) and fp32 scales for quantised layers; k_host == NULL = resident.
 * overlap = 0 runs the sequential schedule (all uploads, then compute) for
 * comparison.  Outputs (each may be NULL): out_dev fp32 [n][h], t_comm_ms[L]
 * (upload time of each layer on the copy stream), total_ms (first upload -> last
 * output), t_comp_ms[L] (compute of each layer -- a diagnostic that re-runs the
 * rows kernel by kernel with the context resident, so it doubles the work; pass
 * NULL outside measurements).  Synchronous. */
typedef struct {
    const void* k_host;
    const void* v_host;
    const float* k_scales_host;
    const float* v_scales_host;
} ekv_layer_upload;
int ekv_session_forward_pipelined(ekv_session_t s, const float* emb_dev, int n, float* out_dev,
                                  const ekv_layer_upload* uploads, int overlap, float* t_comm_ms,
                                  float* t_comp_ms, float* total_ms);

/* Eq. 20 with the context layers delivered by another agent on another stream --
 * e.g. an NCCL receive from the cloud rank (the emulated cloud->edge link,
 * Sim::fetch_deep_layer -> submit_transfer, sim.cpp:802-814, 417-449) landing in
 * this context's storage (ekv_kvctx_layer pointers).  layer_ready[l] is a
 * cudaEvent_t the producer records after layer l landed (NULL entry, or a NULL
 * array = resident); layer l's attention waits on it, so the transfer of layer l
 * overlaps the compute of layers < l.  Asynchronous on the context stream. */
int ekv_session_forward_streamed(ekv_session_t s, const float* emb_dev, int n, float* out_dev,
                                 void* const* layer_ready);

/* ------------------------------------------------------------------ */
/* Batched sessions (BASELINE configs[2], concurrent edge sessions)     */
/* ------------------------------------------------------------------ */
/* B independent sessions that share one assembled context (the paper's
 * shared system prompt; one read-only context cache, many
 * user caches: cache_merge.cpp:252) and advance in lock-step
 * (all sessions have the same number of user rows).  Per session the
 * result is collaborative_decode (cache_merge.cpp:230-273); the weights and
 * the context are streamed once per step for all B sessions (tensor-core
 * projections and a cascade context attention, k_batch.cu).
 * max_rows bounds user + generated rows per session.  Supported: hidden
 * size a multiple of 128; context layers bf16 with head_dim 64. */
int ekv_batch_create(ekv_model_t m, ekv_kvctx_t c, int sessions, int max_rows, ekv_batch_t* out);
int ekv_batch_destroy(ekv_batch_t b);
int ekv_batch_reset(ekv_batch_t b);
/* sessions, rows forwarded so far, and the work splits {QKV split-K,
 * out-proj split-K, context splits per head} (any pointer may be NULL) */
int ekv_batch_info(ekv_batch_t b, int* sessions, int* rows, int* splits);
/* merged_forward of n user rows of every session: emb_dev fp32 [B][n][h];
 * out_dev (may be NULL) receives fp32 [n][B][h]. */
int ekv_batch_forward(ekv_batch_t b, const float* emb_dev, int n, float* out_dev);
/* `steps` decode steps of every session; out_dev (may be NULL) fp32 [steps][B][h]. */
int ekv_batch_decode(ekv_batch_t b, int steps, float* out_dev);
/* One real forward row of every session launched kernel by kernel with CUDA
 * events in between (diagnostics / roofline attribution; advances the batch).
 * kernel_ms[0] = layer-0 input transform; layer l: [1+5l] QKV projection,
 * [2+5l] context attention (0 if the layer has no context), [3+5l] user
 * segment + merge, [4+5l] output projection, [5+5l] split-K sum;
 * [5L+1] = state advance.  Needs capacity >= 5L + 2. */
int ekv_batch_profile_row(ekv_batch_t b, float* kernel_ms, int capacity, int* n_kernels);
/* collaborative_decode of all B sessions with HOST buffers, synchronous:
 * user_emb fp32 [B][U][h]; prefill_out [U][B][h] (may be NULL);
 * step_out [steps][B][h].  Same errors as ekv_collaborative_decode. */
int ekv_collaborative_decode_batch(ekv_batch_t b, const float* user_emb_host, int U, int steps,
                                   float* prefill_out_host, float* step_out_host);

/* ------------------------------------------------------------------ */
/* Packed-KV wire / disk format ("EKVPACK1")                            */
/* ------------------------------------------------------------------ */
/* The compressed cloud layers as one self-describing, checksummed byte
 * stream: what crosses the cloud -> edge link (the transfer the reference
 * simulates in Sim::submit_transfer, sim.cpp:417-449, sized by
 * deep_layer_bytes, sim.cpp:714) or is kept as the historical cache
 * (sim.cpp:885-895).
 * Layout (little-endian):
 *   header 64 B: magic "EKVPACK1", u32 version (2), n_layers, H, S, d_e,
 *     d_c, bits, group, header_bytes, 3 x u32 reserved, u64 header_fnv
 *   i32 edge_layer[n], i32 cloud_layer[n] (the layer map), i32 kept[d_e]
 *   (the channel mask), u64 layer_fnv[n], zero padding to header_bytes
 *   (a multiple of 256)
 *   per layer: K codes [H][S][d_e*bits/8], V codes, K scales fp32
 *   [H][S][d_e/group], V scales
 * Checksums are FNV-1a 64 (the reference's fnv1a64, rng.cpp:7-15): the header
 * (with header_fnv = 0) over its bytes; a layer (version 2) over the u64 FNV-1a
 * 64s, little-endian, of its four arrays cut into 4 KiB chunks in payload order
 * (the last chunk of an array may be shorter) -- independent chunks, so the
 * device hashes a layer where its bytes are.  Version 1 (FNV-1a over the whole
 * layer payload) is still read. */
typedef struct {
    int n_layers, H, S, d_e, d_c, bits, group;
    size_t bytes;
} ekv_kvpack_info;
int ekv_fnv1a64(const void* data, size_t len, uint64_t seed, uint64_t* out);
int ekv_kvpack_size(int n_layers, int H, int S, int d_e, int bits, int group, size_t* bytes);
/* Serialise compressed layers `layers[n]` of the context (with their cloud
 * layers and the channel mask kept[d_e]) into host memory. */
int ekv_kvpack_export(ekv_kvctx_t c, const int* layers, const int* cloud_layers, int n, const int* kept,
                      int d_c, void* host_dst, size_t capacity);
/* Validate a pack (magic, version, sizes, every checksum) and read its
 * description; layers / cloud_layers [n_layers] and kept [d_e] may be NULL.
 * Host only. Errors: "bad magic", "header checksum mismatch", "checksum
 * mismatch in layer N", "truncated ...". */
int ekv_kvpack_parse(const void* host_src, size_t bytes, ekv_kvpack_info* info, int* layers,
                     int* cloud_layers, int* kept);
/* Validate and copy the pack's layers into the context's storage (formats,
 * H, S and d_e must match: "kvpack: dim mismatch").  Version 2: the payload is
 * copied to an HBM staging buffer and hashed there; the context is written only
 * after every layer checksum matched. */
int ekv_kvpack_import(ekv_kvctx_t c, const void* host_src, size_t bytes);
/* Eq. 20 over the wire format: the pack's layers are uploaded one by one (copy
 * stream) into the session's context while the n rows are forwarded layer-major on
 * the compute stream -- layer l's attention waits only for layer l's upload
 * (cost_model.cpp:73-100, sim.cpp:802-814, 909-933).  Every layer is hashed on the
 * device after its upload and checked at the end: on "checksum mismatch" the
 * outputs and the context's imported layers are invalid.  Version-2 packs.
 * Synchronises. */
int ekv_session_forward_pack(ekv_session_t s, const float* emb_dev, int n, float* out_dev,
                             const void* host_src, size_t bytes);

/* ------------------------------------------------------------------ */
/* The emulated cloud -> edge link over NCCL (one process per GPU)      */
/* ------------------------------------------------------------------ */
/* The B200 counterpart of Sim::fetch_deep_layer -> submit_transfer
 * (sim.cpp:802-814, 417-449): the cloud rank sends the compressed deep layers of
 * its assembled context layer by layer (ncclSend, one NCCL group per layer, on the
 * context's copy stream); the edge rank receives them straight into its context's
 * storage while the user rows are forwarded layer-major on the compute stream,
 * layer l's attention waiting only for layer l's receive (Eq. 20,
 * cost_model.cpp:73-100).  NCCL (libnccl.so.2) is resolved at run time.
 * id: the 128-byte ncclUniqueId, made on one rank and shared out of band. */
typedef struct ekv_link_s* ekv_link_t;
int ekv_link_unique_id(void* id128);
int ekv_link_create(ekv_ctx_t ctx, const void* id128, int nranks, int rank, ekv_link_t* out);
int ekv_link_destroy(ekv_link_t link);
/* Sender: `layers` of src (after the context stream's queued work) to rank peer.
 * seconds (optional): link time of the whole transfer.  Synchronises. */
int ekv_link_send_layers(ekv_link_t link, ekv_kvctx_t src, const int* layers, int n, int peer,
                         float* seconds);
/* Receiver: `layers` of the session's context from rank peer; with rows > 0 the
 * session forwards emb_dev (fp32 [rows][h]) layer-major meanwhile (out_dev fp32
 * [rows][h], may be NULL).  seconds (optional): link time.  Synchronises. */
int ekv_link_recv_forward(ekv_link_t link, ekv_session_t s, const int* layers, int n, int peer,
                          const float* emb_dev, int rows, float* out_dev, float* seconds);

/* ------------------------------------------------------------------ */
/* Scheduler interface (cost_model.hpp:53-84)                          */
/* ------------------------------------------------------------------ */

/* cache_source (cost_model.cpp:64-71): 0 local, 1 peer, 2 cloud. */
int ekv_cache_source(int layer, double cost_local, double cost_peer, int boundary, int m,
                     int* source);
/* pipeline_schedule (cost_model.cpp:73-100), Eq. 20. */
int ekv_pipeline_schedule(const double* t_comm, const double* t_comp, int n, double* t_pip,
                          double* sequential_total, double* pipelined_total);

#if defined(__GNUC__)
#pragma GCC visibility pop
#endif
#ifdef __cplusplus
}
#endif
#endif /* EKV_CAPI_H */
