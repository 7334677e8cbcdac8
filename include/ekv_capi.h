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
 * mirror): allocation on the context's device, and synchronous copies on the
 * context stream.  kind: 0 host->device, 1 device->host, 2 device->device. */
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

/* Layer map (match_layers, layer_match.cpp:166-228) over probe outputs
 * [me][n][ce] / [nc][n][cc] (host fp64).  best[le] = matched cloud layer or
 * -1.  cka/rsa outputs [me][nc].  Computed on the host in fp64 (offline, once
 * per model pair; SURVEY.md section 8(f) row 3 moves it to the GPU). */
int ekv_match_layers(const double* edge_outs, int me, int ce, const double* cloud_outs, int nc,
                     int cc, int n, double theta_cka, double theta_rsa, double* cka, double* rsa,
                     int* best);
/* K7: the same layer map on the device.  edge_outs / cloud_outs are DEVICE
 * buffers (the probe-prefill outputs, fp64); cka / rsa / best are host arrays.
 * Bit-identical to match_layers (layer_match.cpp:166-228): fp64 in the
 * reference's operation order.  Same errors and messages.  n <= 256.
 * Synchronises the context's stream. */
int ekv_match_layers_dev(ekv_ctx_t c, const double* edge_outs, int me, int ce,
                         const double* cloud_outs, int nc, int cc, int n, double theta_cka,
                         double theta_rsa, double* cka, double* rsa, int* best);

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
 * comparison.  Outputs: out_dev fp32 [n][h] (may be NULL), t_comm_ms[L]
 * (upload time of each layer on the copy stream), t_comp_ms[L] (compute of each
 * layer, measured by a kernel-by-kernel re-run with the context resident),
 * total_ms (first upload -> last output).  Synchronous. */
typedef struct {
    const void* k_host;
    const void* v_host;
    const float* k_scales_host;
    const float* v_scales_host;
} ekv_layer_upload;
int ekv_session_forward_pipelined(ekv_session_t s, const float* emb_dev, int n, float* out_dev,
                                  const ekv_layer_upload* uploads, int overlap, float* t_comm_ms,
                                  float* t_comp_ms, float* total_ms);

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
 * deep_layer_bytes, sim.cpp:714) or is kept as the historical cache.
 * Layout (little-endian):
 *   header 64 B: magic "EKVPACK1", u32 version (1), n_layers, H, S, d_e,
 *     d_c, bits, group, header_bytes, 3 x u32 reserved, u64 header_fnv
 *   i32 edge_layer[n], i32 cloud_layer[n] (the layer map), i32 kept[d_e]
 *   (the channel mask), u64 layer_fnv[n], zero padding to header_bytes
 *   (a multiple of 256)
 *   per layer: K codes [H][S][d_e*bits/8], V codes, K scales fp32
 *   [H][S][d_e/group], V scales
 * Checksums are FNV-1a 64 (the reference's fnv1a64, rng.cpp:7-15): the
 * header (with header_fnv = 0) and each layer's payload. */
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
 * H, S and d_e must match: "kvpack: dim mismatch"). */
int ekv_kvpack_import(ekv_kvctx_t c, const void* host_src, size_t bytes);

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
