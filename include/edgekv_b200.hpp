// edgekv_b200.hpp -- C++ mirror of the reference's interface for the
// cloud->edge KV-reuse path, backed by the B200 C ABI (ekv_capi.h).
//
// A reference caller links libedgekv_b200.so instead of the hot-path objects
// of edgekv_core (proj/src/CMakeLists.txt:1-13): the declarations below keep
// the reference's namespace, names, argument meaning, member layout of the
// value types and exception texts (the substrings the reference's tests
// assert).  Cited interfaces (file:line under /root/reference/proj):
//   Matrix                  include/edgekv/matrix.hpp:14-35
//   ModelConfig / Model     include/edgekv/transformer.hpp:11-20, 76-83
//   KVCache                 include/edgekv/transformer.hpp:64-74
//   PruneSpec/ChannelMask   include/edgekv/head_prune.hpp:12-31
//   select_channels         include/edgekv/head_prune.hpp:35
//   prune_cache             include/edgekv/head_prune.hpp:70
//   segment_attention       include/edgekv/cache_merge.hpp:29
//   merge_attention         include/edgekv/cache_merge.hpp:38
//   assemble_context        include/edgekv/cache_merge.hpp:58-61
//   collaborative_decode    include/edgekv/cache_merge.hpp:73-75
//   match_layers            include/edgekv/layer_match.hpp:53-55
//   FlopCounts / QkvRows    include/edgekv/transformer.hpp:36-53, 90-92
//   project_qkv             include/edgekv/transformer.hpp:94
//   PrefillResult/prefill   include/edgekv/transformer.hpp:108-118
//   decode_step             include/edgekv/transformer.hpp:120-124
//   forward_rows            include/edgekv/transformer.hpp:129-131
//   cache_source            include/edgekv/cost_model.hpp:61
//   pipeline_schedule       include/edgekv/cost_model.hpp:80-81
//
// Precision contract of the B200 path (DESIGN.md s.5):
//  * exact / reference bits, fp64 on the device in the reference's operation
//    order: project_qkv (bit-identical matmul), segment_attention (libm exp
//    aside), select_channels' column norms (fp64), match_layers (K7,
//    bit-identical CKA/RSA), prune_cache (exact copy), dequantize (exact);
//  * the B200 compute path, bf16 storage with fp32 accumulation (normwise 1e-3):
//    forward_rows / prefill / decode_step / collaborative_decode (the edge
//    forward), b200::build_deep_kv's channel scores (K1 on the tensor cores);
//  * host fp64 scalar arithmetic exactly as the reference: merge_attention,
//    cache_source, pipeline_schedule.
// Operations that have no kernel for a shape throw std::invalid_argument (there
// is no CPU fallback for device work).
#pragma once

#include <cstddef>
#include <cstdint>
#include <map>
#include <optional>
#include <string>
#include <vector>

namespace edgekv {

using Vec = std::vector<double>;

struct Matrix {
    std::size_t rows = 0;
    std::size_t cols = 0;
    std::vector<double> data;  // row-major

    Matrix() = default;
    Matrix(std::size_t r, std::size_t c) : rows(r), cols(c), data(r * c, 0.0) {}
    double& operator()(std::size_t i, std::size_t j) { return data[i * cols + j]; }
    double operator()(std::size_t i, std::size_t j) const { return data[i * cols + j]; }
    double* row_ptr(std::size_t i) { return data.data() + i * cols; }
    const double* row_ptr(std::size_t i) const { return data.data() + i * cols; }
    Vec row(std::size_t i) const { return Vec(row_ptr(i), row_ptr(i) + cols); }
    bool empty() const { return rows == 0 || cols == 0; }
    bool same_shape(const Matrix& o) const { return rows == o.rows && cols == o.cols; }
};

// ---- toy model types (layout-compatible with the reference) ----------------
struct ModelConfig {
    int num_layers = 1;
    int num_heads = 1;
    int head_dim = 1;
    int hidden_size = 1;
    int max_positions = 128;
    std::uint64_t seed = 0;
    void validate() const;
};

struct HeadWeights {
    Matrix wq, wk, wv;  // hidden_size x head_dim
};

struct LayerWeights {
    std::vector<HeadWeights> heads;
    Matrix out_proj;  // hidden_size x hidden_size
    Vec gamma;        // input transform (layer 0)
    Vec bias;
};

enum class PositionKind { context, user, generated };

struct PositionTag {
    PositionKind kind;
    int index;
};

struct KVCache {
    int num_layers = 0;
    int num_heads = 0;
    int head_dim = 0;
    std::vector<std::vector<Matrix>> keys;    // [layer][head], positions x head_dim
    std::vector<std::vector<Matrix>> values;
    std::vector<PositionTag> positions;

    int size() const { return static_cast<int>(positions.size()); }
    static KVCache empty_for(int layers, int heads, int dim);
};

struct Model {
    ModelConfig config;
    std::vector<LayerWeights> layers;
    Matrix pos_embedding;  // max_positions x hidden_size
};

// Exact floating-op counts split by stage (transformer.hpp:36-53); the B200
// forward fills them with the reference's closed forms (transformer.cpp:267-283).
struct FlopCounts {
    std::int64_t proj = 0;
    std::int64_t score = 0;
    std::int64_t softmax = 0;
    std::int64_t value = 0;
    std::int64_t out_proj = 0;
    std::int64_t attention() const { return score + softmax + value; }
    std::int64_t total() const { return proj + score + softmax + value + out_proj; }
    FlopCounts& operator+=(const FlopCounts& o) {
        proj += o.proj;
        score += o.score;
        softmax += o.softmax;
        value += o.value;
        out_proj += o.out_proj;
        return *this;
    }
};

struct QkvRows {
    Matrix q, k, v;
};

// Q = x*W_Q etc. for the addressed head, fp64 on the device, bit-identical to
// the reference (x is n x hidden_size).
QkvRows project_qkv(const Model& model, const Matrix& x, int layer, int head);

struct PrefillResult {
    KVCache cache;
    std::vector<Matrix> layer_outputs;  // per layer, n x hidden_size
};

// The edge/cloud forward on the device (bf16 weights and KV, fp32 accumulate):
// the new rows attend to every cached row and causally to each other; K/V of
// the new rows are appended to `cache`, per-layer outputs returned.
std::vector<Matrix> forward_rows(const Model& model, KVCache& cache, const Matrix& embeddings,
                                 PositionKind kind, FlopCounts* fc);
PrefillResult prefill(const Model& model, const Matrix& embeddings, FlopCounts* fc = nullptr,
                      PositionKind kind = PositionKind::context);
Vec decode_step(const Model& model, KVCache& cache, const Vec& embedding, FlopCounts* fc = nullptr,
                PositionKind kind = PositionKind::generated);

// ---- alignment / projection (head_prune.hpp) --------------------------------
struct PruneSpec {
    double lambda = 0.0;
    int head_dim = 0;
    int retained = 0;
    static PruneSpec from_lambda(double lambda, int head_dim);
    void validate() const;
};

struct ChannelMask {
    int head_dim = 0;
    std::vector<int> kept;  // unique, ascending
    void validate() const;
    static ChannelMask full(int head_dim);
};

// Column norms of the stacked Q and K rows on the GPU in fp64, ranking with the
// reference rule (stable descending, ties to the lower index).
ChannelMask select_channels(const Matrix& q, const Matrix& k, const PruneSpec& spec);

// Exact column slice of every K/V matrix (fp64 gather on the GPU).
KVCache prune_cache(const KVCache& cache, const ChannelMask& mask);

// ---- edge decode attention (cache_merge.hpp) ---------------------------------
struct SegmentAttention {
    Vec o;
    double sigma = 0.0;
    double shift = 0.0;
    double sigma_raw() const;
};

struct MergeWeights {
    double alpha_ctx = 0.0;
    double alpha_user = 0.0;
};

struct MergedAttention {
    Vec o;
    MergeWeights weights;
};

// One query over one segment on the GPU in fp64: o, sigma = sum exp(l - max),
// shift = max logit, as the reference (cache_merge.cpp:12-57).
SegmentAttention segment_attention(const Vec& q, const Matrix& k, const Matrix& v);

// Eq. 5 merge of two segments (scalar arithmetic, fp64, host).
MergedAttention merge_attention(const SegmentAttention& ctx, const SegmentAttention& user);

enum class CacheOrigin { local, peer, cloud };

struct LayerKV {
    std::vector<Matrix> keys;
    std::vector<Matrix> values;
};

struct AssembledContext {
    KVCache cache;
    std::vector<CacheOrigin> provenance;
};

AssembledContext assemble_context(const std::map<int, LayerKV>& shared,
                                  const std::map<int, LayerKV>& local,
                                  const std::map<int, CacheOrigin>& shared_origins = {},
                                  int expected_layers = -1);

struct CollaborativeResult {
    std::vector<Vec> step_outputs;
    std::vector<Vec> prefill_outputs;
};

// User prefill + `steps` decode steps of the edge model over the assembled
// context, entirely on the GPU (one persistent kernel per decode step).
CollaborativeResult collaborative_decode(const Model& edge_model, const AssembledContext& context,
                                         const Matrix& user_embeddings, int steps);

// ---- layer matching (layer_match.hpp) ----------------------------------------
struct SimilarityConfig {
    double theta_cka = 0.5;
    double theta_rsa = 0.3;
    int num_probe_samples = 64;
    void validate() const;
};

struct LayerMatch {
    int edge_layer;
    int cloud_layer;
    double cka;
    double rsa;
};

struct LayerMatchReport {
    Matrix cka;
    Matrix rsa;
    std::vector<LayerMatch> matches;
    std::vector<int> shared_layers;
    std::vector<std::optional<int>> best;
    SimilarityConfig config;
};

LayerMatchReport match_layers(const std::vector<Matrix>& edge_outputs,
                              const std::vector<Matrix>& cloud_outputs,
                              const SimilarityConfig& cfg);

// ---- scheduler interface (cost_model.hpp) -------------------------------------
enum class CacheSource { local, peer, cloud };
CacheSource cache_source(int layer, double cost_local, double cost_peer, int boundary, int m);

struct LayerTimes {
    double t_comm = 0.0;
    double t_comp = 0.0;
};

struct ScheduleEntry {
    CacheSource source = CacheSource::local;
    double t_comm = 0.0;
    double t_comp = 0.0;
    double t_pip = 0.0;
};

struct ScheduleTrace {
    std::vector<ScheduleEntry> layers;
    double sequential_total = 0.0;
    double pipelined_total = 0.0;
};

ScheduleTrace pipeline_schedule(const std::vector<LayerTimes>& layers,
                                const std::vector<CacheSource>& sources = {});

// ---- B200-native extensions ------------------------------------------------------
namespace b200 {

// Device used by the mirror (default 0); must be set before the first call.
void set_device(int device);
// Drop the cached device copy of a model (collaborative_decode caches the
// upload per Model object; call after mutating its weights).
void invalidate(const Model& model);

// The representation-compression step: gather the kept channels of every K/V
// matrix and quantise them (int8 / int4, DESIGN.md s.3).
struct QuantizedLayer {
    int bits = 8, group = 0, head_dim = 0, positions = 0;
    std::vector<std::uint8_t> k_codes, v_codes;  // [head][pos][d*bits/8]
    std::vector<float> k_scales, v_scales;       // [head][pos][d/group]
};
std::vector<QuantizedLayer> compress_cache(const KVCache& cache, const ChannelMask& mask, int bits,
                                           int group = 0);
// The dequantised context as fp64 K/V (code * scale, exact, on the device), e.g.
// for assemble_context.
LayerKV dequantize(const QuantizedLayer& q, int num_heads);
// Artifacts::build_deep_kv (sim.cpp:217-265) with the Q re-projection on the
// tensor cores (K1) instead of project_qkv in fp64 on the host: the channel mask
// over the stacked Q/K rows of every distinct matched cloud layer (the layer
// inputs x0 = gamma*(ctx_emb + pos) + b or cloud_prefill.layer_outputs[lc - 1],
// the cached K of cloud_prefill.cache), and deep_kv[le] = the pruned cloud KV of
// match[le] (an exact column slice).
struct DeepKV {
    ChannelMask mask;
    double cut_margin = 0.0;  // relative score gap at the cut (near-tie audit)
    std::map<int, LayerKV> deep_kv;
};
DeepKV build_deep_kv(const Model& cloud_model, const PrefillResult& cloud_prefill,
                     const Matrix& ctx_emb_cloud, const std::map<int, int>& match,
                     const PruneSpec& spec);

}  // namespace b200
}  // namespace edgekv
