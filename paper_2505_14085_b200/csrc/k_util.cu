// Small device utilities of the stage 1+2 pipeline: the channel ranking of
// select_channels on the device (so align -> rank -> compress needs no host
// round trip), dtype conversions of the prefill outputs, the layer-0 input
// transform, fp64 column norms (the C++ mirror's fp64 select_channels) and an
// exact fp64 dequantiser (the mirror's QuantizedLayer -> LayerKV).
#include "ekv_common.cuh"
#include "ekv_kernels.h"

namespace ekv {

// select_channels ranking (head_prune.cpp:94-107): score_c = sqrt(qn)*sqrt(kn)
// (fp64, IEEE sqrt and product = the host's std::sqrt), std::stable_sort by
// descending score, keep the first `retained`, then ascending.  The stable-sort
// position of c is #{j : s_j > s_c} + #{j < c : s_j == s_c}; one thread per
// channel counts it, so the result is the host ranking bit for bit.
__global__ void rank_channels_kernel(const double* __restrict__ q, const double* __restrict__ k,
                                     int d_c, int retained, int* __restrict__ kept,
                                     double* __restrict__ margin) {
    extern __shared__ double sc[];  // [d_c] scores, then [d_c] ints (rank)
    int* rank = (int*)(sc + d_c);
    const int t = threadIdx.x;
    for (int c = t; c < d_c; c += blockDim.x) sc[c] = sqrt(q[c]) * sqrt(k[c]);
    __syncthreads();
    for (int c = t; c < d_c; c += blockDim.x) {
        const double s = sc[c];
        int r = 0;
        for (int j = 0; j < d_c; ++j) r += (sc[j] > s) || (j < c && sc[j] == s);
        rank[c] = r;
    }
    __syncthreads();
    // kept in ascending channel order: output slot = #{j < c : rank_j < retained}
    for (int c = t; c < d_c; c += blockDim.x) {
        if (rank[c] < retained) {
            int slot = 0;
            for (int j = 0; j < c; ++j) slot += rank[j] < retained;
            kept[slot] = c;
        }
    }
    if (margin != nullptr && t == 0) {
        double a = -1.0, b = -1.0;
        for (int c = 0; c < d_c; ++c) {
            if (rank[c] == retained - 1) a = sc[c];
            if (rank[c] == retained) b = sc[c];
        }
        double mg = INFINITY;
        if (retained > 0 && retained < d_c) mg = a > 0 ? (a - b) / a : 0.0;
        *margin = mg;
    }
}

void launch_rank_channels(const double* q, const double* k, int d_c, int retained, int* kept,
                          double* margin, cudaStream_t st) {
    require(d_c >= 1 && d_c <= 4096, "rank_channels: head_dim outside [1, 4096]", EKV_EUNSUPPORTED);
    const int threads = d_c < 1024 ? ((d_c + 31) / 32) * 32 : 1024;
    rank_channels_kernel<<<1, threads, (size_t)d_c * (sizeof(double) + sizeof(int)), st>>>(
        q, k, d_c, retained, kept, margin);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

static int grid_1d(int64_t n, int per_block) {
    int64_t b = (n + per_block - 1) / per_block;
    const int64_t cap = (int64_t)device_sm_count() * 8;
    return (int)(b < 1 ? 1 : (b > cap ? cap : b));
}

__global__ void f32_to_bf16_kernel(const float* __restrict__ src, uint16_t* __restrict__ dst,
                                   int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = f32_to_bf16_bits(src[i]);
}

void launch_f32_to_bf16(const float* src, uint16_t* dst, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    f32_to_bf16_kernel<<<grid_1d(n, 256), 256, 0, st>>>(src, dst, n);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

__global__ void f32_to_f64_kernel(const float* __restrict__ src, double* __restrict__ dst, int64_t n) {
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += stride)
        dst[i] = (double)src[i];
}

void launch_f32_to_f64(const float* src, double* dst, int64_t n, cudaStream_t st) {
    if (n <= 0) return;
    f32_to_f64_kernel<<<grid_1d(n, 256), 256, 0, st>>>(src, dst, n);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

// x0 = gamma * (emb + pos) + bias (transformer.cpp:198-210, layer 0 only), in the
// same fp32 operation order as the projection kernels' fused staging.
__global__ void input_transform_kernel(const float* __restrict__ emb, const float* __restrict__ gamma,
                                       const float* __restrict__ bias, const uint16_t* __restrict__ pos,
                                       int p0, int n, int h, float* __restrict__ x0) {
    const int64_t total = (int64_t)n * h;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
        const int r = (int)(i / h), c = (int)(i - (int64_t)r * h);
        const float p = __uint_as_float((uint32_t)pos[(int64_t)(p0 + r) * h + c] << 16);
        x0[i] = fmaf(gamma[c], emb[i] + p, bias[c]);
    }
}

void launch_input_transform(const float* emb, const float* gamma, const float* bias,
                            const uint16_t* pos, int p0, int n, int h, float* x0, cudaStream_t st) {
    if (n <= 0) return;
    input_transform_kernel<<<grid_1d((int64_t)n * h, 256), 256, 0, st>>>(emb, gamma, bias, pos, p0, n,
                                                                          h, x0);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

// fp64 column sums of squares: one thread per (column, row slice); fp64 partials
// folded with atomics (order-dependent only at the last bit, ~1e-16 relative).
__global__ void colsq_f64_kernel(const double* __restrict__ m, int64_t rows, int d,
                                 double* __restrict__ colsq) {
    for (int c = threadIdx.x; c < d; c += blockDim.x) {
        double acc = 0.0;
        for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
            const double v = m[r * d + c];
            acc += v * v;
        }
        atomicAdd(&colsq[c], acc);
    }
}

void launch_colsq_f64(const double* m, int64_t rows, int d, double* colsq, cudaStream_t st) {
    if (rows <= 0 || d <= 0) return;
    int64_t blocks = rows < 4096 ? rows : 4096;
    const int threads = d < 256 ? ((d + 31) / 32) * 32 : 256;
    colsq_f64_kernel<<<(unsigned)blocks, threads, 0, st>>>(m, rows, d, colsq);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

__global__ void kv_dequant_f64_kernel(const uint8_t* __restrict__ codes, const float* __restrict__ scales,
                                      int64_t rows, int d_e, int bits, int group, double* __restrict__ dst) {
    const int64_t total = rows * d_e;
    const int64_t stride = (int64_t)gridDim.x * blockDim.x;
    const int rb = d_e * bits / 8, ng = d_e / group;
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < total; i += stride) {
        const int64_t r = i / d_e;
        const int c = (int)(i - r * d_e);
        int code;
        if (bits == 8) {
            code = (int)(int8_t)codes[r * rb + c];
        } else {
            const int nib = (codes[r * rb + (c >> 1)] >> ((c & 1) * 4)) & 0xF;
            code = nib >= 8 ? nib - 16 : nib;
        }
        dst[i] = (double)code * (double)scales[r * ng + c / group];
    }
}

void launch_kv_dequant_f64(const void* codes, const float* scales, int64_t rows, int d_e, int bits,
                           int group, double* dst, cudaStream_t st) {
    if (rows <= 0) return;
    kv_dequant_f64_kernel<<<grid_1d(rows * d_e, 256), 256, 0, st>>>((const uint8_t*)codes, scales, rows,
                                                                     d_e, bits, group, dst);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

// ---- fp64 reference-order kernels (the C++ mirror's exact paths) --------------
// matmul (matrix.cpp:19-36): out(i,j) = sum_k a(i,k)*b(k,j), accumulated from 0.0
// left to right with separate IEEE multiply and add (no FMA contraction), which
// is what the reference's -O2 x86-64 build computes: the result is bit-identical.
__global__ void matmul_f64_kernel(const double* __restrict__ a, const double* __restrict__ b,
                                  int n, int k, int m, double* __restrict__ out) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    const int i = blockIdx.y;
    if (j >= m) return;
    const double* ar = a + (size_t)i * k;
    double acc = 0.0;
    for (int kk = 0; kk < k; ++kk) acc = __dadd_rn(acc, __dmul_rn(ar[kk], b[(size_t)kk * m + j]));
    out[(size_t)i * m + j] = acc;
}

void launch_matmul_f64(const double* a, const double* b, int n, int k, int m, double* out,
                       cudaStream_t st) {
    if (n <= 0 || m <= 0) return;
    require(n <= 65535, "matmul_f64: at most 65535 rows per launch", EKV_EUNSUPPORTED);
    dim3 grid((m + 127) / 128, n);
    matmul_f64_kernel<<<grid, 128, 0, st>>>(a, b, n, k, m, out);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

// segment_attention_prefix (cache_merge.cpp:12-38) in fp64 and the reference's
// order: logits q.k_j left to right (mul + add, bit-identical), shift = max,
// sigma = sum_j exp(logit_j - shift) in j order, o[c] = sum_j w_j v_j[c] / sigma.
// Only exp() may differ from the host libm, by <= 1 ulp.
__global__ void seg_logits_f64_kernel(const double* __restrict__ q, const double* __restrict__ k,
                                      int n, int d, double* __restrict__ logits) {
    const int j = blockIdx.x * blockDim.x + threadIdx.x;
    if (j >= n) return;
    const double* kr = k + (size_t)j * d;
    double acc = 0.0;
    for (int c = 0; c < d; ++c) acc = __dadd_rn(acc, __dmul_rn(q[c], kr[c]));
    logits[j] = acc;
}

__global__ void seg_reduce_f64_kernel(const double* __restrict__ logits, const double* __restrict__ v,
                                      int n, int vd, double* __restrict__ o, double* __restrict__ stats) {
    __shared__ double s_mx, s_sig;
    if (threadIdx.x == 0) {
        double mx = logits[0];
        for (int j = 1; j < n; ++j) mx = fmax(mx, logits[j]);
        double sig = 0.0;
        for (int j = 0; j < n; ++j) sig = __dadd_rn(sig, exp(logits[j] - mx));
        s_mx = mx;
        s_sig = sig;
        stats[0] = sig;
        stats[1] = mx;
    }
    __syncthreads();
    const double mx = s_mx, sig = s_sig;
    for (int c = threadIdx.x; c < vd; c += blockDim.x) {
        double acc = 0.0;
        for (int j = 0; j < n; ++j) acc = __dadd_rn(acc, __dmul_rn(exp(logits[j] - mx), v[(size_t)j * vd + c]));
        o[c] = __ddiv_rn(acc, sig);
    }
}

void launch_segment_attention_f64(const double* q, const double* k, const double* v, int n, int d,
                                  int vd, double* logits, double* o, double* stats, cudaStream_t st) {
    seg_logits_f64_kernel<<<(n + 127) / 128, 128, 0, st>>>(q, k, n, d, logits);
    EKV_CUDA(cudaGetLastError());
    seg_reduce_f64_kernel<<<1, 128, 0, st>>>(logits, v, n, vd, o, stats);
    EKV_CUDA(cudaGetLastError());
    count_launches(2);
}

}  // namespace ekv
