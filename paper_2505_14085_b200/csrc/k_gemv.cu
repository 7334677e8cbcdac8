// K5: the edge model's projections at decode batch sizes (R <= 8 rows):
// y[r][n] = sum_k x[r][k] * W[n][k], W bf16 out-feature-major [N][K], fp32
// inputs and accumulation.  This is project_qkv (transformer.cpp:133-152)
// for all heads of a layer at once plus matmul(concat, out_proj)
// (cache_merge.cpp:219), and it is HBM-bound (every weight byte is read once
// per step): one warp per output row, 16-byte streaming loads of the whole
// row in flight before the FMAs, x staged once per CTA in shared memory
// (held in registers when R == 1), warp-shuffle reduction.
//
// Fusions: the layer-0 input transform x0 = gamma*(emb + pos) + b
// (cache_merge.cpp:167-177) is applied while staging x, and the QKV epilogue
// scatters K and V straight into the session's bf16 user cache at the row
// the reference appends (cache_merge.cpp:189-199), so no separate append or
// transform kernels run.
#include "ekv_common.cuh"
#include "ekv_kernels.h"

namespace ekv {

constexpr int kGemvThreads = 256;

template <int KC>
__device__ __forceinline__ void load_row(const uint16_t* __restrict__ W, int n, int lane, uint4* w) {
    const uint16_t* wrow = W + (size_t)n * (KC * 256);
#pragma unroll
    for (int c = 0; c < KC; ++c) w[c] = ld_stream(wrow + c * 256 + lane * 8);
}

template <int R, int KC>
__global__ void __launch_bounds__(kGemvThreads) gemv_kernel(GemvArgs a) {
    extern __shared__ float xs[];  // [R][K]
    const int K = KC * 256;
    const int lane = threadIdx.x & 31;
    const int warp = (blockIdx.x * kGemvThreads + threadIdx.x) >> 5;
    const int nwarps = (gridDim.x * kGemvThreads) >> 5;
    // The weight stream does not depend on x: put the first row's loads in
    // flight before staging x so HBM latency overlaps the staging.
    uint4 w[KC];
    int n = warp;
    if (n < a.N) load_row<KC>(a.W, n, lane, w);
    // ---- stage x (with the optional layer-0 input transform) ----
    int p0 = 0;
    if (a.pos) p0 = a.pos_offset + (a.pos_base_dev ? *a.pos_base_dev : a.pos_base);
    for (int i = threadIdx.x; i < R * K; i += kGemvThreads) {
        const int r = i / K, k = i - r * K;
        float v = (r < a.R) ? a.x[(size_t)r * K + k] : 0.0f;
        if (a.pos && r < a.R) {
            const float pe = __uint_as_float((uint32_t)a.pos[(size_t)(p0 + r) * K + k] << 16);
            v = a.gamma[k] * (v + pe) + a.bias[k];
        }
        xs[i] = v;
    }
    __syncthreads();
    int ubase = 0;
    if (a.mode == 1) ubase = a.user_base + (a.user_base_dev ? *a.user_base_dev : 0);
    int hrow = 0;
    if (a.y_hist) hrow = a.hist_row_dev ? *a.hist_row_dev : 0;

    float xr[R == 1 ? KC * 8 : 1];
    if constexpr (R == 1) {
#pragma unroll
        for (int c = 0; c < KC; ++c)
#pragma unroll
            for (int e = 0; e < 8; ++e) xr[c * 8 + e] = xs[c * 256 + lane * 8 + e];
    }
    for (; n < a.N; n += nwarps) {
        uint4 wn[KC];
        const int nn = n + nwarps;
        if (nn < a.N) load_row<KC>(a.W, nn, lane, wn);  // software pipeline: next row in flight
        float acc[R];
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = 0.0f;
#pragma unroll
        for (int c = 0; c < KC; ++c) {
            const uint32_t ww[4] = {w[c].x, w[c].y, w[c].z, w[c].w};
            float wf[8];
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                wf[2 * k] = bf16_lo(ww[k]);
                wf[2 * k + 1] = bf16_hi(ww[k]);
            }
            if constexpr (R == 1) {
#pragma unroll
                for (int e = 0; e < 8; ++e) acc[0] = fmaf(wf[e], xr[c * 8 + e], acc[0]);
            } else {
#pragma unroll
                for (int r = 0; r < R; ++r) {
                    const float4* xp = reinterpret_cast<const float4*>(xs + r * K + c * 256 + lane * 8);
                    const float4 x0 = xp[0], x1 = xp[1];
                    acc[r] = fmaf(wf[0], x0.x, acc[r]);
                    acc[r] = fmaf(wf[1], x0.y, acc[r]);
                    acc[r] = fmaf(wf[2], x0.z, acc[r]);
                    acc[r] = fmaf(wf[3], x0.w, acc[r]);
                    acc[r] = fmaf(wf[4], x1.x, acc[r]);
                    acc[r] = fmaf(wf[5], x1.y, acc[r]);
                    acc[r] = fmaf(wf[6], x1.z, acc[r]);
                    acc[r] = fmaf(wf[7], x1.w, acc[r]);
                }
            }
        }
#pragma unroll
        for (int r = 0; r < R; ++r) acc[r] = warp_sum(acc[r]);
        if (lane < R && lane < a.R) {
            float v = acc[0];
#pragma unroll
            for (int r = 1; r < R; ++r)
                if (lane == r) v = acc[r];
            const int r = lane;
            if (a.mode == 0) {
                a.y[(size_t)r * a.N + n] = v;
                if (a.y_hist) a.y_hist[(size_t)(hrow + r) * a.N + n] = v;
            } else {
                const int hd = a.qkv_H * a.qkv_d;
                const int part = n / hd, rem = n - part * hd;
                if (part == 0) {
                    a.q_out[(size_t)r * hd + rem] = v;
                } else {
                    const int head = rem / a.qkv_d, c = rem - head * a.qkv_d;
                    uint16_t* dst = part == 1 ? a.uk : a.uv;
                    dst[((size_t)head * a.ucap + ubase + r) * a.qkv_d + c] = f32_to_bf16_bits(v);
                }
            }
        }
#pragma unroll
        for (int c = 0; c < KC; ++c) w[c] = wn[c];
    }
}

template <int R>
static void launch_r(const GemvArgs& a, cudaStream_t st) {
    const int kc = a.K / 256;
    const size_t smem = (size_t)R * a.K * sizeof(float);
    int blocks = (a.N + (kGemvThreads / 32) - 1) / (kGemvThreads / 32);
    if (blocks > 148 * 4) blocks = 148 * 4;
#define EKV_GEMV_CASE(KC)                                                                        \
    case KC: {                                                                                   \
        auto fn = gemv_kernel<R, KC>;                                                            \
        if (smem > 48 * 1024) ensure_smem_attr((const void*)fn, (int)smem);                      \
        fn<<<blocks, kGemvThreads, smem, st>>>(a);                                               \
        break;                                                                                   \
    }
    switch (kc) {
        EKV_GEMV_CASE(1)
        EKV_GEMV_CASE(2)
        EKV_GEMV_CASE(4)
        EKV_GEMV_CASE(8)
        EKV_GEMV_CASE(16)
        default: require(false, "gemv: K must be 256, 512, 1024, 2048 or 4096", EKV_EUNSUPPORTED);
    }
#undef EKV_GEMV_CASE
}

void launch_gemv(const GemvArgs& a, cudaStream_t st) {
    require(a.R >= 1 && a.R <= 8, "gemv: 1..8 rows per launch");
    if (a.R == 1) launch_r<1>(a, st);
    else if (a.R == 2) launch_r<2>(a, st);
    else if (a.R <= 4) launch_r<4>(a, st);
    else launch_r<8>(a, st);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

__global__ void advance_kernel(DevState* s, int n) {
    s->user_len += n;
    s->step += 1;
}

void launch_advance(DevState* s, int n, cudaStream_t st) {
    advance_kernel<<<1, 1, 0, st>>>(s, n);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

}  // namespace ekv
