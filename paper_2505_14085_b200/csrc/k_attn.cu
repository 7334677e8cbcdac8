// K4: edge decode attention over the reused context KV plus the causal user
// segment, merged by the normaliser rule of Eq. 5.
//
// Reference semantics (cache_merge.cpp:12-38, 59-80, 204-214): per query row
// q (d_e wide) the context segment contributes softmax(q.K_ctx^T) V_ctx over
// all S rows and the user segment over the first base+r+1 user rows; logits
// are raw q.k (no 1/sqrt(d)); the two are combined with weights
// sigma_seg * e^{shift_seg - m}.  Here the context is additionally split into
// chunks (split-KV / flash-decoding); every chunk and the user segment emit a
// partial (m, l, o) and the last CTA of each (row, head) merges them with the
// same rule -- mathematically identical to the reference's two-segment merge
// (the merge identity pinned by cache_merge_test.cpp:153-176).
//
// Context rows may be bf16 (local layers) or int8/int4 codes with fp32
// per-row-group scales (cloud layers, contract in DESIGN.md s.3): the
// dequantised value is code*scale; logits use scale * sum(q*code) and the
// value accumulation uses (p*scale) * code, so codes are never materialised.
//
// Layout: one CTA = 4 warps = one (item, head, row).  Each sub-chunk of 128
// rows is loaded with 16-byte lane loads (LPR lanes cover one row, a warp
// covers 32/LPR rows per pass), K and V for the whole sub-chunk are in
// flight before any math, logits go through shared memory for the block
// softmax, and V is accumulated from registers.
#include <math_constants.h>

#include "ekv_common.cuh"
#include "ekv_kernels.h"

namespace ekv {

constexpr int kAttnThreads = 128;
constexpr int kSub = 128;  // rows per sub-chunk (one per thread in the softmax)
constexpr int kUserRows = 256;  // user-segment rows per item (split like the context)
constexpr float kLog2e = 1.4426950408889634f;

template <int D, int FMT>
struct SegT {
    static constexpr int ROW_BYTES = FMT == 16 ? D * 2 : (FMT == 8 ? D : D / 2);
    static constexpr int LPR = ROW_BYTES / 16;  // lanes per row
    static constexpr int EPL = D / LPR;         // elements per lane
    static constexpr int RPP = 32 / LPR;        // rows per warp pass
    static constexpr int PASSES = 32 / RPP;     // passes per warp (32 rows)
    static_assert(LPR >= 1 && LPR <= 32, "unsupported head_dim/format");
};

// Expand one 16-byte lane chunk into EPL floats.
template <int FMT, int EPL>
__device__ __forceinline__ void expand(const uint4& v, float* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if constexpr (FMT == 16) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            f[2 * k] = bf16_lo(w[k]);
            f[2 * k + 1] = bf16_hi(w[k]);
        }
    } else if constexpr (FMT == 8) {
        // signed byte b -> float via 0x4B0000(b^0x80) - (2^23 + 128)
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t u = w[k] ^ 0x80808080u;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                f[4 * k + b] = __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7440 + b)) - 8388736.0f;
        }
    } else {
        // int4: element 2j low nibble of byte j.  nibble n -> (n^8) - 8
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t lo = (w[k] & 0x0F0F0F0Fu) ^ 0x08080808u;
            const uint32_t hi = ((w[k] >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u;
#pragma unroll
            for (int b = 0; b < 4; ++b) {
                f[8 * k + 2 * b] = __uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7440 + b)) - 8388616.0f;
                f[8 * k + 2 * b + 1] = __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7440 + b)) - 8388616.0f;
            }
        }
    }
}

struct BlockScratch {
    float logit[kSub];
    float red[kAttnThreads / 32];
    float bcast;
};

__device__ __forceinline__ float block_max(float v, BlockScratch& s) {
    v = warp_max(v);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) s.red[w] = v;
    __syncthreads();
    float r = s.red[0];
#pragma unroll
    for (int i = 1; i < kAttnThreads / 32; ++i) r = fmaxf(r, s.red[i]);
    __syncthreads();
    return r;
}
__device__ __forceinline__ float block_sum(float v, BlockScratch& s) {
    v = warp_sum(v);
    const int w = threadIdx.x >> 5;
    if ((threadIdx.x & 31) == 0) s.red[w] = v;
    __syncthreads();
    float r = 0.0f;
#pragma unroll
    for (int i = 0; i < kAttnThreads / 32; ++i) r += s.red[i];
    __syncthreads();
    return r;
}

// Online-softmax attention of q over rows [r0, r1) of one segment.  Returns
// the running (m, l) in *m_io / *l_io and leaves the lane-partial unnormalised
// output in acc[EPL] (lanes with equal `sub` hold partial sums over rows).
template <int D, int FMT>
__device__ __forceinline__ void attend_rows(const float* __restrict__ qf, const uint8_t* __restrict__ kb,
                                            const uint8_t* __restrict__ vb,
                                            const float* __restrict__ ks,
                                            const float* __restrict__ vs, int ng, int group,
                                            int r0, int r1, float* m_io, float* l_io, float* acc,
                                            BlockScratch& sc) {
    using T = SegT<D, FMT>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % T::LPR, rsub = lane / T::LPR;
    const int d0 = sub * T::EPL;
    const int grp = (FMT == 16) ? 0 : d0 / group;
    float q[T::EPL];
#pragma unroll
    for (int e = 0; e < T::EPL; ++e) q[e] = qf[d0 + e];
    float m_run = *m_io, l_run = *l_io;
    for (int base = r0; base < r1; base += kSub) {
        uint4 kv[T::PASSES], vv[T::PASSES];
        float ksc[T::PASSES], vsc[T::PASSES];
#pragma unroll
        for (int p = 0; p < T::PASSES; ++p) {
            const int row = base + warp * 32 + p * T::RPP + rsub;
            if (row < r1) {
                kv[p] = ld_stream(kb + (size_t)row * T::ROW_BYTES + sub * 16);
                vv[p] = ld_stream(vb + (size_t)row * T::ROW_BYTES + sub * 16);
                if constexpr (FMT != 16) {
                    ksc[p] = ks[(size_t)row * ng + grp];
                    vsc[p] = vs[(size_t)row * ng + grp];
                }
            } else {
                kv[p] = make_uint4(0, 0, 0, 0);
                vv[p] = make_uint4(0, 0, 0, 0);
                ksc[p] = vsc[p] = 0.0f;
            }
        }
        // logits
#pragma unroll
        for (int p = 0; p < T::PASSES; ++p) {
            float f[T::EPL];
            expand<FMT, T::EPL>(kv[p], f);
            float dot = 0.0f;
#pragma unroll
            for (int e = 0; e < T::EPL; ++e) dot = fmaf(q[e], f[e], dot);
            if constexpr (FMT != 16) dot *= ksc[p];
#pragma unroll
            for (int o = T::LPR >> 1; o > 0; o >>= 1) dot += __shfl_xor_sync(0xffffffffu, dot, o);
            const int lrow = warp * 32 + p * T::RPP + rsub;
            if (sub == 0) sc.logit[lrow] = (base + lrow < r1) ? dot : -CUDART_INF_F;
        }
        __syncthreads();
        const float my = sc.logit[threadIdx.x];
        const float m_chunk = block_max(my, sc);
        const float m_new = fmaxf(m_run, m_chunk);
        const float p_my = (my == -CUDART_INF_F) ? 0.0f : exp2f((my - m_new) * kLog2e);
        sc.logit[threadIdx.x] = p_my;  // reuse as probabilities (own slot only)
        const float l_chunk = block_sum(p_my, sc);  // contains __syncthreads
        const float corr = (m_run == -CUDART_INF_F) ? 0.0f : exp2f((m_run - m_new) * kLog2e);
        l_run = l_run * corr + l_chunk;
        m_run = m_new;
#pragma unroll
        for (int e = 0; e < T::EPL; ++e) acc[e] *= corr;
        // values
#pragma unroll
        for (int p = 0; p < T::PASSES; ++p) {
            const int lrow = warp * 32 + p * T::RPP + rsub;
            float w = sc.logit[lrow];
            if constexpr (FMT != 16) w *= vsc[p];
            float f[T::EPL];
            expand<FMT, T::EPL>(vv[p], f);
#pragma unroll
            for (int e = 0; e < T::EPL; ++e) acc[e] = fmaf(w, f[e], acc[e]);
        }
        __syncthreads();  // logit slots are rewritten by the next sub-chunk
    }
    *m_io = m_run;
    *l_io = l_run;
}

// Fold the lanes that hold the same dims (xor over the row-subgroup lane
// bits), then the warps through shared memory; returns via s_o.
template <int D, int FMT>
__device__ __forceinline__ void fold_partial(const float* acc, float (*s_o)[D]) {
    using T = SegT<D, FMT>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % T::LPR;
#pragma unroll
    for (int e = 0; e < T::EPL; ++e) {
        float v = acc[e];
#pragma unroll
        for (int o = T::LPR; o < 32; o <<= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
        if (lane < T::LPR) s_o[warp][sub * T::EPL + e] = v;
    }
}

template <int D, int FMT>
__global__ void __launch_bounds__(kAttnThreads) decode_attn_kernel(AttnArgs a, int rows_per_item,
                                                                   int n_ctx_items) {
    __shared__ BlockScratch sc;
    __shared__ float s_o[kAttnThreads / 32][D];
    __shared__ int s_last;
    const int item = blockIdx.x, h = blockIdx.y, r = blockIdx.z;
    const int n_items = gridDim.x;  // context items, then user items of kUserRows rows
    const float* qf = a.q + ((size_t)r * a.H + h) * D;
    float m = -CUDART_INF_F, l = 0.0f;
    if (item < n_ctx_items) {
        using T = SegT<D, FMT>;
        const int r0 = item * rows_per_item;
        const int r1 = min(a.S, r0 + rows_per_item);
        const int ng = (FMT == 16) ? 1 : D / a.group;
        const size_t hoff = (size_t)h * a.S;
        float acc[T::EPL];
#pragma unroll
        for (int e = 0; e < T::EPL; ++e) acc[e] = 0.0f;
        attend_rows<D, FMT>(qf, (const uint8_t*)a.ck + hoff * T::ROW_BYTES,
                            (const uint8_t*)a.cv + hoff * T::ROW_BYTES,
                            FMT == 16 ? nullptr : a.cks + hoff * ng,
                            FMT == 16 ? nullptr : a.cvs + hoff * ng, ng, a.group, r0, r1, &m, &l,
                            acc, sc);
        fold_partial<D, FMT>(acc, s_o);
    } else {
        using T = SegT<D, 16>;
        const int base = a.user_base_dev ? *a.user_base_dev : a.user_base;
        const int vis = base + r + 1;
        const int u0 = (item - n_ctx_items) * kUserRows;
        const int u1 = min(vis, u0 + kUserRows);  // u0 >= u1: empty partial (l = 0)
        const size_t hoff = (size_t)h * a.ucap;
        float acc[T::EPL];
#pragma unroll
        for (int e = 0; e < T::EPL; ++e) acc[e] = 0.0f;
        attend_rows<D, 16>(qf, (const uint8_t*)(a.uk + hoff * D), (const uint8_t*)(a.uv + hoff * D),
                           nullptr, nullptr, 1, D, u0, u1, &m, &l, acc, sc);
        fold_partial<D, 16>(acc, s_o);
    }
    __syncthreads();
    float* part = a.ws + (((size_t)r * a.H + h) * n_items + item) * (D + 2);
    for (int c = threadIdx.x; c < D; c += kAttnThreads) {
        float v = 0.0f;
#pragma unroll
        for (int w = 0; w < kAttnThreads / 32; ++w) v += s_o[w][c];
        part[2 + c] = v;
    }
    if (threadIdx.x == 0) {
        part[0] = m;
        part[1] = l;
    }
    // last CTA of this (row, head) merges all partials (Eq. 5, generalised)
    __threadfence();
    __syncthreads();
    if (threadIdx.x == 0) {
        unsigned* ctr = a.counters + (size_t)r * a.H + h;
        const unsigned prev = atomicAdd(ctr, 1u);
        s_last = (prev == (unsigned)n_items - 1);
        if (s_last) *ctr = 0u;  // re-arm for the next launch / graph replay
    }
    __syncthreads();
    if (!s_last) return;
    __threadfence();
    const float* parts = a.ws + ((size_t)r * a.H + h) * n_items * (D + 2);
    float M = -CUDART_INF_F;
    for (int i = 0; i < n_items; ++i) {
        const float li = __ldcg(parts + (size_t)i * (D + 2) + 1);
        if (li > 0.0f) M = fmaxf(M, __ldcg(parts + (size_t)i * (D + 2)));
    }
    float Lsum = 0.0f;
    for (int i = 0; i < n_items; ++i) {
        const float li = __ldcg(parts + (size_t)i * (D + 2) + 1);
        if (li > 0.0f) Lsum += li * exp2f((__ldcg(parts + (size_t)i * (D + 2)) - M) * kLog2e);
    }
    const float inv = 1.0f / Lsum;
    for (int c = threadIdx.x; c < D; c += kAttnThreads) {
        float o = 0.0f;
        for (int i = 0; i < n_items; ++i) {
            const float* pi = parts + (size_t)i * (D + 2);
            const float li = __ldcg(pi + 1);
            if (li > 0.0f) o += __ldcg(pi + 2 + c) * exp2f((__ldcg(pi) - M) * kLog2e);
        }
        a.out[((size_t)r * a.H + h) * D + c] = o * inv;
    }
    if (a.lse && threadIdx.x == 0) a.lse[(size_t)r * a.H + h] = M + logf(Lsum);
}

int attn_user_items(int ucap) { return (ucap + kUserRows - 1) / kUserRows; }

int attn_items(int R, int H, int S, int* rows_per_item) {
    if (S <= 0) {
        *rows_per_item = kSub;
        return 0;
    }
    // aim for ~4 CTAs per SM over the context items
    int target = (148 * 4 + H * R - 1) / (H * R);
    if (R > 1) {  // prefill chunks: a power-of-two item count splits S into equal items
        int p2 = 1;
        while (p2 < target) p2 <<= 1;
        target = p2;  // (R = 8, S = 2048: 4 items of 512 rows: 2.77 ms vs 2.99 ms for 3 of 768/512)
    }
    if (target < 1) target = 1;
    int rpi = (S + target - 1) / target;
    rpi = ((rpi + kSub - 1) / kSub) * kSub;
    *rows_per_item = rpi;
    return (S + rpi - 1) / rpi;
}

template <int D>
static void launch_d(const AttnArgs& a, int rpi, int nci, cudaStream_t st) {
    dim3 grid(nci + attn_user_items(a.ucap), a.H, a.R);
    switch (a.fmt) {
        case 16: decode_attn_kernel<D, 16><<<grid, kAttnThreads, 0, st>>>(a, rpi, nci); break;
        case 8: decode_attn_kernel<D, 8><<<grid, kAttnThreads, 0, st>>>(a, rpi, nci); break;
        case 4: decode_attn_kernel<D, 4><<<grid, kAttnThreads, 0, st>>>(a, rpi, nci); break;
        default: require(false, "decode_attention: unsupported context format", EKV_EUNSUPPORTED);
    }
}

void launch_decode_attention(const AttnArgs& a, cudaStream_t st) {
    int rpi = kSub;
    const int nci = attn_items(a.R, a.H, a.S, &rpi);
    switch (a.D) {
        case 32: launch_d<32>(a, rpi, nci, st); break;
        case 64: launch_d<64>(a, rpi, nci, st); break;
        case 128: launch_d<128>(a, rpi, nci, st); break;
        default: require(false, "decode_attention: head_dim must be 32, 64 or 128", EKV_EUNSUPPORTED);
    }
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

}  // namespace ekv
