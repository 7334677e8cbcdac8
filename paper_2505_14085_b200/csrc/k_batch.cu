// Batched collaborative decode: B concurrent edge sessions that share one
// assembled context (the paper's shared system prompt; the
// reference serves every request with its own user cache over one read-only
// context cache, cache_merge.cpp:252) advance one row per step
// in lock-step.  Per session the arithmetic is merged_forward
// (cache_merge.cpp:156-226); the kernels below change only how the work of
// the B sessions is laid out on the B200:
//
//   K9  batch_proj_kernel   y^T[n][b] = W[n][:] . x[b][:] on tcgen05 (swap-AB:
//                           the weight rows are the M=128 side, the sessions the
//                           N side), x split into bf16 hi + lo halves (two MMAs
//                           into one fp32 TMEM accumulator: ~2^-17 input
//                           precision), split-K partials written, not atomically
//                           added (deterministic).  Every weight byte is read
//                           once per step for all B sessions.
//   K10 batch_ctx_attn_kernel  the context segment (segment_attention over the S
//                           shared rows, cache_merge.cpp:12-38) of all sessions
//                           of a head as a cascade: S = Q K^T and O = P V on
//                           tcgen05 (Q and P also split hi + lo), online
//                           softmax on the CUDA cores, K/V chunks moved by TMA;
//                           every context byte is read once per step.
//   K11 batch_user_merge_kernel  per (session, head): this step's K/V appended
//                           to the session's bf16 user cache, the user segment
//                           (causal over the session's own rows), the Eq. 5
//                           merge with the context partials
//                           (merge_attention, cache_merge.cpp:59-80), output
//                           split hi + lo as the next projection's operand.
//   K12 batch_xprep_kernel  sums split-K partials; layer-0 input transform
//                           (cache_merge.cpp:167-177); final-layer output row.
#include "ekv_common.cuh"
#include "ekv_batch.h"
#include "ekv_tc.cuh"

namespace ekv {

using namespace tc;

constexpr int kMaxSplitK = 16;

// Programmatic dependent launch: every kernel of the batched row is launched with
// programmatic stream serialization, so the next kernel's CTAs are scheduled while
// this one drains; pdl_wait() blocks until the previous kernel has completed and its
// writes are visible.  Only static data (weights, context) is read before it.
__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" ::: "memory"); }

// packed fp32x2 arithmetic (sm_100: FFMA2 / FADD2 / FMUL2), IEEE per lane
typedef unsigned long long f2x;
__device__ __forceinline__ f2x f2pack(float lo, float hi) {
    f2x r;
    asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(lo), "f"(hi));
    return r;
}
__device__ __forceinline__ float f2lo(f2x v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return lo;
}
__device__ __forceinline__ float f2hi(f2x v) {
    float lo, hi;
    asm("mov.b64 {%0, %1}, %2;" : "=f"(lo), "=f"(hi) : "l"(v));
    return hi;
}
__device__ __forceinline__ f2x ffma2(f2x a, f2x b, f2x c) {
    f2x d;
    asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(d) : "l"(a), "l"(b), "l"(c));
    return d;
}
__device__ __forceinline__ f2x fadd2(f2x a, f2x b) {
    f2x d;
    asm("add.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
__device__ __forceinline__ f2x fmul2(f2x a, f2x b) {
    f2x d;
    asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(d) : "l"(a), "l"(b));
    return d;
}
// a bf16 pair word -> {low element, high element} as fp32
__device__ __forceinline__ f2x bf16x2_to_f2(uint32_t w) {
    return f2pack(__uint_as_float(w << 16), __uint_as_float(w & 0xFFFF0000u));
}

// sum of the KS split-K partials of 4 consecutive floats (16-byte aligned); every
// load is issued before the first add (the split loop is unrolled to kMaxSplitK
// with a predicate), so the sum costs one memory round trip, not KS.
__device__ __forceinline__ float4 sum_splits4(const float* p, size_t stride, int KS) {
    float4 v[kMaxSplitK];
#pragma unroll
    for (int s = 0; s < kMaxSplitK; ++s)
        if (s < KS) v[s] = *reinterpret_cast<const float4*>(p + s * stride);
    float4 r = v[0];
#pragma unroll
    for (int s = 1; s < kMaxSplitK; ++s)
        if (s < KS) {
            r.x += v[s].x;
            r.y += v[s].y;
            r.z += v[s].z;
            r.w += v[s].w;
        }
    return r;
}

// ============================================================================
// K9: projection GEMM  out[ks][b][n] = sum_{k in split ks} W[w_row0 + n][k] * x[b][k]
// ============================================================================
namespace k9 {
constexpr int BM = 128, BK = 64, THREADS = 256;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB weight tile

__global__ void __launch_bounds__(THREADS, 1)
    batch_proj_kernel(const __grid_constant__ CUtensorMap map_w, const __grid_constant__ CUtensorMap map_x,
                      int w_row0, int N_out, int K, int B, int BN, int KS, int stages, uint32_t idesc,
                      float* __restrict__ out) {
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    const int x_bytes = BN * BK * 2;              // one of hi / lo
    const int stage_bytes = A_BYTES + 2 * x_bytes;
    uint64_t* bars = (uint64_t*)(smem + stages * stage_bytes);
    uint64_t* full = bars;
    uint64_t* empty = bars + stages;
    uint64_t* tfull = bars + 2 * stages;
    uint32_t* tmem_slot = (uint32_t*)(tfull + 1);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mt = blockIdx.x, nt = blockIdx.y, ks = blockIdx.z;
    const int kblocks = K / BK;
    const int kb0 = (int)((long long)ks * kblocks / KS), kb1 = (int)((long long)(ks + 1) * kblocks / KS);
    const uint32_t tcols = BN <= 32 ? 32 : (BN <= 64 ? 64 : (BN <= 128 ? 128 : 256));  // power of 2

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
        for (int i = 0; i < stages; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        mbar_init(tfull, 1);
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, tcols);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            // weight tiles of the first ring slots do not depend on the previous kernel:
            // issue them before waiting for it, then the activation tiles
            const int npre = min(stages, kb1 - kb0);
            for (int i = 0; i < npre; ++i) {
                mbar_expect_tx(&full[i], stage_bytes);
                tma_load_2d(&map_w, &full[i], smem + i * stage_bytes, (kb0 + i) * BK, w_row0 + mt * BM);
            }
            pdl_wait();
            for (int i = 0; i < npre; ++i) {
                uint8_t* s = smem + i * stage_bytes;
                tma_load_3d(&map_x, &full[i], s + A_BYTES, (kb0 + i) * BK, nt * BN, 0);
                tma_load_3d(&map_x, &full[i], s + A_BYTES + x_bytes, (kb0 + i) * BK, nt * BN, 1);
            }
            int stage = npre == stages ? 0 : npre;
            uint32_t phase = npre == stages ? 1 : 0;
            for (int kb = kb0 + npre; kb < kb1; ++kb) {
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_expect_tx(&full[stage], stage_bytes);
                uint8_t* s = smem + stage * stage_bytes;
                tma_load_2d(&map_w, &full[stage], s, kb * BK, w_row0 + mt * BM);
                tma_load_3d(&map_x, &full[stage], s + A_BYTES, kb * BK, nt * BN, 0);
                tma_load_3d(&map_x, &full[stage], s + A_BYTES + x_bytes, kb * BK, nt * BN, 1);
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int kb = kb0; kb < kb1; ++kb) {
                mbar_wait(&full[stage], phase);
                fence_after();
                const uint32_t a0 = smem_u32(smem + stage * stage_bytes);
                const uint32_t bh = a0 + A_BYTES, bl = bh + x_bytes;
#pragma unroll
                for (int k = 0; k < BK / 16; ++k) {
                    const uint64_t ad = desc_sw128(a0 + k * 32);
                    mma_bf16(tmem, ad, desc_sw128(bh + k * 32), idesc, (kb > kb0) || (k > 0));
                    mma_bf16(tmem, ad, desc_sw128(bl + k * 32), idesc, 1);
                }
                mma_commit(&empty[stage]);
                if (++stage == stages) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            mma_commit(tfull);
        }
    } else if (warp >= 4) {
        const int quad = warp - 4;
        pdl_wait();  // the partial buffer may still be read by the previous kernel's consumers
        mbar_wait(tfull, 0);
        fence_after();
        const uint32_t taddr = tmem + ((uint32_t)(quad * 32) << 16);
        // 32 sessions at a time through shared memory (the drained ring), transposed so
        // each session's 128 outputs leave as 16-byte stores
        constexpr int TS = BM + 4;
        float* tile = reinterpret_cast<float*>(smem);  // [32][TS]
        const int t = threadIdx.x - 128;
        float* o = out + (size_t)ks * B * N_out + mt * BM;
        for (int c = 0; c < BN / 32; ++c) {
            float v[32];
            tmem_ld32(taddr + c * 32, v);
#pragma unroll
            for (int i = 0; i < 32; ++i) tile[i * TS + quad * 32 + lane] = v[i];
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int b0 = nt * BN + c * 32;
#pragma unroll
            for (int k = 0; k < 8; ++k) {
                const int i = t / 32 + 4 * k, n4 = t % 32;
                if (b0 + i < B)
                    *reinterpret_cast<float4*>(o + (size_t)(b0 + i) * N_out + n4 * 4) =
                        *reinterpret_cast<const float4*>(tile + i * TS + n4 * 4);
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
    }
    pdl_trigger();
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 2) tmem_dealloc(tmem, tcols);
}
}  // namespace k9

// ============================================================================
// K12: x preparation.  x[b] = in (mode 0: xin[b]; else sum_ks part[ks][b]);
// layer-0 transform x0 = gamma*(x + pos[S + user_len]) + bias (mode 0);
// final layer (mode 2): x -> hist[step][b] and xin[b].  Writes hi/lo bf16.
// ============================================================================
__global__ void batch_xprep_kernel(BatchXprep a) {
    pdl_wait();
    pdl_trigger();
    const int b = blockIdx.y;
    const int h = a.h;
    const DevState st = *a.state;
    const int p = a.pos_offset + st.user_len + (a.pos_per_row ? a.row0 + b : 0);
    const int k = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (k >= h) return;
    float4 x;
    if (a.mode == 0) {
        x = *reinterpret_cast<const float4*>(a.xin + (size_t)b * h + k);
        const uint2 pw = *reinterpret_cast<const uint2*>(a.pos + (size_t)p * h + k);
        const float4 g = *reinterpret_cast<const float4*>(a.gamma + k);
        const float4 bb = *reinterpret_cast<const float4*>(a.bias + k);
        x.x = g.x * (x.x + bf16_lo(pw.x)) + bb.x;
        x.y = g.y * (x.y + bf16_hi(pw.x)) + bb.y;
        x.z = g.z * (x.z + bf16_lo(pw.y)) + bb.z;
        x.w = g.w * (x.w + bf16_hi(pw.y)) + bb.w;
    } else {
        x = sum_splits4(a.part + (size_t)b * h + k, (size_t)a.B * h, a.KS);
    }
    if (a.mode == 2) {
        *reinterpret_cast<float4*>(a.hist + ((size_t)st.step * a.B + b) * h + k) = x;
        *reinterpret_cast<float4*>(a.xin + (size_t)b * h + k) = x;
    } else {
        uint16_t hi[4], lo[4];
        split_bf16(x.x, hi[0], lo[0]);
        split_bf16(x.y, hi[1], lo[1]);
        split_bf16(x.z, hi[2], lo[2]);
        split_bf16(x.w, hi[3], lo[3]);
        *reinterpret_cast<uint2*>(a.xhl + (size_t)b * h + k) =
            make_uint2(hi[0] | ((uint32_t)hi[1] << 16), hi[2] | ((uint32_t)hi[3] << 16));
        *reinterpret_cast<uint2*>(a.xhl + ((size_t)a.B + b) * h + k) =
            make_uint2(lo[0] | ((uint32_t)lo[1] << 16), lo[2] | ((uint32_t)lo[3] << 16));
    }
}

// ============================================================================
// K10: context attention of B sessions over the shared context, one head and
// one contiguous range of 128-row chunks per CTA.
// ============================================================================
namespace k10 {
constexpr int BT = 128;        // sessions per CTA (MMA M)
constexpr int CH = 128;        // context rows per chunk (MMA N of S = Q K^T; K of O = P V)
constexpr int THREADS = 384;   // warp 0 TMA, 1 MMA, 2-3 TMEM alloc + int8 expansion, 4-11 softmax
                               // (warp w: TMEM lanes 32*(w%4).., score columns / O columns half (w-4)/4)
constexpr int STAGES = 3;

template <int D, int FMT>
struct Cfg {
    static constexpr int ROWB = D * 2;                  // bf16 row bytes (== swizzle width)
    static constexpr int Q_BYTES = BT * ROWB;           // one of Q hi / lo
    static constexpr int KV_BYTES = CH * ROWB;          // one K or V chunk (bf16)
    static constexpr int P_BYTES = BT * CH * 2;         // one of P hi / lo (2 panels of 64 rows)
    static constexpr int CODE_BYTES = CH * D;           // int8 codes of one K or V chunk
    // TMA stage: bf16 -> K, V tiles; int8 -> K, V codes + K, V row scales
    static constexpr int STAGE_BYTES = FMT == 16 ? 2 * KV_BYTES : 2 * CODE_BYTES + 2 * CH * 4;
    // int8: expanded bf16 K, V tiles (+ scales), double-buffered
    static constexpr int XBUF_BYTES = FMT == 16 ? 0 : 2 * KV_BYTES + 2 * CH * 4;
    static constexpr int NXBUF = FMT == 16 ? 0 : 2;
    static constexpr int XCH_BYTES = 2 * 2 * BT * 4 + 2 * BT * 4;  // row-max exchange (2 parities) + l exchange
    static constexpr int SMEM = 2 * Q_BYTES + STAGES * STAGE_BYTES + NXBUF * XBUF_BYTES + 2 * P_BYTES + XCH_BYTES +
                                1024 + 512;
};

__device__ __forceinline__ void st_shared_v4(uint32_t addr, uint32_t a, uint32_t b, uint32_t c, uint32_t d) {
    asm volatile("st.shared.v4.b32 [%0], {%1,%2,%3,%4};" ::"r"(addr), "r"(a), "r"(b), "r"(c), "r"(d)
                 : "memory");
}

__device__ __forceinline__ uint32_t pack2(uint16_t lo, uint16_t hi) { return (uint32_t)lo | ((uint32_t)hi << 16); }

// 4 signed int8 codes -> 2 words of 2 bf16 each (exact: |code| <= 128 fits bf16's 8-bit
// significand).  No integer->float conversion (quarter rate): each biased byte is
// placed in the significand of 2^23 (0x4B0000xx = 2^23 + byte) and the bias removed
// with one packed FADD2 per pair; one PRMT keeps the two high halves.
__device__ __forceinline__ void i8x4_to_bf16x4(uint32_t w, uint32_t& lo, uint32_t& hi) {
    const uint32_t u = w ^ 0x80808080u;  // code + 128, as unsigned bytes
    const f2x bias = f2pack(-8388736.0f, -8388736.0f);  // -(2^23 + 128)
    const f2x a = fadd2(f2pack(__uint_as_float(__byte_perm(u, 0x4B000000u, 0x7440)),
                               __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7441))), bias);
    const f2x b = fadd2(f2pack(__uint_as_float(__byte_perm(u, 0x4B000000u, 0x7442)),
                               __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7443))), bias);
    lo = __byte_perm(__float_as_uint(f2lo(a)), __float_as_uint(f2hi(a)), 0x7632);
    hi = __byte_perm(__float_as_uint(f2lo(b)), __float_as_uint(f2hi(b)), 0x7632);
}

// This row's k / v of head hd for split `split`'s share of the session tile:
// split-K sum, bf16 rounding, append to the user caches (K11 then reads them
// back).  Run by the 64 threads of warps 2-3 (idle on bf16 contexts, free after
// the expansion on int8) while the softmax warps work; every load of a round
// (4 units x up to 4 partials per thread) is issued before the first add.
template <int D>
__device__ __forceinline__ void append_kv(const BatchCtxAttn& a, int hd, int split, int bt, int t) {
    constexpr int NTH = 64, UPT = 4, SPL = 4;
    const int h = a.n_qkv / 3;
    const size_t stride = (size_t)a.B * a.n_qkv;
    const int ulen = a.state->user_len;
    const int rA = split * BT / a.nsplit, rB = (split + 1) * BT / a.nsplit;
    const int nun = (rB - rA) * 2 * (D / 4);
    for (int u0 = t; u0 < nun; u0 += NTH * UPT) {
        float4 v[UPT][SPL];
        const float* src[UPT];
        int bbs[UPT], kvs[UPT], c4s[UPT];
#pragma unroll
        for (int k = 0; k < UPT; ++k) {
            const int u = u0 + k * NTH;
            const int row = rA + u / (2 * (D / 4));
            const int rem = u - (row - rA) * 2 * (D / 4);
            kvs[k] = rem / (D / 4);
            c4s[k] = rem - kvs[k] * (D / 4);
            bbs[k] = (u < nun && bt * BT + row < a.B) ? bt * BT + row : -1;
            src[k] = a.qkv + (size_t)max(bbs[k], 0) * a.n_qkv + (1 + kvs[k]) * h + hd * D + c4s[k] * 4;
#pragma unroll
            for (int s2 = 0; s2 < SPL; ++s2)
                v[k][s2] = (bbs[k] >= 0 && s2 < a.KS) ? *reinterpret_cast<const float4*>(src[k] + s2 * stride)
                                                      : make_float4(0.f, 0.f, 0.f, 0.f);
        }
#pragma unroll
        for (int k = 0; k < UPT; ++k) {
            if (bbs[k] < 0) continue;
            float4 x = v[k][0];
#pragma unroll
            for (int s2 = 1; s2 < SPL; ++s2) {
                x.x += v[k][s2].x; x.y += v[k][s2].y; x.z += v[k][s2].z; x.w += v[k][s2].w;
            }
            for (int s2 = SPL; s2 < a.KS; ++s2) {  // rare: more than 4 splits
                const float4 y = *reinterpret_cast<const float4*>(src[k] + s2 * stride);
                x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
            }
            uint16_t* dst = (kvs[k] == 0 ? a.uk : a.uv) +
                            ((((size_t)bbs[k] * a.L + a.layer) * a.H + hd) * a.cap + ulen) * D + c4s[k] * 4;
            *reinterpret_cast<uint2*>(dst) =
                make_uint2(f32_to_bf16_bits(x.x) | ((uint32_t)f32_to_bf16_bits(x.y) << 16),
                           f32_to_bf16_bits(x.z) | ((uint32_t)f32_to_bf16_bits(x.w) << 16));
        }
    }
}

template <int D, int FMT>
__global__ void __launch_bounds__(THREADS, 1)
    batch_ctx_attn_kernel(const __grid_constant__ CUtensorMap map_k, const __grid_constant__ CUtensorMap map_v,
                          const __grid_constant__ CUtensorMap map_ks, const __grid_constant__ CUtensorMap map_vs,
                          BatchCtxAttn a) {
    static_assert(D == 64, "batched context attention: head_dim 64");
    static_assert(FMT == 16 || FMT == 8, "batched context attention: bf16 or int8 context");
    using C = Cfg<D, FMT>;
    constexpr bool Q8 = FMT == 8;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sQ = smem;                                   // hi, lo
    uint8_t* sP = sQ + 2 * C::Q_BYTES;                    // hi (2 panels), lo (2 panels)
    uint8_t* sX = sP + 2 * C::P_BYTES;                    // int8: 2 x {K bf16, V bf16, ks, vs}
    uint8_t* sKV = sX + C::NXBUF * C::XBUF_BYTES;         // STAGES x TMA stage
    float* xch = (float*)(sKV + STAGES * C::STAGE_BYTES);  // [2][2][BT] row max, [2][BT] row sum
    uint64_t* bars = (uint64_t*)(xch + 6 * BT);
    uint64_t* full = bars;                 // [STAGES] TMA -> MMA (bf16) / expanders (int8)
    uint64_t* empty = bars + STAGES;       // [STAGES] MMA (bf16) / expanders (int8) -> TMA
    uint64_t* qready = bars + 2 * STAGES;  // softmax warps -> MMA (Q staged), count 4
    uint64_t* sfull = qready + 1;          // [2] MMA -> softmax (S buffer b in TMEM)
    uint64_t* sfree = sfull + 2;           // [2] softmax -> MMA (S buffer b read), count 8
    uint64_t* pready = sfree + 2;          // softmax -> MMA (P staged), count 8
    uint64_t* ofull = pready + 1;          // MMA -> softmax (O chunk in TMEM)
    uint64_t* xready = ofull + 1;          // [2] expanders -> MMA + softmax, count 2
    uint64_t* xfree = xready + 2;          // [2] MMA -> expanders
    uint32_t* tmem_slot = (uint32_t*)(xfree + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int hd = blockIdx.x, split = blockIdx.y, bt = blockIdx.z;
    const int nchunks = (a.S + CH - 1) / CH;
    const int c0 = (int)((long long)split * nchunks / a.nsplit);
    const int c1 = (int)((long long)(split + 1) * nchunks / a.nsplit);
    const int nloc = c1 - c0;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_k) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_v) : "memory");
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], Q8 ? 2 : 1);
        }
        mbar_init(qready, 8);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&sfull[i], 1);
            mbar_init(&sfree[i], 8);
        }
        mbar_init(pready, 8);
        mbar_init(ofull, 1);
        for (int i = 0; i < 2; ++i) {
            mbar_init(&xready[i], 2);
            mbar_init(&xfree[i], 1);
        }
        fence_barrier_init();
    }
    if (warp == 2) tmem_alloc(tmem_slot, 512);
    fence_before();
    __syncthreads();
    fence_after();
    const uint32_t tmem = *tmem_slot;
    // two S buffers (QK^T of chunk i+1 runs while chunk i is in the softmax) + O
    const uint32_t tO = tmem + 2 * CH;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int c = c0; c < c1; ++c) {
                mbar_wait(&empty[stage], phase ^ 1);
                mbar_expect_tx(&full[stage], C::STAGE_BYTES);
                uint8_t* s = sKV + stage * C::STAGE_BYTES;
                const int row = hd * a.S + c * CH;
                if constexpr (Q8) {
                    tma_load_2d(&map_k, &full[stage], s, 0, row);
                    tma_load_2d(&map_v, &full[stage], s + C::CODE_BYTES, 0, row);
                    tma_load_1d(&map_ks, &full[stage], s + 2 * C::CODE_BYTES, row);
                    tma_load_1d(&map_vs, &full[stage], s + 2 * C::CODE_BYTES + CH * 4, row);
                } else {
                    tma_load_2d(&map_k, &full[stage], s, 0, row);
                    tma_load_2d(&map_v, &full[stage], s + C::KV_BYTES, 0, row);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            const uint32_t idS = idesc_bf16(BT, CH);
            const uint32_t idO = idesc_bf16(BT, D, false, true);  // V is MN-major (d contiguous)
            const uint32_t q0 = smem_u32(sQ), q1 = q0 + C::Q_BYTES;
            const uint32_t p0 = smem_u32(sP), p1 = p0 + C::P_BYTES;
            mbar_wait(qready, 0);
            fence_after();
            // K (and V) tiles of chunk j: the TMA stage (bf16) or the expanded buffer (int8)
            auto kv_of = [&](int j) -> uint32_t {
                if constexpr (Q8) {
                    mbar_wait(&xready[j & 1], (j >> 1) & 1);
                    return smem_u32(sX + (j & 1) * C::XBUF_BYTES);
                } else {
                    mbar_wait(&full[j % STAGES], (j / STAGES) & 1);
                    return smem_u32(sKV + (j % STAGES) * C::STAGE_BYTES);
                }
            };
            auto issue_qk = [&](int j, uint32_t kb) {
                mbar_wait(&sfree[j & 1], ((j >> 1) & 1) ^ 1);  // S buffer of chunk j-2 consumed
                fence_after();
                const uint32_t tS = tmem + (j & 1) * CH;
#pragma unroll
                for (int k = 0; k < D / 16; ++k) {
                    const uint64_t bd = desc_sw128(kb + k * 32);
                    mma_bf16(tS, desc_sw128(q0 + k * 32), bd, idS, k > 0);
                    mma_bf16(tS, desc_sw128(q1 + k * 32), bd, idS, 1);
                }
                mma_commit(&sfull[j & 1]);
            };
            uint32_t kb_cur = 0;
            if (nloc > 0) {
                kb_cur = kv_of(0);
                issue_qk(0, kb_cur);
            }
            for (int i = 0; i < nloc; ++i) {
                // S of the next chunk first: it runs on the tensor pipe while this chunk's
                // softmax is computed
                uint32_t kb_next = 0;
                if (i + 1 < nloc) {
                    kb_next = kv_of(i + 1);
                    issue_qk(i + 1, kb_next);
                }
                mbar_wait(pready, i & 1);
                fence_after();
                const uint32_t vb = kb_cur + C::KV_BYTES;
                // O = P V: K dimension = the 128 chunk rows (2 panels of 64), 16 per MMA;
                // V rows are 128-byte MN-major rows, 8-row atoms 1024 B apart.
#pragma unroll
                for (int k = 0; k < CH / 16; ++k) {
                    const uint32_t poff = (k >> 2) * (BT * 128) + (k & 3) * 32;
                    const uint64_t vd = desc_sw128(vb + k * 16 * C::ROWB, 16, 1024);
                    mma_bf16(tO, desc_sw128(p0 + poff), vd, idO, k > 0);
                    mma_bf16(tO, desc_sw128(p1 + poff), vd, idO, 1);
                }
                mma_commit(ofull);
                if constexpr (Q8) mma_commit(&xfree[i & 1]);
                else mma_commit(&empty[i % STAGES]);
                kb_cur = kb_next;
            }
        }
    } else if (warp < 4) {
        if constexpr (!Q8) {
            if (a.qfin) {
                pdl_wait();  // the QKV partials come from the previous kernel
                append_kv<D>(a, hd, split, bt, threadIdx.x - 64);
            }
        }
        if constexpr (Q8) {
            // expand int8 codes to bf16 K-major / MN-major SW128 tiles (identical physical layout)
            const int t = threadIdx.x - 64;  // 0..63
            int stage = 0;
            uint32_t phase = 0;
            for (int i = 0; i < nloc; ++i) {
                mbar_wait(&full[stage], phase);
                mbar_wait(&xfree[i & 1], ((i >> 1) & 1) ^ 1);
                const uint8_t* s = sKV + stage * C::STAGE_BYTES;
                uint8_t* x = sX + (i & 1) * C::XBUF_BYTES;
                const uint32_t xb = smem_u32(x);
#pragma unroll 4
                for (int u = t; u < 2 * CH * (D / 16); u += 64) {
                    const int kv = u / (CH * (D / 16));
                    const int rem = u - kv * (CH * (D / 16));
                    const int r = rem / (D / 16), q = rem - r * (D / 16);
                    const uint4 w = *reinterpret_cast<const uint4*>(s + kv * C::CODE_BYTES + r * D + q * 16);
                    uint32_t e[8];
                    i8x4_to_bf16x4(w.x, e[0], e[1]);
                    i8x4_to_bf16x4(w.y, e[2], e[3]);
                    i8x4_to_bf16x4(w.z, e[4], e[5]);
                    i8x4_to_bf16x4(w.w, e[6], e[7]);
                    const uint32_t base = xb + kv * C::KV_BYTES;
                    st_shared_v4(base + sw128_off(r, 2 * q), e[0], e[1], e[2], e[3]);
                    st_shared_v4(base + sw128_off(r, 2 * q + 1), e[4], e[5], e[6], e[7]);
                }
                // row scales (K then V)
                for (int u = t; u < 2 * CH / 4; u += 64)
                    reinterpret_cast<uint4*>(x + 2 * C::KV_BYTES)[u] =
                        reinterpret_cast<const uint4*>(s + 2 * C::CODE_BYTES)[u];
                fence_async_smem();
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&empty[stage]);
                    mbar_arrive(&xready[i & 1]);
                }
                if (++stage == STAGES) {
                    stage = 0;
                    phase ^= 1;
                }
            }
            if (a.qfin) {  // after the last expansion: overlaps the last chunks' softmax
                pdl_wait();
                append_kv<D>(a, hd, split, bt, threadIdx.x - 64);
            }
        }
    } else {
        const int quad = warp & 3;                  // TMEM lane quadrant of this warp
        const int half = (warp - 4) >> 2;           // score columns [64h, 64h+64), O columns [32h, 32h+32)
        const int r = quad * 32 + lane;             // session row of this CTA's tile
        const int b = bt * BT + r;
        const bool live = b < a.B;
        const uint32_t lane_off = (uint32_t)(quad * 32) << 16;
        const int pair_bar = 1 + quad;              // named barrier of warps quad+4 and quad+8
        const bool warp_live = bt * BT + quad * 32 < a.B;  // some session row of this warp exists
        pdl_wait();  // q comes from the previous kernel (the context K/V are static)
        // ---- stage q (sum of the split-K partials of the QKV projection) as hi / lo:
        //      256 threads, coalesced 16-byte loads, 4 rows' loads in flight per thread ----
        {
            const uint32_t qh = smem_u32(sQ), ql = qh + C::Q_BYTES;
            const int t = threadIdx.x - 128;
            const size_t stride = (size_t)a.B * a.n_qkv;
            constexpr int NU = BT * (D / 4) / 256;  // float4 units per thread (8)
#pragma unroll
            for (int g = 0; g < NU / 4; ++g) {
                float4 v[4][4];
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int u = t + (g * 4 + k) * 256;
                    const int row = u / (D / 4), c4 = u - row * (D / 4);
                    const int bb = bt * BT + row;
                    const float* src = a.qkv + (size_t)bb * a.n_qkv + hd * D + c4 * 4;
#pragma unroll
                    for (int s2 = 0; s2 < 4; ++s2)
                        v[k][s2] = (bb < a.B && s2 < a.KS) ? *reinterpret_cast<const float4*>(src + s2 * stride)
                                                           : make_float4(0.f, 0.f, 0.f, 0.f);
                }
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const int u = t + (g * 4 + k) * 256;
                    const int row = u / (D / 4), c4 = u - row * (D / 4);
                    const int bb = bt * BT + row;
                    float4 x = v[k][0];
#pragma unroll
                    for (int s2 = 1; s2 < 4; ++s2) {
                        x.x += v[k][s2].x; x.y += v[k][s2].y; x.z += v[k][s2].z; x.w += v[k][s2].w;
                    }
                    for (int s2 = 4; s2 < a.KS && bb < a.B; ++s2) {  // rare: more than 4 splits
                        const float4 y = *reinterpret_cast<const float4*>(
                            a.qkv + (size_t)bb * a.n_qkv + hd * D + c4 * 4 + s2 * stride);
                        x.x += y.x; x.y += y.y; x.z += y.z; x.w += y.w;
                    }
                    if (a.qfin && split == 0 && bb < a.B)
                        *reinterpret_cast<float4*>(a.qfin + (size_t)bb * (a.n_qkv / 3) + hd * D + c4 * 4) = x;
                    uint16_t hi[4], lo[4];
                    split_bf16(x.x, hi[0], lo[0]);
                    split_bf16(x.y, hi[1], lo[1]);
                    split_bf16(x.z, hi[2], lo[2]);
                    split_bf16(x.w, hi[3], lo[3]);
                    const uint32_t off = sw128_off(row, c4 >> 1) + (c4 & 1) * 8;
                    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(qh + off), "r"(pack2(hi[0], hi[1])),
                                 "r"(pack2(hi[2], hi[3])) : "memory");
                    asm volatile("st.shared.v2.b32 [%0], {%1,%2};" ::"r"(ql + off), "r"(pack2(lo[0], lo[1])),
                                 "r"(pack2(lo[2], lo[3])) : "memory");
                }
            }
            fence_async_smem();
            __syncwarp();
            if (lane == 0) mbar_arrive(qready);
        }
        constexpr float L2E = 1.4426950408889634f;
        float m = -INFINITY, l = 0.0f;
        float o[32];
#pragma unroll
        for (int i = 0; i < 32; ++i) o[i] = 0.0f;
        const uint32_t ph = smem_u32(sP) + half * (BT * 128), pl = ph + C::P_BYTES;
        float alpha_prev = 0.0f;
        for (int i = 0; i < nloc; ++i) {
            const int cbase = (c0 + i) * CH + half * 64;
            const int valid = min(64, a.S - cbase);  // may be <= 0 for the last chunk's upper half
            const float* ksc = nullptr;
            const float* vsc = nullptr;
            if constexpr (Q8) {
                mbar_wait(&xready[i & 1], (i >> 1) & 1);
                ksc = reinterpret_cast<const float*>(sX + (i & 1) * C::XBUF_BYTES + 2 * C::KV_BYTES) + half * 64;
                vsc = ksc + CH;
            }
            mbar_wait(&sfull[i & 1], (i >> 1) & 1);
            fence_after();
            const uint32_t tS = tmem + (i & 1) * CH;
            if (!warp_live) {  // no session in these 32 rows: their P rows and O rows are never used
                if (i > 0) mbar_wait(ofull, (i - 1) & 1);  // P is rewritten below
                __syncwarp();
                if (lane == 0) {
                    mbar_arrive(&sfree[i & 1]);
                    mbar_arrive(pready);
                }
                continue;
            }
            // pass 1: row max over this warp's 64 columns, exchanged with the partner warp
            float mx = -INFINITY;
            {
                float mq[8];  // 8 independent max chains (short dependency chains)
#pragma unroll
                for (int e = 0; e < 8; ++e) mq[e] = -INFINITY;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float sv[32];
                    tmem_ld32(tS + lane_off + half * 64 + c * 32, sv);
#pragma unroll
                    for (int e = 0; e < 32; ++e) {
                        float x = sv[e];
                        if constexpr (Q8) x *= ksc[c * 32 + e];  // scores of dequantised K = scale * (q . code)
                        if (valid >= 64 || c * 32 + e < valid) mq[e & 7] = fmaxf(mq[e & 7], x);
                    }
                }
                mx = fmaxf(fmaxf(fmaxf(mq[0], mq[1]), fmaxf(mq[2], mq[3])),
                           fmaxf(fmaxf(mq[4], mq[5]), fmaxf(mq[6], mq[7])));
            }
            float* xm = xch + (i & 1) * 2 * BT;
            xm[half * BT + r] = mx;
            asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
            mx = fmaxf(fmaxf(mx, xm[(half ^ 1) * BT + r]), m);
            const float alpha = (m == -INFINITY) ? 0.0f : exp2f((m - mx) * L2E);
            const float mxs = mx * L2E;
            // the previous chunk's O (deferred: its PV ran while this chunk's S was read);
            // P of this chunk may be written only once that PV has finished
            if (i > 0) {
                mbar_wait(ofull, (i - 1) & 1);
                fence_after();
                float v[32];
                tmem_ld32(tO + lane_off + half * 32, v);
#pragma unroll
                for (int e = 0; e < 32; ++e) o[e] = o[e] * alpha_prev + v[e];
                fence_before();
            }
            // pass 2: p = exp(s - max), P (times the V row scale for int8) as hi / lo bf16
            float rs = 0.0f;
            if (valid >= 64) {
                // full 64 columns: packed fp32x2 arithmetic, hi / lo split two at a time
                const f2x l2e2 = f2pack(L2E, L2E), nm2 = f2pack(-mxs, -mxs), neg2 = f2pack(-1.0f, -1.0f);
                f2x rs2 = 0ull;
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float sv[32];
                    tmem_ld32(tS + lane_off + half * 64 + c * 32, sv);
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        uint32_t hw[4], lw[4];
#pragma unroll
                        for (int e = 0; e < 8; e += 2) {
                            const int j = c * 32 + g * 8 + e;
                            f2x x2 = f2pack(sv[g * 8 + e], sv[g * 8 + e + 1]);
                            if constexpr (Q8) x2 = fmul2(x2, f2pack(ksc[j], ksc[j + 1]));
                            const f2x a2 = ffma2(x2, l2e2, nm2);
                            float p0, p1;
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p0) : "f"(f2lo(a2)));
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p1) : "f"(f2hi(a2)));
                            f2x p2 = f2pack(p0, p1);
                            rs2 = fadd2(rs2, p2);
                            if constexpr (Q8) p2 = fmul2(p2, f2pack(vsc[j], vsc[j + 1]));
                            uint32_t h;
                            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(h) : "f"(f2hi(p2)), "f"(f2lo(p2)));
                            const f2x r2 = ffma2(bf16x2_to_f2(h), neg2, p2);  // exact residual
                            uint32_t lo2;
                            asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(lo2) : "f"(f2hi(r2)), "f"(f2lo(r2)));
                            hw[e / 2] = h;
                            lw[e / 2] = lo2;
                        }
                        const uint32_t off = sw128_off(r, c * 4 + g);
                        st_shared_v4(ph + off, hw[0], hw[1], hw[2], hw[3]);
                        st_shared_v4(pl + off, lw[0], lw[1], lw[2], lw[3]);
                    }
                }
                rs = f2lo(rs2) + f2hi(rs2);
            } else {
#pragma unroll
                for (int c = 0; c < 2; ++c) {
                    float sv[32];
                    tmem_ld32(tS + lane_off + half * 64 + c * 32, sv);
#pragma unroll
                    for (int g = 0; g < 4; ++g) {
                        uint16_t hi[8], lo[8];
#pragma unroll
                        for (int e = 0; e < 8; ++e) {
                            const int j = c * 32 + g * 8 + e;
                            float x = sv[g * 8 + e];
                            if constexpr (Q8) x *= ksc[j];
                            float p;
                            asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(p) : "f"(fmaf(x, L2E, -mxs)));
                            p = (j < valid) ? p : 0.0f;
                            rs += p;
                            // O = sum p * (code * vscale): fold the V row scale into P
                            const float pv = Q8 ? p * vsc[j] : p;
                            split_bf16(pv, hi[e], lo[e]);
                        }
                        const int cc = c * 4 + g;  // 16-byte chunk of this warp's 64-row P panel
                        const uint32_t off = sw128_off(r, cc);
                        st_shared_v4(ph + off, pack2(hi[0], hi[1]), pack2(hi[2], hi[3]), pack2(hi[4], hi[5]),
                                     pack2(hi[6], hi[7]));
                        st_shared_v4(pl + off, pack2(lo[0], lo[1]), pack2(lo[2], lo[3]), pack2(lo[4], lo[5]),
                                     pack2(lo[6], lo[7]));
                    }
                }
            }
            m = mx;
            l = l * alpha + rs;
            alpha_prev = alpha;
            fence_async_smem();
            fence_before();
            __syncwarp();
            if (lane == 0) {
                mbar_arrive(&sfree[i & 1]);
                mbar_arrive(pready);
            }
        }
        if (nloc > 0 && warp_live) {  // the last chunk's O
            mbar_wait(ofull, (nloc - 1) & 1);
            fence_after();
            float v[32];
            tmem_ld32(tO + lane_off + half * 32, v);
#pragma unroll
            for (int e = 0; e < 32; ++e) o[e] = o[e] * alpha_prev + v[e];
            fence_before();
        }
        // row sum = both halves' partial sums (same running max in both warps)
        float* xl = xch + 4 * BT;
        xl[half * BT + r] = l;
        asm volatile("bar.sync %0, 64;" ::"r"(pair_bar) : "memory");
        if (live) {
            float* w = a.part + (((size_t)b * a.H + hd) * a.nsplit + split) * (D + 4);
            if (half == 0) *reinterpret_cast<float2*>(w) = make_float2(m, l + xl[BT + r]);
#pragma unroll
            for (int e = 0; e < 32; e += 4)
                *reinterpret_cast<float4*>(w + 4 + half * 32 + e) = make_float4(o[e], o[e + 1], o[e + 2], o[e + 3]);
        }
    }
    pdl_trigger();
    fence_before();
    __syncthreads();
    fence_after();
    if (warp == 2) tmem_dealloc(tmem, 512);
}
}  // namespace k10

// ============================================================================
// K11: user segment + append + Eq. 5 merge, one warp per (session, head).
// ============================================================================
template <int D, int NV>  // NV: split-K partials of the QKV projection held in flight
__global__ void __launch_bounds__(128, NV == 1 ? 4 : 3) batch_user_merge_kernel(BatchUserMerge a) {
    constexpr int G = D / 8;         // lanes per row (8 dims = 16 bytes per lane)
    constexpr int RPI = 32 / G;      // rows per warp-wide load
    constexpr int NT = 32 / RPI;     // rows per lane per 32-row block
    constexpr int NP = 4;            // context partials whose loads are issued up front
    const int lane = threadIdx.x & 31;
    const int item = blockIdx.x * 4 + (threadIdx.x >> 5);
    pdl_wait();
    pdl_trigger();
    if (item >= a.B * a.H) return;
    const int b = item / a.H, hd = item - b * a.H;
    const int grp = lane / G, c = lane - grp * G;  // row group, 8-dim chunk
    const int h = a.H * D;
    const int owner = a.prefill ? 0 : b;  // the session whose user cache this row uses
    const size_t head_off = (((size_t)owner * a.L + a.layer) * a.H + hd) * (size_t)a.cap * D;
    uint16_t* uk = a.uk + head_off;
    uint16_t* uv = a.uv + head_off;
    // ---- every independent load issued before the first use: the user-row count,
    //      this step's q/k/v partials, the first 32 user rows, the context partials ----
    const int ulen = a.state->user_len + (a.prefill ? a.row0 + b : 0);  // this row's cache row
    const size_t stride = (size_t)a.B * a.n_qkv;
    const float* p0 = a.qkv + (size_t)b * a.n_qkv + hd * D + c * 8;
    float4 v[NV][3][2];
    const int ksl = a.qfin ? 0 : a.KS;  // partials to load (none when K10 finalised q/k/v)
#pragma unroll
    for (int s = 0; s < NV; ++s)
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            if (s < ksl) {
                v[s][t][0] = *reinterpret_cast<const float4*>(p0 + s * stride + t * h);
                v[s][t][1] = *reinterpret_cast<const float4*>(p0 + s * stride + t * h + 4);
            } else {
                v[s][t][0] = make_float4(0.f, 0.f, 0.f, 0.f);
                v[s][t][1] = make_float4(0.f, 0.f, 0.f, 0.f);
            }
        }
    uint4 kr[NT], vr[NT];
#pragma unroll
    for (int t = 0; t < NT; ++t) {  // rows < cap are allocated; rows >= ulen are masked below
        const int j = grp + RPI * t;
        if (j < a.cap) {
            kr[t] = *reinterpret_cast<const uint4*>(uk + (size_t)j * D + c * 8);
            vr[t] = *reinterpret_cast<const uint4*>(uv + (size_t)j * D + c * 8);
        } else {
            kr[t] = make_uint4(0, 0, 0, 0);
            vr[t] = make_uint4(0, 0, 0, 0);
        }
    }
    const float* wpart = a.part + ((size_t)b * a.H + hd) * a.nsplit * (D + 4);
    float2 pml[NP];
#pragma unroll
    for (int s = 0; s < NP; ++s)
        if (s < a.nsplit) pml[s] = *reinterpret_cast<const float2*>(wpart + s * (D + 4));
    // ---- q, k, v (k, v rounded to bf16 as stored) ----
    float q[8], kc[8], vc[8];
    if (a.qfin) {  // finalised by the context kernel: q from qfin, k / v already in the cache
        const float4 q0 = *reinterpret_cast<const float4*>(a.qfin + (size_t)b * h + hd * D + c * 8);
        const float4 q1 = *reinterpret_cast<const float4*>(a.qfin + (size_t)b * h + hd * D + c * 8 + 4);
        q[0] = q0.x; q[1] = q0.y; q[2] = q0.z; q[3] = q0.w; q[4] = q1.x; q[5] = q1.y; q[6] = q1.z; q[7] = q1.w;
        const uint4 kw = *reinterpret_cast<const uint4*>(uk + (size_t)ulen * D + c * 8);
        const uint4 vw = *reinterpret_cast<const uint4*>(uv + (size_t)ulen * D + c * 8);
        const uint32_t kk[4] = {kw.x, kw.y, kw.z, kw.w}, vv[4] = {vw.x, vw.y, vw.z, vw.w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            kc[2 * k] = bf16_lo(kk[k]); kc[2 * k + 1] = bf16_hi(kk[k]);
            vc[2 * k] = bf16_lo(vv[k]); vc[2 * k + 1] = bf16_hi(vv[k]);
        }
    } else {
        for (int s = NV; s < a.KS; ++s)
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                const float4 y0 = *reinterpret_cast<const float4*>(p0 + s * stride + t * h);
                const float4 y1 = *reinterpret_cast<const float4*>(p0 + s * stride + t * h + 4);
                v[0][t][0].x += y0.x; v[0][t][0].y += y0.y; v[0][t][0].z += y0.z; v[0][t][0].w += y0.w;
                v[0][t][1].x += y1.x; v[0][t][1].y += y1.y; v[0][t][1].z += y1.z; v[0][t][1].w += y1.w;
            }
        float xs[3][8];
#pragma unroll
        for (int t = 0; t < 3; ++t) {
            xs[t][0] = v[0][t][0].x; xs[t][1] = v[0][t][0].y; xs[t][2] = v[0][t][0].z; xs[t][3] = v[0][t][0].w;
            xs[t][4] = v[0][t][1].x; xs[t][5] = v[0][t][1].y; xs[t][6] = v[0][t][1].z; xs[t][7] = v[0][t][1].w;
        }
#pragma unroll
        for (int s = 1; s < NV; ++s)
#pragma unroll
            for (int t = 0; t < 3; ++t) {
                xs[t][0] += v[s][t][0].x; xs[t][1] += v[s][t][0].y; xs[t][2] += v[s][t][0].z;
                xs[t][3] += v[s][t][0].w; xs[t][4] += v[s][t][1].x; xs[t][5] += v[s][t][1].y;
                xs[t][6] += v[s][t][1].z; xs[t][7] += v[s][t][1].w;
            }
#pragma unroll
        for (int e = 0; e < 8; ++e) {
            q[e] = xs[0][e];
            kc[e] = __bfloat162float(__float2bfloat16_rn(xs[1][e]));
            vc[e] = __bfloat162float(__float2bfloat16_rn(xs[2][e]));
        }
    }
    // append (cache_merge.cpp:189-199): row ulen of this session's user cache
    if (grp == 0 && !a.qfin) {
        uint4 kw, vw;
        kw.x = f32_to_bf16_bits(kc[0]) | ((uint32_t)f32_to_bf16_bits(kc[1]) << 16);
        kw.y = f32_to_bf16_bits(kc[2]) | ((uint32_t)f32_to_bf16_bits(kc[3]) << 16);
        kw.z = f32_to_bf16_bits(kc[4]) | ((uint32_t)f32_to_bf16_bits(kc[5]) << 16);
        kw.w = f32_to_bf16_bits(kc[6]) | ((uint32_t)f32_to_bf16_bits(kc[7]) << 16);
        vw.x = f32_to_bf16_bits(vc[0]) | ((uint32_t)f32_to_bf16_bits(vc[1]) << 16);
        vw.y = f32_to_bf16_bits(vc[2]) | ((uint32_t)f32_to_bf16_bits(vc[3]) << 16);
        vw.z = f32_to_bf16_bits(vc[4]) | ((uint32_t)f32_to_bf16_bits(vc[5]) << 16);
        vw.w = f32_to_bf16_bits(vc[6]) | ((uint32_t)f32_to_bf16_bits(vc[7]) << 16);
        *reinterpret_cast<uint4*>(uk + (size_t)ulen * D + c * 8) = kw;
        *reinterpret_cast<uint4*>(uv + (size_t)ulen * D + c * 8) = vw;
    }
    // user segment over rows [0, ulen) in blocks of 32 rows (NT rows per lane), then the current row
    float m = -INFINITY, l = 0.0f, o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = 0.0f;
    for (int j0 = 0; j0 < ulen; j0 += 32) {
        if (j0 > 0) {
#pragma unroll
            for (int t = 0; t < NT; ++t) {
                const int j = j0 + grp + RPI * t;
                if (j < ulen) {
                    kr[t] = *reinterpret_cast<const uint4*>(uk + (size_t)j * D + c * 8);
                    vr[t] = *reinterpret_cast<const uint4*>(uv + (size_t)j * D + c * 8);
                }
            }
        }
        float sc[NT];
        float bm = -INFINITY;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const uint32_t w[4] = {kr[t].x, kr[t].y, kr[t].z, kr[t].w};
            float acc = 0.0f;
#pragma unroll
            for (int k = 0; k < 4; ++k) acc += q[2 * k] * bf16_lo(w[k]) + q[2 * k + 1] * bf16_hi(w[k]);
#pragma unroll
            for (int off = G / 2; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
            const int j = j0 + grp + RPI * t;
            sc[t] = j < ulen ? acc : -INFINITY;
            bm = fmaxf(bm, sc[t]);
        }
        const float mx = fmaxf(m, warp_max(bm));
        const float alpha = (m == -INFINITY) ? 0.0f : __expf(m - mx);
        float ps = 0.0f;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] *= alpha;
#pragma unroll
        for (int t = 0; t < NT; ++t) {
            const float p = sc[t] == -INFINITY ? 0.0f : __expf(sc[t] - mx);
            ps += p;
            const uint32_t w[4] = {vr[t].x, vr[t].y, vr[t].z, vr[t].w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                o[2 * k] += p * bf16_lo(w[k]);
                o[2 * k + 1] += p * bf16_hi(w[k]);
            }
        }
        // block row sum: one copy per row group (lanes of a group hold identical p)
#pragma unroll
        for (int off = G; off < 32; off <<= 1) ps += __shfl_xor_sync(0xffffffffu, ps, off);
        l = l * alpha + ps;
        m = mx;
    }
    // fold the row groups' partial outputs (same running max in every lane)
#pragma unroll
    for (int off = G; off < 32; off <<= 1)
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] += __shfl_xor_sync(0xffffffffu, o[e], off);
    {   // the current row (attends to itself, causal)
        float acc = 0.0f;
#pragma unroll
        for (int e = 0; e < 8; ++e) acc += q[e] * kc[e];
#pragma unroll
        for (int off = G / 2; off >= 1; off >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, off);
        const float mx = fmaxf(m, acc);
        const float alpha = (m == -INFINITY) ? 0.0f : __expf(m - mx);
        const float p = __expf(acc - mx);
        l = l * alpha + p;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = o[e] * alpha + p * vc[e];
        m = mx;
    }
    // Eq. 5 generalised: log-sum-exp merge of the user partial with the context partials
    if (a.nsplit > 0) {
        float M = m;
#pragma unroll
        for (int s = 0; s < NP; ++s)
            if (s < a.nsplit) M = fmaxf(M, pml[s].x);
        for (int s = NP; s < a.nsplit; ++s) M = fmaxf(M, wpart[s * (D + 4)]);
        const float fu = __expf(m - M);
        float Lt = l * fu, ot[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) ot[e] = o[e] * fu;
        float4 po[NP][2];
#pragma unroll
        for (int s = 0; s < NP; ++s)
            if (s < a.nsplit) {
                po[s][0] = *reinterpret_cast<const float4*>(wpart + s * (D + 4) + 4 + c * 8);
                po[s][1] = *reinterpret_cast<const float4*>(wpart + s * (D + 4) + 8 + c * 8);
            }
#pragma unroll
        for (int s = 0; s < NP; ++s)
            if (s < a.nsplit) {
                const float f = pml[s].x == -INFINITY ? 0.0f : __expf(pml[s].x - M);
                Lt += pml[s].y * f;
                ot[0] += po[s][0].x * f; ot[1] += po[s][0].y * f; ot[2] += po[s][0].z * f;
                ot[3] += po[s][0].w * f; ot[4] += po[s][1].x * f; ot[5] += po[s][1].y * f;
                ot[6] += po[s][1].z * f; ot[7] += po[s][1].w * f;
            }
        for (int s = NP; s < a.nsplit; ++s) {
            const float* ws = wpart + s * (D + 4);
            const float2 ml = *reinterpret_cast<const float2*>(ws);
            const float4 o0 = *reinterpret_cast<const float4*>(ws + 4 + c * 8);
            const float4 o1 = *reinterpret_cast<const float4*>(ws + 8 + c * 8);
            const float f = ml.x == -INFINITY ? 0.0f : __expf(ml.x - M);
            Lt += ml.y * f;
            ot[0] += o0.x * f; ot[1] += o0.y * f; ot[2] += o0.z * f; ot[3] += o0.w * f;
            ot[4] += o1.x * f; ot[5] += o1.y * f; ot[6] += o1.z * f; ot[7] += o1.w * f;
        }
        l = Lt;
#pragma unroll
        for (int e = 0; e < 8; ++e) o[e] = ot[e];
    }
    if (grp == 0) {
        const float inv = 1.0f / l;
        uint16_t hi[8], lo[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) split_bf16(o[e] * inv, hi[e], lo[e]);
        const size_t k = (size_t)b * h + hd * D + c * 8;
        *reinterpret_cast<uint4*>(a.xhl + k) =
            make_uint4(hi[0] | ((uint32_t)hi[1] << 16), hi[2] | ((uint32_t)hi[3] << 16),
                       hi[4] | ((uint32_t)hi[5] << 16), hi[6] | ((uint32_t)hi[7] << 16));
        *reinterpret_cast<uint4*>(a.xhl + (size_t)a.B * h + k) =
            make_uint4(lo[0] | ((uint32_t)lo[1] << 16), lo[2] | ((uint32_t)lo[3] << 16),
                       lo[4] | ((uint32_t)lo[5] << 16), lo[6] | ((uint32_t)lo[7] << 16));
    }
}

// ============================================================================
// host launchers
// ============================================================================
CUtensorMap make_map_2d(const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t inner,
                        uint64_t rows, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw);
CUtensorMap make_map_3d_bf16(const void* base, uint64_t inner, uint64_t rows, uint64_t depth,
                             uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw);

int batch_proj_bn(int B) {
    int bn = ((B + 31) / 32) * 32;
    return bn > 256 ? 256 : bn;
}

int batch_proj_splits(int N_out, int K, int B, int num_sms) {
    const int tiles = (N_out / k9::BM) * ((B + batch_proj_bn(B) - 1) / batch_proj_bn(B));
    int ks = num_sms / tiles;  // floor: a second partial wave costs more than fewer splits
    const int kblocks = K / k9::BK;
    if (ks < 1) ks = 1;
    if (ks > kblocks) ks = kblocks;
    if (ks > kMaxSplitK) ks = kMaxSplitK;
    return ks;
}

template <class... KArgs, class... Args>
static void launch_pdl(void (*fn)(KArgs...), dim3 grid, dim3 block, size_t smem, cudaStream_t st,
                       Args... args) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid;
    cfg.blockDim = block;
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    EKV_CUDA(cudaLaunchKernelEx(&cfg, fn, args...));
}

void launch_batch_proj(const CUtensorMap& map_w, int w_row0, int N_out, int K, const CUtensorMap& map_x,
                       int B, int KS, float* out, cudaStream_t st) {
    using namespace k9;
    require(N_out % BM == 0 && K % BK == 0, "batch projection: h must be a multiple of 128",
            EKV_EUNSUPPORTED);
    const int BN = batch_proj_bn(B);
    const int stage_bytes = A_BYTES + 2 * BN * BK * 2;
    int stages = (200 * 1024) / stage_bytes;
    if (stages > 6) stages = 6;
    const int smem = stages * stage_bytes + 1024 + 256;
    ensure_smem_attr((const void*)batch_proj_kernel, 227 * 1024);
    dim3 grid(N_out / BM, (B + BN - 1) / BN, KS);
    launch_pdl(batch_proj_kernel, grid, dim3(THREADS), smem, st, map_w, map_x, w_row0, N_out, K, B, BN, KS,
               stages, idesc_bf16(BM, BN), out);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

void launch_batch_xprep(const BatchXprep& a, cudaStream_t st) {
    dim3 grid((a.h / 4 + 127) / 128, a.B);
    launch_pdl(batch_xprep_kernel, grid, dim3(128), 0, st, a);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

int batch_ctx_splits(int S, int H, int B, int num_sms) {
    if (S <= 0) return 0;
    const int nchunks = (S + k10::CH - 1) / k10::CH;
    const int nbt = (B + k10::BT - 1) / k10::BT;
    int ns = num_sms / (H * nbt);  // one wave: CTAs <= SMs (one CTA per SM)
    if (ns > nchunks) ns = nchunks;
    if (ns < 1) ns = 1;
    return ns;
}

bool batch_ctx_supported(int D, int fmt, int group) {
    return D == 64 && (fmt == EKV_KV_BF16 || (fmt == EKV_KV_INT8 && group == D));
}

template <int FMT>
static void launch_ctx(const BatchCtxMaps& mp, const BatchCtxAttn& a, cudaStream_t st) {
    using namespace k10;
    using Cf = Cfg<64, FMT>;
    ensure_smem_attr((const void*)batch_ctx_attn_kernel<64, FMT>, Cf::SMEM);
    dim3 grid(a.H, a.nsplit, (a.B + BT - 1) / BT);
    launch_pdl(batch_ctx_attn_kernel<64, FMT>, grid, dim3(THREADS), Cf::SMEM, st, mp.k, mp.v, mp.ks, mp.vs, a);
}

void launch_batch_ctx_attn(const BatchCtxMaps& mp, const BatchCtxAttn& a, cudaStream_t st) {
    require(a.D == 64, "batched context attention supports head_dim 64", EKV_EUNSUPPORTED);
    if (mp.fmt == EKV_KV_BF16)
        launch_ctx<16>(mp, a, st);
    else
        launch_ctx<8>(mp, a, st);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

// ============================================================================
// Prefill finish: split-K sum of K9's partials + the consumer's layout
// ============================================================================
__global__ void prefill_finish_kernel(PrefillFinish a) {
    pdl_wait();
    pdl_trigger();
    const int r = blockIdx.y;
    const int n = 4 * (blockIdx.x * blockDim.x + threadIdx.x);
    if (n >= a.N) return;
    const float4 x = sum_splits4(a.part + (size_t)r * a.N + n, (size_t)a.R * a.N, a.KS);
    const int base = a.state->user_len + a.row0;
    if (a.mode == 0) {
        const int h = a.N / 3;
        if (n < h) {
            *reinterpret_cast<float4*>(a.q_out + (size_t)r * h + n) = x;
        } else {
            const int nn = n < 2 * h ? n - h : n - 2 * h;
            const int head = nn / a.d, c = nn - head * a.d;
            uint16_t* dst = (n < 2 * h ? a.uk : a.uv) + ((size_t)head * a.cap + base + r) * a.d + c;
            *reinterpret_cast<uint2*>(dst) =
                make_uint2(f32_to_bf16_bits(x.x) | ((uint32_t)f32_to_bf16_bits(x.y) << 16),
                           f32_to_bf16_bits(x.z) | ((uint32_t)f32_to_bf16_bits(x.w) << 16));
        }
    } else {
        *reinterpret_cast<float4*>(a.y + (size_t)r * a.N + n) = x;
        if (a.y_hist) *reinterpret_cast<float4*>(a.y_hist + (size_t)(base + r) * a.N + n) = x;
    }
}

void launch_prefill_finish(const PrefillFinish& a, cudaStream_t st) {
    dim3 grid((a.N / 4 + 127) / 128, a.R);
    launch_pdl(prefill_finish_kernel, grid, dim3(128), 0, st, a);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

void launch_batch_user_merge(const BatchUserMerge& a, cudaStream_t st) {
    const int items = a.B * a.H;
    const int grid = (items + 3) / 4;
    switch (a.D) {
        case 32:
            if (a.KS == 1 || a.qfin) launch_pdl(batch_user_merge_kernel<32, 1>, dim3(grid), dim3(128), 0, st, a);
            else launch_pdl(batch_user_merge_kernel<32, 3>, dim3(grid), dim3(128), 0, st, a);
            break;
        case 64:
            if (a.KS == 1 || a.qfin) launch_pdl(batch_user_merge_kernel<64, 1>, dim3(grid), dim3(128), 0, st, a);
            else launch_pdl(batch_user_merge_kernel<64, 3>, dim3(grid), dim3(128), 0, st, a);
            break;
        case 128:
            if (a.KS == 1 || a.qfin) launch_pdl(batch_user_merge_kernel<128, 1>, dim3(grid), dim3(128), 0, st, a);
            else launch_pdl(batch_user_merge_kernel<128, 3>, dim3(grid), dim3(128), 0, st, a);
            break;
        default: require(false, "batched decode: head_dim must be 32, 64 or 128", EKV_EUNSUPPORTED);
    }
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

}  // namespace ekv
