// K1: the alignment projection Q = X * W_Q of every matched cloud layer, on
// the 5th-generation tensor cores, reduced in the epilogue to per-column sums
// of squares (the Q half of the channel score of select_channels,
// head_prune.cpp:92-97).  Q itself is never written to memory.
//
// Replaces project_qkv (transformer.cpp:133-152) as used by build_deep_kv
// (sim.cpp:240-253), which recomputes Q for each distinct matched cloud layer
// lc from that layer's input hidden state X_lc.
//
// Structure (one CTA per SM, persistent over (layer, m-block, n-block) tiles):
//   warp 0      TMA producer: X tile 128x64 and W tile 256x64 (bf16, 128-byte
//               swizzle) per k-step into a 4-stage shared-memory ring
//   warp 1      MMA issuer: one elected thread issues tcgen05.mma
//               (kind::f16, M=128, N=256, K=16, fp32 accumulate in TMEM)
//   warp 2      TMEM allocator (512 columns = two 256-column accumulators)
//   warps 4..7  epilogue: tcgen05.ld 32 columns at a time, square, reduce the
//               128 rows with a 31-shuffle butterfly reduce-scatter, combine
//               the 4 warps in shared memory, one fp64 atomic per column.
// The two TMEM accumulators let the epilogue of tile i overlap the MMAs of
// tile i+1.  Every mbarrier wait is bounded (trap after ~2 s) so a pipeline
// bug fails the launch instead of hanging the device.
#include <cuda.h>

#include <algorithm>

#include "ekv_common.cuh"
#include "ekv_kernels.h"

namespace ekv {

namespace k1 {

constexpr int BM = 128, BN = 256, BK = 64, STAGES = 4;
constexpr int A_BYTES = BM * BK * 2;  // 16 KB
constexpr int B_BYTES = BN * BK * 2;  // 32 KB
constexpr int STAGE_BYTES = A_BYTES + B_BYTES;
constexpr int TMEM_COLS = 512;
constexpr int THREADS = 256;
constexpr int SMEM_BYTES = STAGES * STAGE_BYTES + 4 * BN * 4 /*red*/ + 256 /*barriers*/ + 1024;

// instruction descriptor: D fp32 (bits 4-5 = 1), A bf16 (7-9 = 1), B bf16
// (10-12 = 1), both K-major, N>>3 at 17-22, M>>4 at 24-28.
constexpr uint32_t IDESC = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(BN >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);

__device__ __forceinline__ uint32_t smem_u32(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
                 "r"(bytes)
                 : "memory");
}

__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
    const uint32_t addr = smem_u32(bar);
    uint32_t done = 0;
    const long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(addr), "r"(parity)
            : "memory");
        if (done) return;
        if (clock64() - t0 > 4000000000ll) __trap();  // pipeline bug: fail, do not hang
    }
}

__device__ __forceinline__ void tma_load_3d(const CUtensorMap* map, uint64_t* bar, void* dst, int c0,
                                            int c1, int c2) {
    asm volatile(
        "cp.async.bulk.tensor.3d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
        "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2)
        : "memory");
}

// UMMA shared-memory descriptor, K-major, 128-byte swizzle: LBO = 16 B
// (field 1), SBO = 1024 B between 8-row groups (field 64), version 1,
// layout type 2 (SWIZZLE_128B).  Stage buffers are 1024-byte aligned.
__device__ __forceinline__ uint64_t umma_desc_sw128(uint32_t saddr) {
    uint64_t d = 0;
    d |= (uint64_t)((saddr >> 4) & 0x3FFF);
    d |= (uint64_t)1 << 16;
    d |= (uint64_t)64 << 32;
    d |= (uint64_t)1 << 46;
    d |= (uint64_t)2 << 61;
    return d;
}

__device__ __forceinline__ void umma_bf16(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t accumulate) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
        "l"(adesc), "l"(bdesc), "r"(IDESC), "r"(accumulate));
}

__device__ __forceinline__ void umma_commit(uint64_t* bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                     smem_u32(bar))
                 : "memory");
}

__device__ __forceinline__ void tc_fence_before() {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}

__device__ __forceinline__ void tmem_ld32(uint32_t taddr, float* v) {
    uint32_t r[32];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
        "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
        "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]),
          "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]),
          "=r"(r[14]), "=r"(r[15]), "=r"(r[16]), "=r"(r[17]), "=r"(r[18]), "=r"(r[19]),
          "=r"(r[20]), "=r"(r[21]), "=r"(r[22]), "=r"(r[23]), "=r"(r[24]), "=r"(r[25]),
          "=r"(r[26]), "=r"(r[27]), "=r"(r[28]), "=r"(r[29]), "=r"(r[30]), "=r"(r[31])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
    for (int i = 0; i < 32; ++i) v[i] = __uint_as_float(r[i]);
}

// Sum over the 32 lanes of each of the 32 values; lane j returns column j.
__device__ __forceinline__ float butterfly_colsum(float* v, int lane) {
#pragma unroll
    for (int off = 16, n = 32; off >= 1; off >>= 1, n >>= 1) {
        const bool upper = lane & off;
#pragma unroll
        for (int i = 0; i < n / 2; ++i) {
            const float send = upper ? v[i] : v[i + n / 2];
            const float keep = upper ? v[i + n / 2] : v[i];
            v[i] = keep + __shfl_xor_sync(0xffffffffu, send, off);
        }
    }
    return v[0];
}

// Fused K2 (warps 2-3, otherwise idle): per-column sums of squares of the cached
// cloud K rows (d_c bf16 each) of every matched layer, the K half of the channel
// score (head_prune.cpp:92-97).  Each CTA streams a contiguous slice of the rows
// with 16-byte loads (8 in flight per thread) while the tensor pipe runs K1, so
// the K read (m*H*S*d_c*2 B) hides under the GEMM.  fp32 partials over <= 32 rows
// per thread are folded into fp64.
__device__ __forceinline__ void fused_kcolsq(const AlignArgs& a, int t) {
    const int lpr = a.d_c / 8;  // lanes per row
    const int rpi = 64 / lpr;   // rows per pass of the 64 threads
    const int cseg = t % lpr;
    const int64_t T = (int64_t)a.k_layers * a.k_rows;
    const int64_t r1 = T * (blockIdx.x + 1) / gridDim.x;
    int64_t r = T * blockIdx.x / gridDim.x + t / lpr;
    int layer = (int)(r / a.k_rows);
    int64_t row = r - (int64_t)layer * a.k_rows;
    double acc64[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    constexpr int U = 8;
    while (r < r1) {
        uint4 v[U];
        int n = 0;
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (r < r1) {
                v[u] = ld_stream(a.k[layer] + row * a.d_c + cseg * 8);
                ++n;
                r += rpi;
                row += rpi;
                while (row >= a.k_rows && layer + 1 < a.k_layers) {
                    row -= a.k_rows;
                    ++layer;
                }
            }
        }
        float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
#pragma unroll
        for (int u = 0; u < U; ++u) {
            if (u < n) {
                const uint32_t w[4] = {v[u].x, v[u].y, v[u].z, v[u].w};
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    const float lo = bf16_lo(w[k]), hi = bf16_hi(w[k]);
                    acc[2 * k] = fmaf(lo, lo, acc[2 * k]);
                    acc[2 * k + 1] = fmaf(hi, hi, acc[2 * k + 1]);
                }
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) acc64[k] += (double)acc[k];
    }
    const int lane = t & 31;
    for (int o = lpr; o < 32; o <<= 1)
#pragma unroll
        for (int k = 0; k < 8; ++k) acc64[k] += __shfl_xor_sync(0xffffffffu, acc64[k], o);
    if (lane < lpr)
#pragma unroll
        for (int k = 0; k < 8; ++k) atomicAdd(&a.kcolsq[cseg * 8 + k], acc64[k]);
}

__global__ void __launch_bounds__(THREADS, 1)
    align_qnorm_kernel(const __grid_constant__ CUtensorMap map_x,
                       const __grid_constant__ CUtensorMap map_w, const __grid_constant__ AlignArgs a) {
    const int m_layers = a.m_layers, S = a.S, h_c = a.h_c, n_cols = a.n_cols;
    double* __restrict__ colsq = a.colsq;
    extern __shared__ uint8_t smem_raw[];
    uint8_t* smem = (uint8_t*)(((uintptr_t)smem_raw + 1023) & ~(uintptr_t)1023);
    uint8_t* sA = smem;
    uint8_t* sB = smem + STAGES * A_BYTES;
    float* red = (float*)(smem + STAGES * STAGE_BYTES);  // [4][BN]
    uint64_t* bars = (uint64_t*)(red + 4 * BN);
    uint64_t* full = bars;               // [STAGES]
    uint64_t* empty = bars + STAGES;     // [STAGES]
    uint64_t* tfull = bars + 2 * STAGES; // [2]
    uint64_t* tempty = tfull + 2;        // [2]
    uint32_t* tmem_slot = (uint32_t*)(tempty + 2);

    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int mblocks = S / BM, nblocks = n_cols / BN, kblocks = h_c / BK;
    const int tiles_per_layer = mblocks * nblocks;
    const int total = m_layers * tiles_per_layer;

    if (warp == 0 && lane == 0) {
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_x) : "memory");
        asm volatile("prefetch.tensormap [%0];" ::"l"(&map_w) : "memory");
        for (int i = 0; i < STAGES; ++i) {
            mbar_init(&full[i], 1);
            mbar_init(&empty[i], 1);
        }
        for (int i = 0; i < 2; ++i) {
            mbar_init(&tfull[i], 1);
            mbar_init(&tempty[i], 4);  // one arrive per epilogue warp
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    }
    if (warp == 2) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                         smem_u32(tmem_slot)),
                     "r"(TMEM_COLS)
                     : "memory");
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    const uint32_t tmem_base = *tmem_slot;

    if (warp == 0) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x) {
                const int layer = t / tiles_per_layer;
                const int rem = t - layer * tiles_per_layer;
                const int mb = rem / nblocks, nb = rem - (rem / nblocks) * nblocks;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&empty[stage], phase ^ 1);
                    mbar_expect_tx(&full[stage], STAGE_BYTES);
                    tma_load_3d(&map_x, &full[stage], sA + stage * A_BYTES, kb * BK, mb * BM,
                                a.x_index[layer]);
                    tma_load_3d(&map_w, &full[stage], sB + stage * B_BYTES, kb * BK, nb * BN,
                                a.w_index[layer]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
            }
        }
    } else if (warp == 1) {
        if (lane == 0) {
            int stage = 0;
            uint32_t phase = 0;
            int local = 0;
            for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
                const int acc = local & 1;
                mbar_wait(&tempty[acc], ((local >> 1) & 1) ^ 1);
                tc_fence_after();
                const uint32_t dtmem = tmem_base + acc * BN;
                for (int kb = 0; kb < kblocks; ++kb) {
                    mbar_wait(&full[stage], phase);
                    tc_fence_after();
                    const uint32_t a0 = smem_u32(sA + stage * A_BYTES);
                    const uint32_t b0 = smem_u32(sB + stage * B_BYTES);
#pragma unroll
                    for (int k = 0; k < BK / 16; ++k) {
                        umma_bf16(dtmem, umma_desc_sw128(a0 + k * 32), umma_desc_sw128(b0 + k * 32),
                                  (kb | k) != 0);
                    }
                    umma_commit(&empty[stage]);
                    if (++stage == STAGES) {
                        stage = 0;
                        phase ^= 1;
                    }
                }
                umma_commit(&tfull[acc]);
            }
        }
    } else if (warp >= 4) {
        const int quad = warp - 4;  // TMEM lanes quad*32 .. quad*32+31
        int local = 0;
        for (int t = blockIdx.x; t < total; t += gridDim.x, ++local) {
            const int layer = t / tiles_per_layer;
            const int rem = t - layer * tiles_per_layer;
            const int nb = rem - (rem / nblocks) * nblocks;
            const int acc = local & 1;
            mbar_wait(&tfull[acc], (local >> 1) & 1);
            tc_fence_after();
            const uint32_t taddr = tmem_base + acc * BN + ((uint32_t)(quad * 32) << 16);
#pragma unroll 1
            for (int c = 0; c < BN / 32; ++c) {
                float v[32];
                tmem_ld32(taddr + c * 32, v);
#pragma unroll
                for (int i = 0; i < 32; ++i) v[i] = v[i] * v[i];
                red[quad * BN + c * 32 + lane] = butterfly_colsum(v, lane);
            }
            tc_fence_before();
            __syncwarp();
            if (lane == 0) mbar_arrive(&tempty[acc]);
            asm volatile("bar.sync 1, 128;" ::: "memory");
            const int et = threadIdx.x - 128;
            if (a.fold == 0) {
                for (int col = et; col < BN; col += 128) {
                    const float s = red[col] + red[BN + col] + red[2 * BN + col] + red[3 * BN + col];
                    atomicAdd(&colsq[(size_t)layer * n_cols + nb * BN + col], (double)s);
                }
            } else {
                // fold heads (and, across tiles, layers) into [d_c]: the reference scores
                // one mask over every stacked (layer, head) row (sim.cpp:236-256)
                for (int col = et; col < BN; col += 128)
                    red[col] = red[col] + red[BN + col] + red[2 * BN + col] + red[3 * BN + col];
                asm volatile("bar.sync 1, 128;" ::: "memory");
                for (int c = et; c < a.fold; c += 128) {
                    double s = 0.0;
                    for (int j = c; j < BN; j += a.fold) s += (double)red[j];
                    atomicAdd(&colsq[c], s);
                }
            }
            asm volatile("bar.sync 1, 128;" ::: "memory");
        }
    } else if (a.kcolsq != nullptr) {  // warps 2-3
        fused_kcolsq(a, threadIdx.x - 64);
    }
    tc_fence_before();
    __syncthreads();
    tc_fence_after();
    if (warp == 2) {
        asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                     "r"(TMEM_COLS)
                     : "memory");
    }
}

}  // namespace k1

// ---------------------------------------------------------------------------
// Host side: TMA descriptors through the driver entry point (no -lcuda).
// ---------------------------------------------------------------------------
typedef CUresult (*PFN_encodeTiled)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                                    const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                                    const cuuint32_t*, CUtensorMapInterleave, CUtensorMapSwizzle,
                                    CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

static PFN_encodeTiled get_encode() {
    static PFN_encodeTiled fn = nullptr;
    if (!fn) {
        void* p = nullptr;
        cudaDriverEntryPointQueryResult q;
        EKV_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
        require(p != nullptr && q == cudaDriverEntryPointSuccess,
                "cuTensorMapEncodeTiled unavailable", EKV_ECUDA);
        fn = (PFN_encodeTiled)p;
    }
    return fn;
}

CUtensorMap make_map_2d(const void* base, CUtensorMapDataType dt, int elem_bytes, uint64_t inner,
                        uint64_t rows, uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {inner * (uint64_t)elem_bytes};
    cuuint32_t box[2] = {box_inner, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, dt, 2, const_cast<void*>(base), dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, sw, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    require(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (2-D) failed (" + std::to_string((int)r) + ")",
            EKV_ECUDA);
    return m;
}

CUtensorMap make_map_1d(const void* base, CUtensorMapDataType dt, uint64_t n, uint32_t box) {
    CUtensorMap m;
    cuuint64_t dims[1] = {n};
    cuuint64_t strides[1] = {0};
    cuuint32_t bx[1] = {box};
    cuuint32_t estr[1] = {1};
    CUresult r = get_encode()(&m, dt, 1, const_cast<void*>(base), dims, strides, bx, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    require(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (1-D) failed (" + std::to_string((int)r) + ")",
            EKV_ECUDA);
    return m;
}

CUtensorMap make_map_3d_bf16(const void* base, uint64_t inner, uint64_t rows, uint64_t depth,
                             uint32_t box_inner, uint32_t box_rows, CUtensorMapSwizzle sw) {
    CUtensorMap m;
    cuuint64_t dims[3] = {inner, rows, depth};
    cuuint64_t strides[2] = {inner * 2, inner * rows * 2};
    cuuint32_t box[3] = {box_inner, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    require(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (3-D) failed (" + std::to_string((int)r) + ")",
            EKV_ECUDA);
    return m;
}

// 2-D bf16 map without swizzle (row-major [rows][inner]); used by the decode
// kernel to gather head column blocks of the output projection.
CUtensorMap make_map_2d_bf16(const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                             uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[2] = {inner, rows};
    cuuint64_t strides[1] = {inner * 2};
    cuuint32_t box[2] = {box_inner, box_rows};
    cuuint32_t estr[2] = {1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(base), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    require(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled (2-D) failed (" + std::to_string((int)r) + ")",
            EKV_ECUDA);
    return m;
}

static CUtensorMap make_map_layers(const void* base, uint64_t inner, uint64_t rows, uint64_t layers,
                                   uint64_t layer_stride_elems, uint32_t box_rows) {
    CUtensorMap m;
    cuuint64_t dims[3] = {inner, rows, layers};
    cuuint64_t strides[2] = {inner * 2, layer_stride_elems * 2};
    cuuint32_t box[3] = {(cuuint32_t)k1::BK, box_rows, 1};
    cuuint32_t estr[3] = {1, 1, 1};
    CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(base), dims,
                              strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                              CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                              CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    require(r == CUDA_SUCCESS, "cuTensorMapEncodeTiled failed (" + std::to_string((int)r) + ")",
            EKV_ECUDA);
    return m;
}

void launch_align(const AlignLaunch& p, cudaStream_t st) {
    using namespace k1;
    require(p.m >= 1 && p.m <= kMaxAlignLayers,
            "align_qnorm: 1.." + std::to_string(kMaxAlignLayers) + " matched layers per launch",
            EKV_EUNSUPPORTED);
    require(p.S % BM == 0, "align_qnorm: S must be a multiple of 128", EKV_EUNSUPPORTED);
    require(p.n_cols % BN == 0, "align_qnorm: H*d_c must be a multiple of 256", EKV_EUNSUPPORTED);
    require(p.h_c % BK == 0, "align_qnorm: h_c must be a multiple of 64", EKV_EUNSUPPORTED);
    require(p.fold == 0 || (p.fold >= 1 && BN % p.fold == 0),
            "align_qnorm: folded head_dim must divide 256", EKV_EUNSUPPORTED);
    AlignArgs a{};
    a.m_layers = p.m;
    a.S = p.S;
    a.h_c = p.h_c;
    a.n_cols = p.n_cols;
    a.fold = p.fold;
    a.colsq = p.colsq;
    int x_hi = 0, w_hi = 0;
    for (int i = 0; i < p.m; ++i) {
        a.x_index[i] = p.x_index ? p.x_index[i] : i;
        a.w_index[i] = p.w_index ? p.w_index[i] : i;
        require(a.x_index[i] >= 0 && a.w_index[i] >= 0, "align_qnorm: negative layer index");
        x_hi = std::max(x_hi, a.x_index[i]);
        w_hi = std::max(w_hi, a.w_index[i]);
    }
    if (p.kcolsq) {
        require(p.d_c >= 8 && p.d_c <= 256 && (p.d_c & (p.d_c - 1)) == 0,
                "kv_colnorm (fused): head_dim must be a power of two in [8, 256]", EKV_EUNSUPPORTED);
        require(p.k_layers >= 1 && p.k_layers <= kMaxAlignLayers, "kv_colnorm (fused): bad layer count");
        a.kcolsq = p.kcolsq;
        a.k_layers = p.k_layers;
        a.k_rows = p.k_rows;
        a.d_c = p.d_c;
        for (int i = 0; i < p.k_layers; ++i) {
            require(((uintptr_t)p.k[i] & 15) == 0, "kv_colnorm (fused): K must be 16-byte aligned");
            a.k[i] = (const uint16_t*)p.k[i];
        }
    }
    const uint64_t xs = p.x_stride ? (uint64_t)p.x_stride : (uint64_t)p.S * p.h_c;
    const uint64_t ws = p.w_stride ? (uint64_t)p.w_stride : (uint64_t)p.n_cols * p.h_c;
    require(xs >= (uint64_t)p.S * p.h_c && ws >= (uint64_t)p.n_cols * p.h_c,
            "align_qnorm: layer stride smaller than one layer");
    const CUtensorMap mx = make_map_layers(p.X, p.h_c, p.S, x_hi + 1, xs, BM);
    const CUtensorMap mw = make_map_layers(p.WqT, p.h_c, p.n_cols, w_hi + 1, ws, BN);
    ensure_smem_attr((const void*)align_qnorm_kernel, SMEM_BYTES);
    const int total = p.m * (p.S / BM) * (p.n_cols / BN);
    const int sms = device_sm_count();
    const int grid = total < sms ? total : sms;
    align_qnorm_kernel<<<grid, THREADS, SMEM_BYTES, st>>>(mx, mw, a);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

void launch_align_qnorm_batched(const void* X, const void* WqT, int m_layers, int S, int h_c,
                                int n_cols, double* colsq, int /*num_sms*/, cudaStream_t st) {
    AlignLaunch p{};
    p.X = X;
    p.WqT = WqT;
    p.m = m_layers;
    p.S = S;
    p.h_c = h_c;
    p.n_cols = n_cols;
    p.colsq = colsq;
    launch_align(p, st);
}

void launch_align_qnorm(const void* X, const void* WqT, int S, int h_c, int n_cols, double* colsq,
                        cudaStream_t st) {
    launch_align_qnorm_batched(X, WqT, 1, S, h_c, n_cols, colsq, 0, st);
}

}  // namespace ekv
