// Stage 2 kernels: gather (prune_cache), K3 quantise+pack, K6 dequant,
// K2 K-column norms, and the counter-hash synthetic generator.
//
// All of these are HBM-bound byte/integer work: 128-bit or row-wide coalesced
// loads, one warp per row, warp-shuffle reductions, grid sized to a multiple
// of the SM count (grid-stride loops).  No tensor cores.
#include <string>

#include "ekv_common.cuh"
#include "ekv_kernels.h"

namespace ekv {

// ---------------------------------------------------------------------------
// Counter-hash generator (oracle: ekvo_fill_uniform_bf16).
// ---------------------------------------------------------------------------
__global__ void fill_uniform_bf16_kernel(uint16_t* __restrict__ dst, int64_t n, uint64_t base,
                                         double lo, double span) {
    for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n;
         i += (int64_t)gridDim.x * blockDim.x) {
        const double u = (double)(mix64(base, (uint64_t)i) >> 11) * 0x1.0p-53;
        const double x = __dadd_rn(lo, __dmul_rn(span, u));
        __nv_bfloat16 b = __double2bfloat16(x);
        dst[i] = *reinterpret_cast<uint16_t*>(&b);
    }
}

void launch_fill_uniform_bf16(void* dst, int64_t n, uint64_t seed, uint64_t stream_id, double lo,
                              double hi, cudaStream_t st) {
    if (n <= 0) return;
    const int threads = 256;
    int64_t blocks = (n + threads - 1) / threads;
    if (blocks > 148 * 16) blocks = 148 * 16;
    fill_uniform_bf16_kernel<<<(unsigned)blocks, threads, 0, st>>>(
        (uint16_t*)dst, n, mix64(seed, stream_id), lo, hi - lo);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

// ---------------------------------------------------------------------------
// K3: gather + quantise + pack.  Quantiser contract (DESIGN.md s.3, oracle
// ekvo_kv_compress): per row and group, amax = max|x|; amax < 2^-120 -> zero
// group; scale = RN(amax/Q), inv = RN(Q/amax); code = rne(RN(x*inv)).  The
// round-half-even of the fp32 product is done with the 1.5*2^23 magic add,
// whose low mantissa bits ARE the two's-complement code, so a code costs one
// FMUL + one FADD + a byte select (no F2I, no clamp: |x*inv| <= Q(1+2^-22)).
// ---------------------------------------------------------------------------
constexpr float kMagic = 12582912.0f;  // 1.5 * 2^23
constexpr float kTiny = 0x1.0p-120f;

__device__ __forceinline__ uint32_t quant_bits(float x, float inv) {
    return __float_as_uint(__fadd_rn(__fmul_rn(x, inv), kMagic));
}

// Tile kernel: TILE contiguous rows of one job are moved global -> shared by a
// single bulk-async copy (TMA 1D, mbarrier completion) into an NS-stage ring,
// so NS-1 tiles per CTA stay in flight while one is quantised.  Persistent:
// the grid is exactly the resident CTAs, each walking the flattened (job, tile)
// space with a grid stride (no second wave).  8 kept channels per lane, LPR =
// DE/8 lanes per row, 32/LPR rows per warp pass; per-group absmax by xor
// shuffles inside the row's lanes; 8 (int8) or 4 (int4) code bytes stored per
// lane (coalesced rows).
template <int DC>
struct TileCfg {
    static constexpr int TILE = 8192 / DC;              // rows per stage (16 KB)
    static constexpr int BYTES = TILE * DC * 2;         // 16 KB
};
template <int DC, int TB>
struct TileCfgB {                                       // TB-byte stages
    static constexpr int TILE = TB / (2 * DC);
    static constexpr int BYTES = TILE * DC * 2;
};
constexpr int kCompressStages = 2;
// 16 KB x 2 stages.  Round 1 (before the bank-conflict-free gather order) measured 8 KB x 2
// best (4.75-4.80 TB/s; 16 KB x 2 4.61); with the rotated gather (round 2, C2 22 jobs / C4
// 32k 22 jobs, fraction of the 6551 GB/s peak): 8 KB x 2 0.73 / 0.82, 8 KB x 3 0.73 / 0.80,
// 16 KB x 2 0.77-0.79 / 0.87-0.88, 16 KB x 3 0.73 / 0.80, 16 KB x 4 0.64 / 0.69, 32 KB x 2
// 0.69 / 0.75 (profiles/r02_megakernel_experiments.txt has the log).
constexpr int kCompressTileBytes = 16384;

__device__ __forceinline__ uint32_t smem_addr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}

template <int DC, int DE, int BITS, int TB = kCompressTileBytes, int NS = kCompressStages>
__global__ void __launch_bounds__(128) kv_compress_tile_kernel(CompressJobs jobs, int n_jobs, int64_t rows,
                                                               const int* __restrict__ kept,
                                                               int group) {
    using TC = TileCfgB<DC, TB>;
    constexpr int LPR = DE / 8, RPW = 32 / LPR, NWARP = 4;
    constexpr int PASSES = TC::TILE / (RPW * NWARP);
    constexpr float Q = BITS == 8 ? 127.0f : 7.0f;
    static_assert(PASSES >= 1 && TC::TILE % (RPW * NWARP) == 0, "tile shape");
    extern __shared__ __align__(1024) uint8_t dyn[];
    uint8_t (*buf)[TC::BYTES] = reinterpret_cast<uint8_t (*)[TC::BYTES]>(dyn);
    uint64_t* bar = reinterpret_cast<uint64_t*>(dyn + NS * TC::BYTES);
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int sub = lane % LPR, rsub = lane / LPR;
    const int glanes = group / 8;  // lanes per group (power of two, <= LPR)
    const int ng = DE / group;
    // Byte offsets of my kept channels inside a row.  Rows sit 2*DC bytes apart (a
    // multiple of 128 B), so a channel falls in the same shared-memory bank in every
    // row: the RPW row groups of a warp would all hit the same banks when they gather
    // the same channel index.  Each row group walks its 8 channels rotated by 2*rsub
    // instead (different channels -> different banks at every step), and the codes
    // are rotated back into channel order when packed.
    const int rot = 2 * (rsub & 3);
    int ch2[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) ch2[e] = 2 * kept[sub * 8 + ((e + rot) & 7)];
    const int64_t ntiles = (rows + TC::TILE - 1) / TC::TILE;
    const int64_t total = ntiles * n_jobs;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NS; ++i)
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(&bar[i])));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    auto issue = [&](int64_t T, int stage) {
        const int jb = (int)(T / ntiles);
        const int64_t r0 = (T - (int64_t)jb * ntiles) * TC::TILE;
        const int n = (int)min((int64_t)TC::TILE, rows - r0);
        const uint32_t bytes = (uint32_t)n * DC * 2;
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(
                         smem_addr(&bar[stage])),
                     "r"(bytes)
                     : "memory");
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                smem_addr(buf[stage])),
            "l"((const uint8_t*)jobs.job[jb].src + r0 * DC * 2), "r"(bytes), "r"(smem_addr(&bar[stage]))
            : "memory");
    };
    if (threadIdx.x == 0)
        for (int i = 0; i < NS; ++i) {
            const int64_t T = blockIdx.x + (int64_t)i * gridDim.x;
            if (T < total) issue(T, i);
        }
    int it = 0;
    for (int64_t T = blockIdx.x; T < total; T += gridDim.x, ++it) {
        const int stage = it % NS;
        {
            const uint32_t parity = (uint32_t)((it / NS) & 1);
            uint32_t done = 0;
            while (!done) {
                asm volatile(
                    "{\n\t.reg .pred p;\n\t"
                    "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
                    "selp.u32 %0, 1, 0, p;\n\t}"
                    : "=r"(done)
                    : "r"(smem_addr(&bar[stage])), "r"(parity)
                    : "memory");
            }
        }
        const int jb = (int)(T / ntiles);
        const CompressJob job = jobs.job[jb];
        const int64_t r0 = (T - (int64_t)jb * ntiles) * TC::TILE;
        const uint8_t* tile = buf[stage];
#pragma unroll
        for (int p = 0; p < PASSES; ++p) {
            const int lr = (p * NWARP + warp) * RPW + rsub;
            const int64_t row = r0 + lr;
            const uint8_t* rp = tile + lr * (DC * 2);
            float x[8];
            float amax = 0.0f;
#pragma unroll
            for (int e = 0; e < 8; ++e) {
                x[e] = __uint_as_float((uint32_t)(*(const uint16_t*)(rp + ch2[e])) << 16);
                amax = fmaxf(amax, fabsf(x[e]));
            }
            for (int o = glanes >> 1; o > 0; o >>= 1)
                amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            const bool zero = !(amax >= kTiny);
            const float scale = zero ? 0.0f : __fdiv_rn(amax, Q);
            const float inv = zero ? 0.0f : __fdiv_rn(Q, amax);
            uint32_t q[8];
#pragma unroll
            for (int e = 0; e < 8; ++e) q[e] = zero ? 0u : quant_bits(x[e], inv);
            if (row < rows) {
                if ((sub % glanes) == 0) job.scales[row * ng + sub / glanes] = scale;
                if constexpr (BITS == 8) {
                    uint32_t lo = __byte_perm(__byte_perm(q[0], q[1], 0x0040),
                                              __byte_perm(q[2], q[3], 0x0040), 0x5410);
                    uint32_t hi = __byte_perm(__byte_perm(q[4], q[5], 0x0040),
                                              __byte_perm(q[6], q[7], 0x0040), 0x5410);
                    // byte e holds channel (e + rot) & 7: rotate left by rot bytes
                    const uint64_t w = ((uint64_t)hi << 32) | lo;
                    const uint64_t r = rot ? (w << (8 * rot)) | (w >> (64 - 8 * rot)) : w;
                    reinterpret_cast<uint2*>((uint8_t*)job.codes + row * DE)[sub] =
                        make_uint2((uint32_t)r, (uint32_t)(r >> 32));
                } else {
                    uint32_t w = 0;
#pragma unroll
                    for (int e = 0; e < 8; ++e) w |= (q[e] & 0xFu) << (4 * e);
                    // nibble e holds channel (e + rot) & 7: rotate left by rot nibbles
                    w = rot ? (w << (4 * rot)) | (w >> (32 - 4 * rot)) : w;
                    reinterpret_cast<uint32_t*>((uint8_t*)job.codes + row * (DE / 2))[sub] = w;
                }
            }
        }
        __syncthreads();  // every warp is done with this stage before it is refilled
        if (threadIdx.x == 0) {
            const int64_t Tn = T + (int64_t)NS * gridDim.x;
            if (Tn < total) issue(Tn, stage);
        }
    }
}

// Generic path (any d_c, d_e, group): one thread per (row, group).
template <int BITS>
__global__ void kv_compress_generic_kernel(const uint16_t* __restrict__ src, int64_t rows, int d_c,
                                           const int* __restrict__ kept, int d_e, int group,
                                           uint8_t* __restrict__ codes,
                                           float* __restrict__ scales) {
    constexpr float Q = BITS == 8 ? 127.0f : 7.0f;
    const int ng = d_e / group;
    const int row_bytes = d_e * BITS / 8;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * ng;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / ng;
        const int g = (int)(t % ng);
        const uint16_t* s = src + row * d_c;
        float amax = 0.0f;
        for (int c = g * group; c < (g + 1) * group; ++c)
            amax = fmaxf(amax, fabsf(__uint_as_float((uint32_t)s[kept[c]] << 16)));
        const bool zero = !(amax >= kTiny);
        const float scale = zero ? 0.0f : __fdiv_rn(amax, Q);
        const float inv = zero ? 0.0f : __fdiv_rn(Q, amax);
        scales[row * ng + g] = scale;
        uint8_t* crow = codes + row * row_bytes;
        for (int c = g * group; c < (g + 1) * group; ++c) {
            const uint32_t q = zero ? 0u : quant_bits(__uint_as_float((uint32_t)s[kept[c]] << 16), inv);
            if (BITS == 8) {
                crow[c] = (uint8_t)(q & 0xFF);
            } else if ((c & 1) == 0) {
                crow[c >> 1] = (uint8_t)(q & 0xF);  // low nibble first
            } else {
                crow[c >> 1] |= (uint8_t)((q & 0xF) << 4);
            }
        }
    }
}

static int grid_for(int64_t work, int per_block) {
    int64_t b = (work + per_block - 1) / per_block;
    const int64_t cap = 148 * 8;
    if (b > cap) b = cap;
    if (b < 1) b = 1;
    return (int)b;
}

template <int DC, int DE, int BITS, int TB = kCompressTileBytes, int NS = kCompressStages>
static bool try_fast(const CompressJobs& jobs, int n_jobs, int64_t rows, int d_c, const int* kept,
                     int d_e, int group, cudaStream_t st) {
    if (d_c != DC || d_e != DE) return false;
    constexpr int LPR = DE / 8;
    if (group % 8 != 0) return false;
    const int gl = group / 8;
    if (gl < 1 || gl > LPR || (gl & (gl - 1))) return false;
    for (int i = 0; i < n_jobs; ++i)  // bulk copies need 16-byte aligned sources
        if (((uintptr_t)jobs.job[i].src & 15) || ((uintptr_t)jobs.job[i].codes & 7))
            return false;
    using TC = TileCfgB<DC, TB>;
    const int64_t total = (rows + TC::TILE - 1) / TC::TILE * n_jobs;
    auto fn = kv_compress_tile_kernel<DC, DE, BITS, TB, NS>;
    const int smem = NS * TC::BYTES + 64;
    const int occ = blocks_per_sm((const void*)fn, 128, smem);
    const int sms = device_sm_count();
    int64_t grid = (int64_t)sms * occ;  // persistent: exactly the resident CTAs
    if (grid > total) grid = total;
    fn<<<(unsigned)grid, 128, smem, st>>>(jobs, n_jobs, rows, kept, group);
    return true;
}

void launch_kv_compress_jobs(const CompressJob* job, int n_jobs, int64_t rows, int d_c,
                             const int* kept, int d_e, int bits, int group, cudaStream_t st) {
    if (rows <= 0 || n_jobs <= 0) return;
    require(n_jobs <= kMaxCompressJobs, "kv_compress: at most " +
                                            std::to_string(kMaxCompressJobs) + " jobs per launch");
    CompressJobs jobs{};
    for (int i = 0; i < n_jobs; ++i) jobs.job[i] = job[i];
    bool done = false;
    if (bits == 8) {
        done = try_fast<128, 64, 8>(jobs, n_jobs, rows, d_c, kept, d_e, group, st) ||
               try_fast<64, 32, 8>(jobs, n_jobs, rows, d_c, kept, d_e, group, st) ||
               try_fast<128, 128, 8>(jobs, n_jobs, rows, d_c, kept, d_e, group, st) ||
               try_fast<256, 128, 8>(jobs, n_jobs, rows, d_c, kept, d_e, group, st) ||
               try_fast<64, 64, 8>(jobs, n_jobs, rows, d_c, kept, d_e, group, st);
    } else {
        done = try_fast<128, 64, 4>(jobs, n_jobs, rows, d_c, kept, d_e, group, st) ||
               try_fast<64, 32, 4>(jobs, n_jobs, rows, d_c, kept, d_e, group, st) ||
               try_fast<128, 128, 4>(jobs, n_jobs, rows, d_c, kept, d_e, group, st) ||
               try_fast<256, 128, 4>(jobs, n_jobs, rows, d_c, kept, d_e, group, st) ||
               try_fast<64, 64, 4>(jobs, n_jobs, rows, d_c, kept, d_e, group, st);
    }
    if (done) {
        count_launches(1);
    } else {
        const int64_t work = rows * (d_e / group);
        for (int i = 0; i < n_jobs; ++i) {
            if (bits == 8)
                kv_compress_generic_kernel<8><<<grid_for(work, 256), 256, 0, st>>>(
                    (const uint16_t*)job[i].src, rows, d_c, kept, d_e, group,
                    (uint8_t*)job[i].codes, job[i].scales);
            else
                kv_compress_generic_kernel<4><<<grid_for(work, 256), 256, 0, st>>>(
                    (const uint16_t*)job[i].src, rows, d_c, kept, d_e, group,
                    (uint8_t*)job[i].codes, job[i].scales);
        }
        count_launches(n_jobs);
    }
    EKV_CUDA(cudaGetLastError());
}

void launch_kv_compress(const void* src, int64_t rows, int d_c, const int* kept, int d_e, int bits,
                        int group, void* codes, float* scales, cudaStream_t st) {
    CompressJob j{src, codes, scales};
    launch_kv_compress_jobs(&j, 1, rows, d_c, kept, d_e, bits, group, st);
}

// ---------------------------------------------------------------------------
// prune_cache gather (bf16 copy of the kept channels).
// ---------------------------------------------------------------------------
__global__ void kv_gather_kernel(const uint16_t* __restrict__ src, int64_t rows, int d_c,
                                 const int* __restrict__ kept, int d_e,
                                 uint16_t* __restrict__ dst) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * d_e;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / d_e;
        const int c = (int)(t % d_e);
        dst[t] = src[row * d_c + kept[c]];
    }
}

template <class T>
__global__ void gather_columns_kernel(const T* __restrict__ src, int64_t rows, int d_c,
                                      const int* __restrict__ kept, int d_e, T* __restrict__ dst) {
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * d_e;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / d_e;
        dst[t] = src[row * d_c + kept[t - row * d_e]];
    }
}

void launch_gather_columns(const void* src, int64_t rows, int d_c, const int* kept, int d_e,
                           int elem_bytes, void* dst, cudaStream_t st) {
    if (rows <= 0) return;
    const int g = grid_for(rows * d_e, 256);
    switch (elem_bytes) {
        case 2: gather_columns_kernel<uint16_t><<<g, 256, 0, st>>>((const uint16_t*)src, rows, d_c, kept, d_e, (uint16_t*)dst); break;
        case 4: gather_columns_kernel<uint32_t><<<g, 256, 0, st>>>((const uint32_t*)src, rows, d_c, kept, d_e, (uint32_t*)dst); break;
        case 8: gather_columns_kernel<uint64_t><<<g, 256, 0, st>>>((const uint64_t*)src, rows, d_c, kept, d_e, (uint64_t*)dst); break;
        default: require(false, "gather_columns: element size must be 2, 4 or 8 bytes");
    }
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

void launch_kv_gather(const void* src, int64_t rows, int d_c, const int* kept, int d_e, void* dst,
                      cudaStream_t st) {
    if (rows <= 0) return;
    kv_gather_kernel<<<grid_for(rows * d_e, 256), 256, 0, st>>>((const uint16_t*)src, rows, d_c,
                                                                kept, d_e, (uint16_t*)dst);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

// ---------------------------------------------------------------------------
// K6 dequant: bf16_rn(fp32(code) * scale).
// ---------------------------------------------------------------------------
template <int BITS>
__global__ void kv_dequant_kernel(const uint8_t* __restrict__ codes,
                                  const float* __restrict__ scales, int64_t rows, int d_e,
                                  int group, uint16_t* __restrict__ dst) {
    const int ng = d_e / group;
    const int row_bytes = d_e * BITS / 8;
    for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < rows * d_e;
         t += (int64_t)gridDim.x * blockDim.x) {
        const int64_t row = t / d_e;
        const int c = (int)(t % d_e);
        int code;
        if (BITS == 8) {
            code = (int)(int8_t)codes[row * row_bytes + c];
        } else {
            int nib = (codes[row * row_bytes + (c >> 1)] >> ((c & 1) * 4)) & 0xF;
            code = nib >= 8 ? nib - 16 : nib;
        }
        const float v = __fmul_rn((float)code, scales[row * ng + c / group]);
        dst[t] = f32_to_bf16_bits(v);
    }
}

void launch_kv_dequant(const void* codes, const float* scales, int64_t rows, int d_e, int bits,
                       int group, void* dst, cudaStream_t st) {
    if (rows <= 0) return;
    if (bits == 8)
        kv_dequant_kernel<8><<<grid_for(rows * d_e, 256), 256, 0, st>>>(
            (const uint8_t*)codes, scales, rows, d_e, group, (uint16_t*)dst);
    else
        kv_dequant_kernel<4><<<grid_for(rows * d_e, 256), 256, 0, st>>>(
            (const uint8_t*)codes, scales, rows, d_e, group, (uint16_t*)dst);
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

// ---------------------------------------------------------------------------
// K2: per-column sums of squares of K [rows][d_c] (bf16) -> fp64 (+=).
// Each thread owns 8 consecutive channels (one 16-byte load per row), sums
// its rows in fp32, the block folds its threads in fp64, one double atomic
// per column per block.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) kv_colnorm_kernel(const uint16_t* __restrict__ K,
                                                         int64_t rows, int d_c,
                                                         double* __restrict__ colsq) {
    extern __shared__ double red[];  // [d_c]
    const int tpr = d_c / 8;         // threads per row
    const int rpp = blockDim.x / tpr;  // rows per pass
    const int t = threadIdx.x;
    for (int c = t; c < d_c; c += blockDim.x) red[c] = 0.0;
    __syncthreads();
    float acc[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (t < rpp * tpr) {
        const int cseg = t % tpr;
        for (int64_t r = blockIdx.x * (int64_t)rpp + t / tpr; r < rows; r += (int64_t)gridDim.x * rpp) {
            uint4 v = ld_stream(K + r * d_c + cseg * 8);
            const uint32_t w[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
            for (int k = 0; k < 4; ++k) {
                const float a = bf16_lo(w[k]), b = bf16_hi(w[k]);
                acc[2 * k] = fmaf(a, a, acc[2 * k]);
                acc[2 * k + 1] = fmaf(b, b, acc[2 * k + 1]);
            }
        }
#pragma unroll
        for (int k = 0; k < 8; ++k) atomicAdd(&red[cseg * 8 + k], (double)acc[k]);
    }
    __syncthreads();
    for (int c = t; c < d_c; c += blockDim.x) atomicAdd(&colsq[c], red[c]);
}

__global__ void kv_colnorm_generic_kernel(const uint16_t* __restrict__ K, int64_t rows, int d_c,
                                          double* __restrict__ colsq) {
    // one thread per column, grid-stride over row blocks of 256
    const int c = threadIdx.x;
    if (c >= d_c) return;
    double acc = 0.0;
    for (int64_t r = blockIdx.x; r < rows; r += gridDim.x) {
        const float a = __uint_as_float((uint32_t)K[r * d_c + c] << 16);
        acc += (double)(a * a);
    }
    atomicAdd(&colsq[c], acc);
}

void launch_kv_colnorm(const void* K, int64_t rows, int d_c, double* colsq, cudaStream_t st) {
    if (rows <= 0) return;
    if (d_c % 8 == 0 && d_c / 8 <= 256) {
        const int tpr = d_c / 8, rpp = 256 / tpr;
        int64_t blocks = (rows + rpp - 1) / rpp;
        if (blocks > 148 * 4) blocks = 148 * 4;
        kv_colnorm_kernel<<<(unsigned)blocks, 256, sizeof(double) * d_c, st>>>(
            (const uint16_t*)K, rows, d_c, colsq);
    } else {
        require(d_c <= 1024, "kv_colnorm: head_dim > 1024", EKV_EUNSUPPORTED);
        kv_colnorm_generic_kernel<<<148 * 4, d_c, 0, st>>>((const uint16_t*)K, rows, d_c, colsq);
    }
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

}  // namespace ekv
