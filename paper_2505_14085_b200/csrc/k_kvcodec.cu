// Stage 2 kernels: gather (prune_cache), K3 quantise+pack, K6 dequant,
// K2 K-column norms, and the counter-hash synthetic generator.
//
// All of these are HBM-bound byte/integer work: 128-bit or row-wide coalesced
// loads, one warp per row, warp-shuffle reductions, grid sized to a multiple
// of the SM count (grid-stride loops).  No tensor cores.
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
// K3 fast path: one warp per row of DC bf16 channels (row-wide coalesced
// load, DC/32 channels per lane), gather of the DE kept channels by warp
// shuffles, per-group absmax by shuffles, quantise, pack, coalesced store.
// Quantiser contract (DESIGN.md s.3 / oracle ekvo_kv_compress):
//   scale = amax / Q; code = clamp(rint(x / scale), -Q, Q); scale==0 -> 0.
// ---------------------------------------------------------------------------
template <int DC>
struct RowLoad;  // lane-local slice of one row
template <>
struct RowLoad<64> {
    uint32_t w[1];
};
template <>
struct RowLoad<128> {
    uint32_t w[2];
};
template <>
struct RowLoad<256> {
    uint32_t w[4];
};

template <int DC>
__device__ __forceinline__ RowLoad<DC> load_row(const uint16_t* row, int lane) {
    RowLoad<DC> r;
    if constexpr (DC == 64) {
        r.w[0] = __ldcs(reinterpret_cast<const uint32_t*>(row) + lane);
    } else if constexpr (DC == 128) {
        uint2 v = __ldcs(reinterpret_cast<const uint2*>(row) + lane);
        r.w[0] = v.x;
        r.w[1] = v.y;
    } else {
        uint4 v = __ldcs(reinterpret_cast<const uint4*>(row) + lane);
        r.w[0] = v.x;
        r.w[1] = v.y;
        r.w[2] = v.z;
        r.w[3] = v.w;
    }
    return r;
}

// Channel ch lives in lane ch / (DC/32), word (ch % (DC/32)) / 2, half ch & 1.
template <int DC>
__device__ __forceinline__ float fetch_channel(const RowLoad<DC>& r, int ch) {
    constexpr int EPL = DC / 32;  // elements per lane
    const int src = ch / EPL;
    const int wsel = (ch % EPL) >> 1;
    uint32_t got = 0;
#pragma unroll
    for (int k = 0; k < EPL / 2; ++k) {
        uint32_t v = __shfl_sync(0xffffffffu, r.w[k], src);
        if (k == wsel) got = v;
    }
    return (ch & 1) ? bf16_hi(got) : bf16_lo(got);
}

template <int DC, int DE, int BITS>
__global__ void __launch_bounds__(256) kv_compress_fast_kernel(CompressJobs jobs, int64_t rows,
                                                               const int* __restrict__ kept,
                                                               int group) {
    // one job (layer x {K, V}) per blockIdx.y: a single launch compresses every deep layer
    const uint16_t* __restrict__ src = (const uint16_t*)jobs.job[blockIdx.y].src;
    uint8_t* __restrict__ codes = (uint8_t*)jobs.job[blockIdx.y].codes;
    float* __restrict__ scales = jobs.job[blockIdx.y].scales;
    constexpr int EPL = DE / 32;  // kept channels per lane (1, 2 or 4)
    constexpr float Q = BITS == 8 ? 127.0f : 7.0f;
    const int lane = threadIdx.x & 31;
    const int ng = DE / group;
    const int glanes = group / EPL;  // lanes per group (power of two)
    int ch[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e) ch[e] = kept[lane * EPL + e];
    const int64_t warp0 = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5;
    const int64_t nwarps = ((int64_t)gridDim.x * blockDim.x) >> 5;
    constexpr int UNROLL = 4;
    for (int64_t base = warp0 * UNROLL; base < rows; base += nwarps * UNROLL) {
        RowLoad<DC> rl[UNROLL];
#pragma unroll
        for (int u = 0; u < UNROLL; ++u)
            if (base + u < rows) rl[u] = load_row<DC>(src + (base + u) * DC, lane);
#pragma unroll
        for (int u = 0; u < UNROLL; ++u) {
            const int64_t row = base + u;
            if (row >= rows) break;
            float x[EPL];
            float amax = 0.0f;
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                x[e] = fetch_channel<DC>(rl[u], ch[e]);
                amax = fmaxf(amax, fabsf(x[e]));
            }
            for (int o = glanes >> 1; o > 0; o >>= 1)
                amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
            const float scale = __fdiv_rn(amax, Q);
            int code[EPL];
#pragma unroll
            for (int e = 0; e < EPL; ++e) {
                int c = 0;
                if (scale != 0.0f) {
                    float r = rintf(__fdiv_rn(x[e], scale));
                    r = fminf(fmaxf(r, -Q), Q);
                    c = (int)r;
                }
                code[e] = c;
            }
            if ((lane % glanes) == 0) scales[row * ng + lane / glanes] = scale;
            if constexpr (BITS == 8) {
                uint8_t* crow = codes + row * DE;
                if constexpr (EPL == 1) {
                    crow[lane] = (uint8_t)code[0];
                } else if constexpr (EPL == 2) {
                    reinterpret_cast<uint16_t*>(crow)[lane] =
                        (uint16_t)((code[0] & 0xFF) | ((code[1] & 0xFF) << 8));
                } else {
                    reinterpret_cast<uint32_t*>(crow)[lane] =
                        (uint32_t)((code[0] & 0xFF) | ((code[1] & 0xFF) << 8) |
                                   ((code[2] & 0xFF) << 16) | ((uint32_t)(code[3] & 0xFF) << 24));
                }
            } else {
                uint8_t* crow = codes + row * (DE / 2);
                if constexpr (EPL == 1) {
                    // pair lanes (2j, 2j+1) into one byte
                    int other = __shfl_down_sync(0xffffffffu, code[0], 1);
                    if ((lane & 1) == 0) crow[lane >> 1] = (uint8_t)((code[0] & 0xF) | ((other & 0xF) << 4));
                } else if constexpr (EPL == 2) {
                    crow[lane] = (uint8_t)((code[0] & 0xF) | ((code[1] & 0xF) << 4));
                } else {
                    reinterpret_cast<uint16_t*>(crow)[lane] =
                        (uint16_t)((code[0] & 0xF) | ((code[1] & 0xF) << 4) | ((code[2] & 0xF) << 8) |
                                   ((code[3] & 0xF) << 12));
                }
            }
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
        const float scale = __fdiv_rn(amax, Q);
        scales[row * ng + g] = scale;
        uint8_t* crow = codes + row * row_bytes;
        for (int c = g * group; c < (g + 1) * group; ++c) {
            int code = 0;
            if (scale != 0.0f) {
                float r = rintf(__fdiv_rn(__uint_as_float((uint32_t)s[kept[c]] << 16), scale));
                code = (int)fminf(fmaxf(r, -Q), Q);
            }
            if (BITS == 8) {
                crow[c] = (uint8_t)code;
            } else if ((c & 1) == 0) {
                crow[c >> 1] = (uint8_t)(code & 0xF);  // low nibble first
            } else {
                crow[c >> 1] |= (uint8_t)((code & 0xF) << 4);
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

template <int DC, int DE, int BITS>
static bool try_fast(const CompressJobs& jobs, int n_jobs, int64_t rows, int d_c, const int* kept,
                     int d_e, int group, cudaStream_t st) {
    if (d_c != DC || d_e != DE) return false;
    constexpr int EPL = DE / 32;
    if (group % EPL != 0) return false;
    const int gl = group / EPL;
    if (gl < 1 || gl > 32 || (gl & (gl - 1))) return false;
    const int64_t warps = (rows + 3) / 4;
    int bx = grid_for(warps * 32, 256);
    const int cap = (148 * 8 + n_jobs - 1) / n_jobs;  // ~8 CTAs per SM over all jobs
    if (bx > cap) bx = cap < 1 ? 1 : cap;
    kv_compress_fast_kernel<DC, DE, BITS><<<dim3(bx, n_jobs), 256, 0, st>>>(jobs, rows, kept, group);
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
