// Shared helpers for the sm_100a kernels of the CE-LSLM KV-reuse path.
#pragma once

#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <stdexcept>
#include <string>

#include "ekv_capi.h"

namespace ekv {

// Error carried through the C-ABI layer as (status, message).
struct Error : std::runtime_error {
    int status;
    Error(int s, const std::string& m) : std::runtime_error(m), status(s) {}
};

inline void check_cuda(cudaError_t e, const char* what) {
    if (e != cudaSuccess)
        throw Error(EKV_ECUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
#define EKV_CUDA(x) ::ekv::check_cuda((x), #x)

inline void require(bool ok, const std::string& msg, int status = EKV_EINVAL) {
    if (!ok) throw Error(status, msg);
}

// Kernel launch accounting (ekv_ctx_kernel_launches).
void count_launches(int64_t n);

// Per-device launch properties.  The dynamic shared-memory attribute and the
// occupancy of a kernel belong to the device context, and one process may drive
// several GPUs (one ekv_ctx per host thread), so both are cached per
// (device ordinal, kernel) under a lock, never process-wide.
void ensure_smem_attr(const void* fn, int bytes);   // on the current device
int device_sm_count();                              // SMs of the current device
int blocks_per_sm(const void* fn, int threads, int smem);  // occupancy, current device

constexpr int kWarp = 32;

__device__ __forceinline__ float bf16_lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16_hi(uint32_t w) { return __uint_as_float(w & 0xFFFF0000u); }

__device__ __forceinline__ uint16_t f32_to_bf16_bits(float f) {
    __nv_bfloat16 b = __float2bfloat16_rn(f);
    return *reinterpret_cast<uint16_t*>(&b);
}

__device__ __forceinline__ float warp_sum(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    return v;
}
__device__ __forceinline__ float warp_max(float v) {
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
    return v;
}

// 128-bit streaming load that does not allocate in L1 (weights / KV read once).
__device__ __forceinline__ uint4 ld_stream(const void* p) {
    uint4 r;
    asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                 : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
                 : "l"(p));
    return r;
}

// Rng::mix (rng.hpp:35-40), the counter hash behind every synthetic tensor.
__host__ __device__ __forceinline__ uint64_t mix64(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9E3779B97F4A7C15ull * (b + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

}  // namespace ekv
