// Microbenchmark: HBM -> shared-memory streaming with cp.async.bulk (TMA 1-D)
// through an mbarrier ring, one producer lane per CTA, consumers that only
// touch and release each stage.  Measures the achievable chip bandwidth for a
// given stage size / ring depth (design input for k_decode_mega.cu).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o bulk_bw tools/bulk_bw.cu
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t sa(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void wait(uint64_t* b, uint32_t par) {
    uint32_t d = 0;
    while (!d)
        asm volatile("{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\tselp.u32 %0,1,0,p;\n\t}"
                     : "=r"(d) : "r"(sa(b)), "r"(par) : "memory");
}

template <int STAGE, int NST, int NCW>
__global__ void __launch_bounds__((NCW + 1) * 32, 1) stream(const uint8_t* src, size_t per_cta, float* sink) {
    extern __shared__ __align__(128) uint8_t sm[];
    uint64_t* full = (uint64_t*)(sm + NST * STAGE);
    uint64_t* empty = full + NST;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&full[i])));
            asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sa(&empty[i])));
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const uint8_t* base = src + (size_t)blockIdx.x * per_cta;
    const long long nst = per_cta / STAGE;
    if (warp == NCW) {
        if (lane == 0)
            for (long long k = 0; k < nst; ++k) {
                const int s = k % NST;
                wait(&empty[s], ((k / NST) & 1) ^ 1);
                asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sa(&full[s])), "r"(STAGE) : "memory");
                asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                             ::"r"(sa(sm + s * STAGE)), "l"(base + k * STAGE), "r"(STAGE), "r"(sa(&full[s])) : "memory");
            }
        return;
    }
    float acc = 0.f;
    for (long long k = warp; k < nst; k += NCW) {
        const int s = k % NST;
        wait(&full[s], (k / NST) & 1);
        acc += ((const float*)(sm + s * STAGE))[lane];
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sa(&empty[s])) : "memory");
    }
    if (acc == 12345.f) sink[0] = acc;
}

template <int STAGE, int NST, int NCW>
void run(const uint8_t* src, size_t total, float* sink, int sms) {
    auto fn = stream<STAGE, NST, NCW>;
    const int smem = NST * STAGE + 2 * NST * 8;
    cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    size_t per = (total / sms) / STAGE * STAGE;
    cudaEvent_t a, b;
    cudaEventCreate(&a); cudaEventCreate(&b);
    for (int w = 0; w < 3; ++w) fn<<<sms, (NCW + 1) * 32, smem>>>(src, per, sink);
    cudaEventRecord(a);
    const int it = 20;
    for (int w = 0; w < it; ++w) fn<<<sms, (NCW + 1) * 32, smem>>>(src, per, sink);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    printf("stage %6d B x %2d slots, %d consumer warps: %7.1f GB/s  (err %s)\n", STAGE, NST, NCW,
           (double)per * sms * it / (ms * 1e-3) / 1e9, cudaGetErrorString(cudaGetLastError()));
}

int main(int argc, char** argv) {
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    if (argc > 1) {  // aggregate bandwidth of only G streaming CTAs (one per SM)
        const size_t total = (size_t)2 << 30;
        uint8_t* src; float* sink;
        cudaMalloc(&src, total); cudaMalloc(&sink, 4);
        cudaMemset(src, 1, total);
        for (int i = 1; i < argc; ++i) {
            const int g = atoi(argv[i]);
            printf("G=%d ", g);
            run<16384, 12, 4>(src, total, sink, g);
            printf("G=%d ", g);
            run<32768, 6, 2>(src, total, sink, g);
        }
        return 0;
    }
    const size_t total = (size_t)2 << 30;
    uint8_t* src; float* sink;
    cudaMalloc(&src, total); cudaMalloc(&sink, 4);
    cudaMemset(src, 1, total);
    run<4096, 48, 8>(src, total, sink, sms);
    run<8192, 24, 8>(src, total, sink, sms);
    run<12288, 16, 8>(src, total, sink, sms);
    run<16384, 12, 4>(src, total, sink, sms);
    run<24576, 8, 8>(src, total, sink, sms);
    run<32768, 6, 2>(src, total, sink, sms);
    run<65536, 3, 1>(src, total, sink, sms);
    run<12288, 8, 8>(src, total, sink, sms);
    run<12288, 4, 4>(src, total, sink, sms);
    return 0;
}
