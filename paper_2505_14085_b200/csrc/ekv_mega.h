// Launch interface of the persistent decode-step kernel (k_decode_mega.cu).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "ekv_kernels.h"

namespace ekv {

constexpr int kMegaMaxLayers = 64;

struct MegaLayer {
    const uint16_t* wqkv;  // [3h][h] bf16
    const uint16_t* wo;    // [h][h] bf16
    int fmt, group;        // context format of this layer (16 bf16, 8 int8, 4 int4)
    const uint8_t* ck;     // [H][S][row bytes]
    const uint8_t* cv;
    const float* cks;      // [H][S][d/group]
    const float* cvs;
    uint16_t* uk;          // session user cache [H][cap][D]
    uint16_t* uv;
};

struct MegaArgs {
    int L, H, D, S, cap;
    const float* gamma;
    const float* bias;
    const uint16_t* pos;   // [max_pos][h]
    DevState* state;
    float* x;              // [h] layer input / output (token input at entry)
    float* q;              // [h]
    float* concat;         // [h]
    float* hist;           // [cap][h] step outputs
    float* ws;             // [G][2][D+2] attention partials
    unsigned* head_ctr;    // [H], zero
    unsigned long long* sync;  // grid barrier {count, count at launch start}, zero
    unsigned long long* trace;  // optional [3L][2][G] barrier arrival/release + [G] start (ns)
    MegaLayer layer[kMegaMaxLayers];
};

bool mega_supported(int L, int H, int D, int S, int h);
size_t mega_smem_bytes(int D);
void launch_decode_mega(const MegaArgs& a, int num_sms, cudaStream_t st);

}  // namespace ekv
