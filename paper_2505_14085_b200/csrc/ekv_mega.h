// Launch interface of the persistent decode-step kernel (k_decode_mega.cu).
#pragma once

#include <cuda.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include "ekv_kernels.h"

namespace ekv {

constexpr int kMegaMaxLayers = 64;

struct MegaLayer {
    const uint16_t* wqkv;  // [3h][h] bf16 (rows: q | k | v, head-major inside each)
    int fmt, group;        // context format of this layer (16 bf16, 8 int8, 4 int4)
    const uint8_t* ck;     // [H][S][row bytes]
    const uint8_t* cv;
    const float* cks;      // [H][S][d/group]
    const float* cvs;
    uint16_t* uk;          // session user cache [H][cap][D]
    uint16_t* uv;
};

// Tagged words ("LL" words): 64-bit {value bits, tag}, written and read with
// single 8-byte accesses, so a reader polling a word sees either a stale tag
// or the complete value -- data and its ready flag travel together.
struct MegaArgs {
    int L, H, D, S, cap;
    const float* gamma;
    const float* bias;
    const uint16_t* pos;   // [max_pos][h]
    DevState* state;
    float* x;              // [h] token input at entry, last-layer output at exit
    float* hist;           // [cap][h] step outputs
    uint64_t* ll_x;        // [h]        layer output (sum over heads), tagged
    uint64_t* ll_xpart;    // [H][h]     per-head output-projection partials, tagged
    uint64_t* ll_qkv;      // [H][3][D]  this token's q, k, v (k, v bf16-rounded), tagged
    uint64_t* ll_part;     // [G][2][D+2] attention partials (m, l, o) per CTA piece, tagged
    unsigned* sync;        // [0] launch epoch (tags are epoch*128 + layer + 1), zero-initialised
    unsigned long long* trace;  // optional [L][G][8] phase stamps + [G] start (ns)
    CUtensorMap wo_map;    // 2-D map over the weight buffer: rows [L*4h] x cols [h], box {D, rows}
    int wo_row0, wo_layer_rows;  // row of layer l's W_o = wo_row0 + l*wo_layer_rows
    int prefetch_stages;   // L2 prefetch warp distance ahead of the ring, in stages (0 = off; default 16)
    int prefetch_ctx;      // the prefetch warp also covers the context stages (else weights only)
    MegaLayer layer[kMegaMaxLayers];
};

bool mega_supported(int L, int H, int D, int S, int h);
size_t mega_smem_bytes(int D);
int mega_wo_box_rows(int D);
int mega_grid(const MegaArgs& a, int num_sms);  // CTAs of the persistent kernel (a multiple of H)
void launch_decode_mega(const MegaArgs& a, int num_sms, cudaStream_t st);
CUtensorMap make_map_2d_bf16(const void* base, uint64_t inner, uint64_t rows, uint32_t box_inner,
                             uint32_t box_rows);

}  // namespace ekv
