// The decode step as ONE persistent kernel (batch-1 collaborative decode).
//
// merged_forward (cache_merge.cpp:156-226) for one new row, all layers:
//   P1  QKV projection of the layer input (input transform fused at layer 0),
//       K/V appended to the session's user cache
//   P2  segment attention over the reused context + causal user segment,
//       merged by the Eq. 5 normaliser rule (cache_merge.cpp:12-80)
//   P3  output projection -> next layer's input (history row at the last layer)
// separated by grid-wide barriers (one CTA per SM, cooperative launch).
//
// Why one kernel: at batch 1 every phase is a few microseconds of HBM traffic
// (25 MB QKV, 8 MB out-proj, 9-17 MB of context per layer), so separate
// kernels spend most of their time ramping up and draining.  Here every byte
// that does not depend on the running activations -- all weights and all
// context K/V -- is streamed by a dedicated producer warp with bulk-async
// copies (TMA 1-D, mbarrier completion) into a 3-stage shared-memory ring, in
// exactly the order the consumer warps will use it, across phase and layer
// boundaries.  The producer never waits on the grid barriers, so HBM keeps
// streaming while the consumers synchronise.  Only the small dynamic data
// (x, q, the user rows, partials) moves through L2 with ld.global.cg.
//
// Work split (static, identical on every CTA): P1 rows [c*3h/G, (c+1)*3h/G),
// P3 rows [c*h/G, ...); P2 splits the flattened (head, 16-row unit) space of
// context ++ user rows evenly, so a CTA touches at most two heads; each head's
// partials (m, l, o) are merged by the last CTA to finish it (atomic counter).
// User rows written by earlier steps are static during a step, so they are
// streamed through the ring like the context; only this step's row is read
// directly.  The activations a phase consumes (x, the attention output, q)
// are staged once per phase into shared memory with 16-byte loads.
#include <math_constants.h>

#include "ekv_common.cuh"
#include "ekv_kernels.h"
#include "ekv_mega.h"

namespace ekv {

namespace mk {

constexpr int NCW = 8;                  // consumer warps
constexpr int THREADS = (NCW + 1) * 32; // + 1 producer warp
constexpr int NST = 16;                 // ring stages (a multiple of NCW: see the ring protocol)
constexpr int STAGE = 12 * 1024;        // bytes per stage
constexpr int UNIT = 16;                // attention rows per partition unit
constexpr float kLog2e = 1.4426950408889634f;
static_assert(NST % NCW == 0, "ring slots must map to a fixed consumer warp");

__device__ __forceinline__ uint32_t saddr(const void* p) {
    return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(saddr(b)), "r"(n));
}
__device__ __forceinline__ void mbar_expect(uint64_t* b, uint32_t bytes) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(saddr(b)), "r"(bytes)
                 : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    const long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(saddr(b)), "r"(parity)
            : "memory");
        if (done) return;
        if (clock64() - t0 > 4000000000ll) __trap();
    }
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            saddr(dst)),
        "l"(src), "r"(bytes), "r"(saddr(bar))
        : "memory");
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    if (bytes) asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// Grid barrier over the consumer warps of every CTA: one 64-bit counter that
// only grows; barrier k of a launch completes when it reaches base + (k+1)*G,
// where base (= the counter value when the launch started) is published by
// CTA 0 at the end of the previous launch.  One red.release + acquire polling,
// no reset on the critical path.
// trace (optional): [2][G] arrival / release timestamps of this barrier.
__device__ __forceinline__ void grid_sync(unsigned long long* count, unsigned long long target,
                                          unsigned long long* trace = nullptr) {
    consumers_sync();
    if (threadIdx.x == 0) {
        if (trace) trace[blockIdx.x] = gtimer();
        asm volatile("red.release.gpu.global.add.u64 [%0], 1;" ::"l"(count) : "memory");
        const long long t0 = clock64();
        unsigned long long v;
        while (true) {
            asm volatile("ld.acquire.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(count) : "memory");
            if (v >= target) break;
            if (clock64() - t0 > 4000000000ll) __trap();
        }
        if (trace) trace[gridDim.x + blockIdx.x] = gtimer();
    }
    consumers_sync();
}

// ---------------------------------------------------------------------------
// Deterministic schedule shared by producer and consumers.
// ---------------------------------------------------------------------------
struct Split {
    int r0, r1;
};
__device__ __forceinline__ Split rows_of(int c, int G, int N) {
    return Split{(int)((long long)c * N / G), (int)((long long)(c + 1) * N / G)};
}

// One CTA's attention work for one head: context rows [c0, c1) (through the
// ring) and user rows [u0, u1) (direct loads).
struct Piece {
    int head, c0, c1, u0, u1, slot;
};

struct AttnPlan {
    int n;
    Piece p[2];
};

__device__ __forceinline__ int ctx_units(int S) { return (S + UNIT - 1) / UNIT; }

__device__ __forceinline__ AttnPlan plan_attention(int c, int G, int H, int S, int nuser) {
    const int cu = ctx_units(S), uu = (nuser + UNIT - 1) / UNIT, per = cu + uu;
    const long long TU = (long long)H * per;
    const long long a = (long long)c * TU / G, b = (long long)(c + 1) * TU / G;
    AttnPlan pl;
    pl.n = 0;
    for (long long u = a; u < b;) {
        const int h = (int)(u / per);
        const long long hend = (long long)(h + 1) * per;
        const long long e = b < hend ? b : hend;
        const int lo = (int)(u - (long long)h * per), hi = (int)(e - (long long)h * per);  // units
        Piece pc;
        pc.head = h;
        pc.c0 = min(lo, cu) * UNIT;
        pc.c1 = min(min(hi, cu) * UNIT, S);
        pc.u0 = max(lo - cu, 0) * UNIT;
        pc.u1 = min(max(hi - cu, 0) * UNIT, nuser);
        pc.slot = pl.n;
        pl.p[pl.n++] = pc;
        u = e;
    }
    return pl;
}

// largest c with floor(c*TU/G) <= unit (32-bit: TU * G < 2^31)
__device__ __forceinline__ int owner32(int unit, int G, int TU) {
    int lo = 0, hi = G - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if (mid * TU / G <= unit) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

// number of CTAs whose unit range intersects head h (the merge fan-in)
__device__ __forceinline__ int owner(long long unit, int G, long long TU) {
    // largest c with floor(c*TU/G) <= unit
    int lo = 0, hi = G - 1;
    while (lo < hi) {
        const int mid = (lo + hi + 1) >> 1;
        if ((long long)mid * TU / G <= unit) lo = mid;
        else hi = mid - 1;
    }
    return lo;
}

template <int D, int FMT>
struct Fmt {
    static constexpr int ROW = FMT == 16 ? D * 2 : (FMT == 8 ? D : D / 2);  // bytes per row
    static constexpr int LPR = ROW / 16;
    static constexpr int EPL = D / LPR;
    static constexpr int RPP = 32 / LPR;
};

// Rows per attention stage: what fits a slot, capped at ATT_ROWS so a head's
// chunk spreads over several consumer warps.
constexpr int ATT_ROWS = 64;
__device__ __forceinline__ int att_stage_rows(int row_bytes, int ng) {
    const int per = 2 * (row_bytes + ng * 4);
    int r = STAGE / per;
    r -= r % UNIT;
    return r < ATT_ROWS ? r : ATT_ROWS;
}

// ---------------------------------------------------------------------------
// expand 16 bytes of K/V into floats (same encoding as k_attn.cu)
// ---------------------------------------------------------------------------
template <int FMT>
__device__ __forceinline__ void expand16(const uint4& v, float* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if constexpr (FMT == 16) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            f[2 * k] = bf16_lo(w[k]);
            f[2 * k + 1] = bf16_hi(w[k]);
        }
    } else if constexpr (FMT == 8) {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t u = w[k] ^ 0x80808080u;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                f[4 * k + b] = __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7440 + b)) - 8388736.0f;
        }
    } else {
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

// Online-softmax state of one lane group (the LPR lanes of one row subgroup).
template <int EPL>
struct OState {
    float m, l, o[EPL];
};

template <int EPL>
__device__ __forceinline__ void ostate_init(OState<EPL>& s) {
    s.m = -CUDART_INF_F;
    s.l = 0.0f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) s.o[e] = 0.0f;
}

// absorb one row: logit x, value row f (already scaled by its dequant scale)
template <int EPL>
__device__ __forceinline__ void ostate_add(OState<EPL>& s, float x, const float* f, float vscale) {
    const float mn = fmaxf(s.m, x);
    const float corr = exp2f((s.m - mn) * kLog2e);  // exp(-inf) = 0 on the first row
    const float p = exp2f((x - mn) * kLog2e);
    s.l = s.l * corr + p;
    const float pv = p * vscale;
#pragma unroll
    for (int e = 0; e < EPL; ++e) s.o[e] = fmaf(pv, f[e], s.o[e] * corr);
    s.m = mn;
}

template <int EPL>
__device__ __forceinline__ void ostate_merge_from(OState<EPL>& s, float m2, float l2, const float* o2) {
    const float mn = fmaxf(s.m, m2);
    if (mn == -CUDART_INF_F) return;
    const float a = exp2f((s.m - mn) * kLog2e), b = exp2f((m2 - mn) * kLog2e);
    s.l = s.l * a + l2 * b;
#pragma unroll
    for (int e = 0; e < EPL; ++e) s.o[e] = s.o[e] * a + o2[e] * b;
    s.m = mn;
}

// ---------------------------------------------------------------------------
// The kernel
// ---------------------------------------------------------------------------
template <int D>
struct Smem {
    uint8_t ring[NST][STAGE];
    uint64_t full[NST];
    uint64_t empty[NST];
    float xs[2048];            // phase input (x or the attention output)
    float qs[2][D];            // q of the (<= 2) heads of this CTA's attention pieces
    uint16_t nk[2][D], nv[2][D];  // this step's user K/V row of those heads (bf16)
    float ws_o[2][2][NCW][D];  // per (piece, context/user, warp) partial output
    float ws_m[2][2][NCW], ws_l[2][2][NCW];
    int merge_heads_n;         // heads this CTA must merge (last to finish them)
    int merge_head[2];
    int hfirst[160], hlast[160];   // head merge: contributing CTA range per head
    int hcount[160];               // head merge: number of contributing (non-idle) CTAs
    int ch0[160];                  // head merge: first head of each CTA (-1: idle CTA)
    int trace_on;
    int phase_id;
    unsigned long long wait_cycles[4];
};

// Diagnostics: %globaltimer stamps of sub-phases of the last layer
// (trace region [(6L+1)G + 32c + idx]).
template <int D>
__device__ __forceinline__ void stamp(const MegaArgs& a, Smem<D>& sm, int idx) {
    if (a.trace && sm.trace_on && threadIdx.x == 0)
        a.trace[(size_t)(6 * a.L + 1) * gridDim.x + (size_t)blockIdx.x * 32 + idx] = gtimer();
}

// Per-piece schedule pieces that go through the ring: context rows [c0, c1) and
// the static user rows [u0, min(u1, ulen)) (written by earlier steps).
__device__ __forceinline__ int user_static_end(const Piece& pc, int ulen) { return min(pc.u1, ulen); }

// The producer's stage sequence as a generator (the consumers walk the same
// sequence implicitly).  A stage is up to 4 contiguous global ranges copied
// back to back into one ring slot.
struct StageDesc {
    int n = 0;
    const void* src[4];
    uint32_t bytes[4];
    uint32_t total = 0;
    __device__ void add(const void* p, uint32_t b) {
        src[n] = p;
        bytes[n++] = b;
        total += b;
    }
};

template <int D>
struct StageGen {
    const MegaArgs* a;
    Split q, o;
    AttnPlan pl;
    int h, ulen, rows_per_w, ucap;
    // cursor: layer, section (0 qkv, 1 attention, 2 out), piece, part (0 ctx, 1 user), row
    int l = 0, sec = 0, piece = 0, part = 0, r = -1;

    __device__ StageGen(const MegaArgs& args, int c, int G, int ul)
        : a(&args), q(rows_of(c, G, 3 * args.H * D)), o(rows_of(c, G, args.H * D)),
          pl(plan_attention(c, G, args.H, args.S, ul + 1)), h(args.H * D), ulen(ul),
          rows_per_w(STAGE / (args.H * D * 2)), ucap(att_stage_rows(D * 2, 0)) {}

    __device__ bool next(StageDesc& d) {
        d = StageDesc{};
        while (l < a->L) {
            const MegaLayer& ly = a->layer[l];
            if (sec == 0 || sec == 2) {
                const Split sp = sec == 0 ? q : o;
                if (r < 0) r = sp.r0;
                if (r < sp.r1) {
                    const int n = min(rows_per_w, sp.r1 - r);
                    d.add((sec == 0 ? ly.wqkv : ly.wo) + (size_t)r * h, (uint32_t)n * h * 2);
                    r += n;
                    return true;
                }
                r = -1;
                if (sec == 0) {
                    sec = 1;
                    piece = 0;
                    part = 0;
                } else {
                    sec = 0;
                    ++l;
                }
                continue;
            }
            // attention section
            if (piece >= pl.n) {
                sec = 2;
                r = -1;
                continue;
            }
            const Piece& pc = pl.p[piece];
            if (part == 0) {
                const int row_b = ly.fmt == 16 ? D * 2 : (ly.fmt == 8 ? D : D / 2);
                const int ng = ly.fmt == 16 ? 0 : D / ly.group;
                const int cap = att_stage_rows(row_b, ng);
                if (r < 0) r = pc.c0;
                if (r < pc.c1) {
                    const int n = min(cap, pc.c1 - r);
                    const size_t base = (size_t)pc.head * a->S + r;
                    const uint32_t kb = n * row_b, sb = n * ng * 4;
                    d.add(ly.ck + base * row_b, kb);
                    d.add(ly.cv + base * row_b, kb);
                    if (ng) {
                        d.add(ly.cks + base * ng, sb);
                        d.add(ly.cvs + base * ng, sb);
                    }
                    r += n;
                    return true;
                }
                part = 1;
                r = -1;
                continue;
            }
            const int ue = user_static_end(pc, ulen);
            if (r < 0) r = pc.u0;
            if (r < ue) {
                const int n = min(ucap, ue - r);
                const size_t base = (size_t)pc.head * a->cap + r;
                d.add(ly.uk + base * D, (uint32_t)n * D * 2);
                d.add(ly.uv + base * D, (uint32_t)n * D * 2);
                r += n;
                return true;
            }
            ++piece;
            part = 0;
            r = -1;
        }
        return false;
    }
};

template <int D>
__device__ void produce(const MegaArgs& a, Smem<D>& sm, int c, int G, int ulen) {
    int stage = 0;
    uint32_t phase = 0;
    // (an HBM->L2 prefetch cursor running ahead of this one was measured to
    // slow the step down -- profiles/r01_megakernel_experiments.txt -- so the
    // ring is fed straight from HBM)
    StageGen<D> main(a, c, G, ulen);
    StageDesc d;
    while (main.next(d)) {
        mbar_wait(&sm.empty[stage], phase ^ 1);
        mbar_expect(&sm.full[stage], d.total);
        uint32_t off = 0;
        for (int i = 0; i < d.n; ++i) {
            bulk_g2s(sm.ring[stage] + off, d.src[i], d.bytes[i], &sm.full[stage]);
            off += d.bytes[i];
        }
        if (++stage == NST) {
            stage = 0;
            phase ^= 1;
        }
    }
}

// Ring protocol.  Producer and consumers walk the same global sequence of
// stages; stage k lives in slot k % NST (phase bit (k / NST) & 1) and is owned
// by consumer warp k % NCW, which alone waits for it, uses it and releases it
// (empty barriers count one arrival), so up to NCW stages are worked on
// concurrently while the producer refills the rest.  NST % NCW == 0 makes every
// slot belong to one warp forever: a warp waits for round r of a slot only
// after it released round r-1 itself, so the parity wait cannot alias.
struct Cursor {
    long long k = 0;  // global index of the first stage of the current phase
};

template <int D>
__device__ __forceinline__ const uint8_t* ring_acquire(Smem<D>& sm, long long k) {
    const long long t0 = clock64();
    mbar_wait(&sm.full[k % NST], (uint32_t)((k / NST) & 1));
    if (sm.trace_on && (threadIdx.x & 31) == 0) atomicAdd(&sm.wait_cycles[sm.phase_id], (unsigned long long)(clock64() - t0));
    return sm.ring[k % NST];
}
template <int D>
__device__ __forceinline__ void ring_release(Smem<D>& sm, long long k) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&sm.empty[k % NST]);
}

// Stage a phase input vector (h floats, in global, written by other CTAs) into
// shared memory with 16-byte coherent loads; optional layer-0 input transform.
template <int D>
__device__ __forceinline__ void stage_vector(Smem<D>& sm, const float* src, int h,
                                             const float* gamma, const float* bias,
                                             const uint16_t* pos_row) {
    for (int i = threadIdx.x; i < h / 4; i += NCW * 32) {
        float4 v = __ldcg(reinterpret_cast<const float4*>(src) + i);
        if (pos_row) {
            const float4 g = reinterpret_cast<const float4*>(gamma)[i];
            const float4 b = reinterpret_cast<const float4*>(bias)[i];
            const uint2 p = reinterpret_cast<const uint2*>(pos_row)[i];
            v.x = g.x * (v.x + bf16_lo(p.x)) + b.x;
            v.y = g.y * (v.y + bf16_hi(p.x)) + b.y;
            v.z = g.z * (v.z + bf16_lo(p.y)) + b.z;
            v.w = g.w * (v.w + bf16_hi(p.y)) + b.w;
        }
        reinterpret_cast<float4*>(sm.xs)[i] = v;
    }
    consumers_sync();
}

// y[n] = sum_k x[k] W[n][k] for the CTA's rows, weights from the ring, x from
// shared memory into registers once (lane holds x[c*256 + lane*8 + e]).
template <int D, int KC, class Epi>
__device__ __forceinline__ void proj_rows(Smem<D>& sm, Cursor& cu, Split rows, int h, Epi epi) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float xr[KC * 8];
#pragma unroll
    for (int c = 0; c < KC; ++c) {
        const float4 a0 = *reinterpret_cast<const float4*>(sm.xs + c * 256 + lane * 8);
        const float4 a1 = *reinterpret_cast<const float4*>(sm.xs + c * 256 + lane * 8 + 4);
        xr[c * 8 + 0] = a0.x; xr[c * 8 + 1] = a0.y; xr[c * 8 + 2] = a0.z; xr[c * 8 + 3] = a0.w;
        xr[c * 8 + 4] = a1.x; xr[c * 8 + 5] = a1.y; xr[c * 8 + 6] = a1.z; xr[c * 8 + 7] = a1.w;
    }
    const int rows_per_w = STAGE / (h * 2);
    const int nst = (rows.r1 - rows.r0 + rows_per_w - 1) / rows_per_w;
    for (int j = (int)((warp - cu.k % NCW + NCW) % NCW); j < nst; j += NCW) {
        const int r = rows.r0 + j * rows_per_w;
        const int n = min(rows_per_w, rows.r1 - r);
        const uint8_t* st = ring_acquire(sm, cu.k + j);
        for (int i = 0; i < n; ++i) {
            const uint16_t* w = (const uint16_t*)(st + (size_t)i * h * 2);
            float acc[KC];
#pragma unroll
            for (int c = 0; c < KC; ++c) {
                const uint4 v = *reinterpret_cast<const uint4*>(w + c * 256 + lane * 8);
                const uint32_t ww[4] = {v.x, v.y, v.z, v.w};
                float a0 = 0.0f;
#pragma unroll
                for (int k = 0; k < 4; ++k) {
                    a0 = fmaf(bf16_lo(ww[k]), xr[c * 8 + 2 * k], a0);
                    a0 = fmaf(bf16_hi(ww[k]), xr[c * 8 + 2 * k + 1], a0);
                }
                acc[c] = a0;
            }
#pragma unroll
            for (int c = 1; c < KC; ++c) acc[0] += acc[c];
            const float v = warp_sum(acc[0]);
            if (lane == 0) epi(r + i, v);
        }
        ring_release(sm, cu.k + j);
    }
    cu.k += nst;
}

// Attention of q over n <= ATT_ROWS rows (a ring stage, or global memory for
// this step's user row) owned by the calling warp, into this lane's state.
// Two passes per stage: all logits of the lane-group's rows first (registers),
// then one rescale of the running state and one exp per row.
template <int D, int FMT>
__device__ __forceinline__ void attend_rows_mk(const uint8_t* kb, const uint8_t* vb, const float* ks,
                                               const float* vs, int ng, int group, int n,
                                               const float* qreg, OState<Fmt<D, FMT>::EPL>& st,
                                               bool global_src) {
    using F = Fmt<D, FMT>;
    constexpr int MAXR = (ATT_ROWS + F::RPP - 1) / F::RPP;  // rows per lane group per stage
    const int lane = threadIdx.x & 31;
    const int sub = lane % F::LPR, rsub = lane / F::LPR;
    const int grp = FMT == 16 ? 0 : (sub * F::EPL) / group;
    // pass 1: lane-partial dots of every row (independent LDS + FMA chains),
    // then the LPR-lane reductions of all rows together (independent shuffles)
    float lg[MAXR];
#pragma unroll
    for (int p = 0; p < MAXR; ++p) {
        const int row = p * F::RPP + rsub;
        lg[p] = 0.0f;
        if (p * F::RPP < n && row < n) {
            const uint8_t* kp = kb + (size_t)row * F::ROW + sub * 16;
            const uint4 kv = global_src ? __ldcg(reinterpret_cast<const uint4*>(kp))
                                        : *reinterpret_cast<const uint4*>(kp);
            float f[F::EPL];
            expand16<FMT>(kv, f);
            float d0 = 0.0f, d1 = 0.0f;
#pragma unroll
            for (int e = 0; e < F::EPL; e += 2) {
                d0 = fmaf(qreg[e], f[e], d0);
                d1 = fmaf(qreg[e + 1], f[e + 1], d1);
            }
            float dot = d0 + d1;
            if constexpr (FMT != 16) dot *= ks[(size_t)row * ng + grp];
            lg[p] = dot;
        }
    }
#pragma unroll
    for (int o = F::LPR >> 1; o > 0; o >>= 1)
#pragma unroll
        for (int p = 0; p < MAXR; ++p)
            if (p * F::RPP < n) lg[p] += __shfl_xor_sync(0xffffffffu, lg[p], o);
    float mx = -CUDART_INF_F;
#pragma unroll
    for (int p = 0; p < MAXR; ++p) {
        const int row = p * F::RPP + rsub;
        if (p * F::RPP < n && row < n) mx = fmaxf(mx, lg[p]);
    }
    if (mx == -CUDART_INF_F) return;  // no rows for this lane group
    const float mn = fmaxf(st.m, mx);
    const float corr = exp2f((st.m - mn) * kLog2e);
    st.l *= corr;
#pragma unroll
    for (int e = 0; e < F::EPL; ++e) st.o[e] *= corr;
    st.m = mn;
#pragma unroll
    for (int p = 0; p < MAXR; ++p) {
        const int row = p * F::RPP + rsub;
        if (p * F::RPP < n && row < n) {
            const float pr = exp2f((lg[p] - mn) * kLog2e);
            const uint8_t* vp = vb + (size_t)row * F::ROW + sub * 16;
            const uint4 vv = global_src ? __ldcg(reinterpret_cast<const uint4*>(vp))
                                        : *reinterpret_cast<const uint4*>(vp);
            float vsc = 1.0f;
            if constexpr (FMT != 16) vsc = vs[(size_t)row * ng + grp];
            float f[F::EPL];
            expand16<FMT>(vv, f);
            st.l += pr;
            const float pv = pr * vsc;
#pragma unroll
            for (int e = 0; e < F::EPL; ++e) st.o[e] = fmaf(pv, f[e], st.o[e]);
        }
    }
}

// Fold the lane-group states of this warp (xor over the row-subgroup lane
// bits) and park the warp's (m, l, o[D]) in shared memory slot [piece][kind].
template <int D, int FMT>
__device__ __forceinline__ void park_warp_state(Smem<D>& sm, OState<Fmt<D, FMT>::EPL>& st, int piece,
                                                int kind) {
    using F = Fmt<D, FMT>;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int sub = lane % F::LPR;
    for (int off = F::LPR; off < 32; off <<= 1) {
        float o2[F::EPL];
        const float m2 = __shfl_xor_sync(0xffffffffu, st.m, off);
        const float l2 = __shfl_xor_sync(0xffffffffu, st.l, off);
#pragma unroll
        for (int e = 0; e < F::EPL; ++e) o2[e] = __shfl_xor_sync(0xffffffffu, st.o[e], off);
        ostate_merge_from<F::EPL>(st, m2, l2, o2);
    }
    if (lane < F::LPR) {
#pragma unroll
        for (int e = 0; e < F::EPL; ++e) sm.ws_o[piece][kind][warp][sub * F::EPL + e] = st.o[e];
    }
    if (lane == 0) {
        sm.ws_m[piece][kind][warp] = st.m;
        sm.ws_l[piece][kind][warp] = st.l;
    }
}

// Merge of one head's partials by one warp (Eq. 5 generalised to the CTAs
// that attended the head): every load issued before any use, shuffle-free
// per-lane math (each lane owns D/32 output columns), result to a.concat.
template <int D>
__device__ __forceinline__ void merge_one_head(const MegaArgs& a, Smem<D>& sm, int hh) {
    constexpr int MAXC = 8;
    constexpr int VPL = (D + 31) / 32;
    const int lane = threadIdx.x & 31;
    const int first = sm.hfirst[hh], last = sm.hlast[hh];
    float M = -CUDART_INF_F, Ls = 0.0f, O[VPL];
#pragma unroll
    for (int t = 0; t < VPL; ++t) O[t] = 0.0f;
    for (int c0 = first; c0 <= last; c0 += MAXC) {
        float m[MAXC], l[MAXC], v[MAXC][VPL];
#pragma unroll
        for (int j = 0; j < MAXC; ++j) {
            const int cc = c0 + j;
            const bool ok = cc <= last && sm.ch0[cc] >= 0;
            const int sl = ok && sm.ch0[cc] == hh ? 0 : 1;
            const float* pp = a.ws + ((size_t)(ok ? cc : first) * 2 + sl) * (D + 2);
            m[j] = ok ? __ldcg(pp) : -CUDART_INF_F;
            l[j] = ok ? __ldcg(pp + 1) : 0.0f;
#pragma unroll
            for (int t = 0; t < VPL; ++t) {
                const int cix = lane + 32 * t;
                v[j][t] = (ok && cix < D) ? __ldcg(pp + 2 + cix) : 0.0f;
            }
        }
        float Mn = M;
#pragma unroll
        for (int j = 0; j < MAXC; ++j)
            if (l[j] > 0.0f) Mn = fmaxf(Mn, m[j]);
        const float corr = M == -CUDART_INF_F ? 0.0f : exp2f((M - Mn) * kLog2e);
        Ls *= corr;
#pragma unroll
        for (int t = 0; t < VPL; ++t) O[t] *= corr;
#pragma unroll
        for (int j = 0; j < MAXC; ++j) {
            const float w = l[j] > 0.0f ? exp2f((m[j] - Mn) * kLog2e) : 0.0f;
            Ls += l[j] * w;
#pragma unroll
            for (int t = 0; t < VPL; ++t) O[t] += w * v[j][t];
        }
        M = Mn;
    }
    const float inv = 1.0f / Ls;
#pragma unroll
    for (int t = 0; t < VPL; ++t) {
        const int cix = lane + 32 * t;
        if (cix < D) a.concat[hh * D + cix] = O[t] * inv;
    }
}

template <int D, int FMT>
__device__ __forceinline__ void attention_phase(const MegaArgs& a, const MegaLayer& ly, Smem<D>& sm,
                                                Cursor& cu, const AttnPlan& pl, int c, int G,
                                                int ulen) {
    stamp(a, sm, 10);
    using F = Fmt<D, FMT>;
    using FU = Fmt<D, 16>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ng = FMT == 16 ? 0 : D / ly.group;
    const int cap = att_stage_rows(F::ROW, ng);
    const int ucap = att_stage_rows(D * 2, 0);
    // q and this step's user K/V row of the heads this CTA attends (written by
    // P1 on other CTAs): one round of coherent loads into shared memory
    for (int i = 0; i < pl.n; ++i) {
        for (int t = threadIdx.x; t < D / 4; t += NCW * 32)
            reinterpret_cast<float4*>(sm.qs[i])[t] =
                __ldcg(reinterpret_cast<const float4*>(a.q + pl.p[i].head * D) + t);
        if (ulen >= pl.p[i].u0 && ulen < pl.p[i].u1) {
            const size_t row = ((size_t)pl.p[i].head * a.cap + ulen) * D;
            for (int t = threadIdx.x; t < D / 8; t += NCW * 32) {
                reinterpret_cast<uint4*>(sm.nk[i])[t] = __ldcg(reinterpret_cast<const uint4*>(ly.uk + row) + t);
                reinterpret_cast<uint4*>(sm.nv[i])[t] = __ldcg(reinterpret_cast<const uint4*>(ly.uv + row) + t);
            }
        }
    }
    consumers_sync();
    stamp(a, sm, 11);
    for (int i = 0; i < pl.n; ++i) {
        const Piece& pc = pl.p[i];
        {   // context rows (ring)
            float qreg[F::EPL];
            const int sub = lane % F::LPR;
#pragma unroll
            for (int e = 0; e < F::EPL; ++e) qreg[e] = sm.qs[i][sub * F::EPL + e];
            OState<F::EPL> st;
            ostate_init<F::EPL>(st);
            const int nst = (pc.c1 - pc.c0 + cap - 1) / cap;
            for (int j = (int)((warp - cu.k % NCW + NCW) % NCW); j < nst; j += NCW) {
                const int r = pc.c0 + j * cap;
                const int n = min(cap, pc.c1 - r);
                const uint8_t* s = ring_acquire(sm, cu.k + j);
                const int kbytes = n * F::ROW;
                attend_rows_mk<D, FMT>(s, s + kbytes, (const float*)(s + 2 * kbytes),
                                       (const float*)(s + 2 * kbytes + n * ng * 4), ng, ly.group, n,
                                       qreg, st, false);
                ring_release(sm, cu.k + j);
            }
            cu.k += nst;
            park_warp_state<D, FMT>(sm, st, i, 0);
        }
        {   // user rows: earlier steps through the ring, this step's row directly
            float qreg[FU::EPL];
            const int sub = lane % FU::LPR;
#pragma unroll
            for (int e = 0; e < FU::EPL; ++e) qreg[e] = sm.qs[i][sub * FU::EPL + e];
            OState<FU::EPL> su;
            ostate_init<FU::EPL>(su);
            const int ue = user_static_end(pc, ulen);
            const int nst = ue > pc.u0 ? (ue - pc.u0 + ucap - 1) / ucap : 0;
            for (int j = (int)((warp - cu.k % NCW + NCW) % NCW); j < nst; j += NCW) {
                const int r = pc.u0 + j * ucap;
                const int n = min(ucap, ue - r);
                const uint8_t* s = ring_acquire(sm, cu.k + j);
                attend_rows_mk<D, 16>(s, s + n * D * 2, nullptr, nullptr, 0, D, n, qreg, su, false);
                ring_release(sm, cu.k + j);
            }
            cu.k += nst;
            if (ulen >= pc.u0 && ulen < pc.u1 && warp == (int)((cu.k + i) % NCW))
                attend_rows_mk<D, 16>((const uint8_t*)sm.nk[i], (const uint8_t*)sm.nv[i], nullptr,
                                      nullptr, 0, D, 1, qreg, su, false);
            park_warp_state<D, 16>(sm, su, i, 1);
        }
    }
    consumers_sync();
    stamp(a, sm, 12);
    // one CTA-level fold of every (piece, kind, warp) state -> this CTA's partials
    for (int t = threadIdx.x; t < pl.n * D; t += NCW * 32) {
        const int i = t / D, cix = t - i * D;
        float M = -CUDART_INF_F;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int w = 0; w < NCW; ++w)
                if (sm.ws_l[i][k][w] > 0.0f) M = fmaxf(M, sm.ws_m[i][k][w]);
        float Ls = 0.0f, O = 0.0f;
#pragma unroll
        for (int k = 0; k < 2; ++k)
#pragma unroll
            for (int w = 0; w < NCW; ++w) {
                const float l = sm.ws_l[i][k][w];
                if (l > 0.0f) {
                    const float sc = exp2f((sm.ws_m[i][k][w] - M) * kLog2e);
                    Ls += l * sc;
                    O += sm.ws_o[i][k][w][cix] * sc;
                }
            }
        float* outp = a.ws + ((size_t)c * 2 + i) * (D + 2);
        outp[2 + cix] = O;
        if (cix == 0) {
            outp[0] = M;
            outp[1] = Ls;
        }
    }
    consumers_sync();
    // publish; the last CTA to finish a head merges it (one warp per head, every
    // load of the merge in flight at once) into the attention output
    if (threadIdx.x == 0) {
        int nm = 0;
        for (int i = 0; i < pl.n; ++i) {
            const int hh = pl.p[i].head;
            unsigned prev;
            // release: this CTA's partials (ordered by the bar.sync above);
            // acquire: every other contributor's partials for the merger
            asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], 1;"
                         : "=r"(prev) : "l"(&a.head_ctr[hh]) : "memory");
            if (prev == (unsigned)sm.hcount[hh] - 1) {
                a.head_ctr[hh] = 0u;  // re-arm (next use is after a grid barrier)
                sm.merge_head[nm++] = hh;
            }
        }
        sm.merge_heads_n = nm;
    }
    consumers_sync();
    stamp(a, sm, 13);
    if (warp < sm.merge_heads_n) merge_one_head<D>(a, sm, sm.merge_head[warp]);
    consumers_sync();
    stamp(a, sm, 14);
}

// Per-step merge topology (depends only on the step's user length): the first
// head of every CTA's unit range and the contiguous CTA range attending each head.
template <int D>
__device__ __forceinline__ void plan_merge(const MegaArgs& a, Smem<D>& sm, int G, int nuser) {
    const int per = ctx_units(a.S) + (nuser + UNIT - 1) / UNIT;
    const int TU = a.H * per;  // < 2^31 / G for every supported shape (checked at launch)
    for (int cc = threadIdx.x; cc < G; cc += NCW * 32) {
        const int u0 = cc * TU / G, u1 = (cc + 1) * TU / G;
        sm.ch0[cc] = u0 < u1 ? u0 / per : -1;
    }
    consumers_sync();
    for (int hh = threadIdx.x; hh < a.H; hh += NCW * 32) {
        const int f = owner32(hh * per, G, TU), l = owner32((hh + 1) * per - 1, G, TU);
        int n = 0;
        for (int cc = f; cc <= l; ++cc) n += sm.ch0[cc] >= 0;
        sm.hfirst[hh] = f;
        sm.hlast[hh] = l;
        sm.hcount[hh] = n;
    }
    consumers_sync();
}

template <int D, int KC>
__global__ void __launch_bounds__(THREADS, 1) decode_step_kernel(const __grid_constant__ MegaArgs a) {
    extern __shared__ uint8_t smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(((uintptr_t)smem_raw + 127) & ~(uintptr_t)127);
    const int c = blockIdx.x, G = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = a.H * D;
    const int ulen = a.state->user_len;  // user rows before this token
    const int step = a.state->step;
    const unsigned long long base = a.sync[1];  // barrier counter value at launch
    if (a.trace && threadIdx.x == 0) a.trace[(size_t)a.L * 6 * G + c] = gtimer();  // start
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (warp == NCW) {  // producer
        if (lane == 0) produce<D>(a, sm, c, G, ulen);
        return;
    }
    Cursor cu;
    const Split qrows = rows_of(c, G, 3 * h), orows = rows_of(c, G, h);
    const AttnPlan pl = plan_attention(c, G, a.H, a.S, ulen + 1);
    plan_merge<D>(a, sm, G, ulen + 1);
    unsigned long long nb = 0;  // barriers passed in this launch
    for (int l = 0; l < a.L; ++l) {
        const MegaLayer& ly = a.layer[l];
        unsigned long long* tr = a.trace ? a.trace + (size_t)(3 * l) * 2 * G : nullptr;
        // ---- P1: QKV (input transform fused at layer 0) ----
        if (threadIdx.x == 0) {
            sm.trace_on = (l == a.L - 1);
            sm.phase_id = 0;
            for (int i = 0; i < 4; ++i) sm.wait_cycles[i] = 0;
        }
        consumers_sync();
        stamp(a, sm, 0);
        stage_vector<D>(sm, a.x, h, a.gamma, a.bias,
                        l == 0 ? a.pos + (size_t)(a.S + ulen) * h : nullptr);
        stamp(a, sm, 1);
        proj_rows<D, KC>(sm, cu, qrows, h, [&](int n, float v) {
            const int part = n / h, rem = n - part * h;
            if (part == 0) {
                a.q[rem] = v;
            } else {
                const int head = rem / D, cix = rem - head * D;
                uint16_t* dst = part == 1 ? ly.uk : ly.uv;
                dst[((size_t)head * a.cap + ulen) * D + cix] = f32_to_bf16_bits(v);
            }
        });
        stamp(a, sm, 3);
        grid_sync(a.sync, base + (++nb) * G, tr);
        if (threadIdx.x == 0) sm.phase_id = 1;
        // ---- P2: attention ----
        if (ly.fmt == 16) attention_phase<D, 16>(a, ly, sm, cu, pl, c, G, ulen);
        else if (ly.fmt == 8) attention_phase<D, 8>(a, ly, sm, cu, pl, c, G, ulen);
        else attention_phase<D, 4>(a, ly, sm, cu, pl, c, G, ulen);
        grid_sync(a.sync, base + (++nb) * G, tr ? tr + 2 * G : nullptr);
        // ---- P3: output projection ----
        if (threadIdx.x == 0) sm.phase_id = 2;
        stamp(a, sm, 20);
        stage_vector<D>(sm, a.concat, h, nullptr, nullptr, nullptr);
        stamp(a, sm, 21);
        const bool last = l == a.L - 1;
        proj_rows<D, KC>(sm, cu, orows, h, [&](int n, float v) {
            a.x[n] = v;
            if (last) a.hist[(size_t)step * h + n] = v;
        });
        stamp(a, sm, 22);
        if (sm.trace_on && threadIdx.x == 0 && a.trace)
            for (int i = 0; i < 3; ++i)
                a.trace[(size_t)(6 * a.L + 1) * G + (size_t)c * 32 + 28 + i] = sm.wait_cycles[i];

        grid_sync(a.sync, base + (++nb) * G, tr ? tr + 4 * G : nullptr);
    }
    if (c == 0 && threadIdx.x == 0) {
        a.state->user_len = ulen + 1;
        a.state->step = step + 1;
        a.sync[1] = base + nb * G;  // every CTA read `base` before the first barrier
    }
}

}  // namespace mk

size_t mega_smem_bytes(int D) {
    switch (D) {
        case 32: return sizeof(mk::Smem<32>) + 128;
        case 64: return sizeof(mk::Smem<64>) + 128;
        default: return sizeof(mk::Smem<128>) + 128;
    }
}

bool mega_supported(int L, int H, int D, int S, int h) {
    if (L > kMegaMaxLayers || H > 148 || S % mk::UNIT != 0) return false;
    if (!(D == 32 || D == 64 || D == 128)) return false;
    if (h % 256 != 0 || h > 2048) return false;  // x held in registers (KC <= 8)
    if (mk::STAGE / (h * 2) < 1) return false;
    return true;
}

template <int D, int KC>
static void launch_dk(const MegaArgs& a, int grid, cudaStream_t st) {
    auto fn = mk::decode_step_kernel<D, KC>;
    const size_t smem = mega_smem_bytes(D);
    static bool set = false;
    if (!set) {
        EKV_CUDA(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        set = true;
    }
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(mk::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    EKV_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
}

template <int D>
static void launch_d(const MegaArgs& a, int grid, int kc, cudaStream_t st) {
    switch (kc) {
        case 1: launch_dk<D, 1>(a, grid, st); break;
        case 2: launch_dk<D, 2>(a, grid, st); break;
        case 4: launch_dk<D, 4>(a, grid, st); break;
        case 8: launch_dk<D, 8>(a, grid, st); break;
        default: require(false, "decode megakernel: hidden size must be 256/512/1024/2048",
                         EKV_EUNSUPPORTED);
    }
}

void launch_decode_mega(const MegaArgs& a, int num_sms, cudaStream_t st) {
    require(num_sms <= 160, "decode megakernel: at most 160 SMs", EKV_EUNSUPPORTED);
    const int kc = a.H * a.D / 256;
    switch (a.D) {
        case 32: launch_d<32>(a, num_sms, kc, st); break;
        case 64: launch_d<64>(a, num_sms, kc, st); break;
        case 128: launch_d<128>(a, num_sms, kc, st); break;
        default: require(false, "decode megakernel: head_dim must be 32, 64 or 128", EKV_EUNSUPPORTED);
    }
    EKV_CUDA(cudaGetLastError());
    count_launches(1);
}

}  // namespace ekv
