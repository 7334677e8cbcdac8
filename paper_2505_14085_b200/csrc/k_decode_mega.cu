// The decode step as ONE persistent kernel (batch-1 collaborative decode).
//
// merged_forward (cache_merge.cpp:156-226) for one new row, all layers, as a
// dataflow over four phases per layer, with no grid-wide barrier:
//   A  QKV projection of the layer input (input transform fused at layer 0);
//      K/V appended to the session's user cache
//   B  segment attention of each head over the reused context + causal user
//      segment, split over CTAs; per-CTA partials (m, l, o)
//   C  per head: merge of the partials by the Eq. 5 normaliser rule
//      (cache_merge.cpp:12-80), then that head's column block of the output
//      projection (split-K over heads): W_o[:, head] . o_head
//   R  per output element: sum of the per-head partials in head order
//      (deterministic) -> next layer's input
// Dependencies are carried by tagged 64-bit words (value | tag, one 8-byte
// store, polled by the reader), so a phase waits only for the few CTAs that
// produce its inputs: B(h) for the A rows of head h, C(h) for the B pieces of
// head h, R for every head's C rows of its elements, A for every element of R.
// One of those waits (A on R) is the per-layer all-to-all of the
// computation itself; nothing else is global.
//
// Why one kernel: at batch 1 every phase is a few microseconds of HBM traffic
// (25 MB QKV, 8 MB out-proj, 9-17 MB of context per layer), so separate
// kernels spend most of their time ramping up and draining.  Every byte that
// does not depend on the running activations -- all weights and all context
// K/V -- is streamed by a dedicated producer warp (TMA: 1-D bulk copies for
// rows, a 2-D tensor map for the W_o head column blocks) into a 16-stage
// shared-memory ring, in exactly the order the consumer warps use it, across
// phase and layer boundaries.  The producer never waits on the dataflow, so
// HBM keeps streaming while the consumers wait for their inputs.
//
// Work split (static, proportional, identical on every CTA): A covers virtual
// rows [c*3h/G, (c+1)*3h/G) of the head-major (head, q|k|v, d) order; B splits
// the flattened (head, 16-row unit) space of context ++ user rows; C splits
// the (head, output row) space; R splits the h output elements.  The three
// head-ordered splits line up, so the CTAs producing and consuming one head's
// data are neighbours, and each CTA touches at most two heads per phase.
#include <math_constants.h>

#include <cmath>
#include <cstdlib>
#include <map>
#include <mutex>
#include <tuple>

#include "ekv_common.cuh"
#include "ekv_kernels.h"
#include "ekv_mega.h"

namespace ekv {

namespace mk {

constexpr int NCW = 8;                  // consumer warps
constexpr int NPW = 2;                  // producer warps (one issuing thread each)
constexpr int THREADS = (NCW + NPW + 1) * 32;  // + the L2 prefetch warp
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
// Slot release.  Relaxed, not release: a consumer has used every value it
// loaded from the slot before it arrives (the loads feed its arithmetic), and a
// release would also wait for the consumer's outstanding global stores (the
// tagged words written from the slot's results) to reach L2 -- a round trip
// per stage on the critical path.
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
    asm volatile("mbarrier.arrive.relaxed.cta.shared::cta.b64 _, [%0];" ::"r"(saddr(b)) : "memory");
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
__device__ __forceinline__ void tma_2d(void* dst, const CUtensorMap* map, int c0, int c1, uint64_t* bar) {
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4}], [%2];" ::"r"(saddr(dst)),
        "l"(map), "r"(saddr(bar)), "r"(c0), "r"(c1)
        : "memory");
}
__device__ __forceinline__ uint4 lds128(const void* p) {
    uint4 v;
    asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
                 : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
                 : "r"(saddr(p)));
    return v;
}
__device__ __forceinline__ void prefetch_l2(const void* src, uint32_t bytes) {
    asm volatile("cp.async.bulk.prefetch.L2.global [%0], %1;" ::"l"(src), "r"(bytes) : "memory");
}
__device__ __forceinline__ void prefetch_tile_l2(const CUtensorMap* map, int c0, int c1) {
    asm volatile("cp.async.bulk.prefetch.tensor.2d.L2.global.tile [%0, {%1, %2}];" ::"l"(map), "r"(c0),
                 "r"(c1)
                 : "memory");
}
// Packed fp32x2 arithmetic (sm_100 FFMA2 / FADD2 / FMUL2): two lanes of fp32
// math per instruction, exactly the IEEE result of each lane.
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

__device__ __forceinline__ void consumers_sync() {
    asm volatile("bar.sync 1, %0;" ::"n"(NCW * 32) : "memory");
}

__device__ __forceinline__ unsigned long long gtimer() {
    unsigned long long t;
    asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
    return t;
}

// ---------------------------------------------------------------------------
// Tagged words.  A word is {float bits (low 32), tag (high 32)}; writers use
// one 8-byte relaxed store, readers one 8-byte relaxed load (single-copy
// atomic), so a matching tag implies the value.  Tags are unique per (launch,
// layer) and never 0, so zero-initialised buffers read as "not ready".
// ---------------------------------------------------------------------------
__device__ __forceinline__ void ll_st(uint64_t* p, float v, uint32_t tag) {
    const unsigned long long w = ((unsigned long long)tag << 32) | __float_as_uint(v);
    asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(w) : "memory");
}
__device__ __forceinline__ unsigned long long ll_ld(const uint64_t* p) {
    unsigned long long w;
    asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(w) : "l"(p) : "memory");
    return w;
}
// finish a word whose first load is w: spin until its tag matches
__device__ __forceinline__ float ll_spin(const uint64_t* p, unsigned long long w, uint32_t tag) {
    if ((uint32_t)(w >> 32) != tag) {
        const long long t0 = clock64();
        do {
            w = ll_ld(p);
            if (clock64() - t0 > 4000000000ll) __trap();
        } while ((uint32_t)(w >> 32) != tag);
    }
    return __uint_as_float((uint32_t)w);
}

// ---------------------------------------------------------------------------
// Head clusters (CL kernels).  When every head has the same number of CTAs
// (G = cs * H, cs <= 8), the CTAs of one head form a thread-block cluster and
// the two intra-head exchanges -- A's q/k/v rows to B, B's partials to the
// merge -- go through distributed shared memory: st.async into every cluster
// CTA's buffer, each store counting its bytes on that CTA's mbarrier, which
// the CTA armed with the layer's byte count (arrive.expect_tx, one arrival).
// No global round trip, no polling, no fence.  The buffers are single: a CTA
// rewrites a peer's buffer for layer l+1 only after that layer's input
// exists, i.e. after every CTA (the peer included) finished reading layer l's
// and re-armed its barrier.
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t cl_rank() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
    return r;
}
__device__ __forceinline__ uint32_t cl_size() {
    uint32_t r;
    asm volatile("mov.u32 %0, %%cluster_nctarank;" : "=r"(r));
    return r;
}
// the same shared-memory offset in cluster CTA `rank`
__device__ __forceinline__ uint32_t cl_map(uint32_t local, uint32_t rank) {
    uint32_t r;
    asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(local), "r"(rank));
    return r;
}
// an asynchronous 4-byte store into a cluster CTA's shared memory that counts
// its bytes on that CTA's mbarrier (complete_tx): no fence, no arrive
__device__ __forceinline__ void cl_st_async(uint32_t addr, float v, uint32_t bar) {
    asm volatile("st.async.shared::cluster.mbarrier::complete_tx::bytes.f32 [%0], %1, [%2];" ::"r"(addr), "f"(v),
                 "r"(bar)
                 : "memory");
}
__device__ __forceinline__ void cl_wait(uint64_t* b, uint32_t parity) {
    uint32_t done = 0;
    const long long t0 = clock64();
    while (true) {
        asm volatile(
            "{\n\t.reg .pred p;\n\t"
            "mbarrier.try_wait.parity.acquire.cluster.shared::cta.b64 p, [%1], %2;\n\t"
            "selp.u32 %0, 1, 0, p;\n\t}"
            : "=r"(done)
            : "r"(saddr(b)), "r"(parity)
            : "memory");
        if (done) return;
        if (clock64() - t0 > 4000000000ll) __trap();
    }
}
__device__ __forceinline__ void cl_sync_all() {
    asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;" ::: "memory");
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

// One CTA's attention work for one head: context rows [c0, c1) and user rows
// [u0, u1); slot = its index in the CTA's plan (0 or 1).
struct Piece {
    int head, c0, c1, u0, u1, slot;
};

struct AttnPlan {
    int n;
    Piece p[2];
};

__device__ __forceinline__ int ctx_units(int S) { return (S + UNIT - 1) / UNIT; }

// Attention split: every head gets its own CTAs (G/H or G/H + 1 of them, the
// first G%H heads one more), and a head's 16-row units are divided evenly among
// them.  A CTA never straddles two heads: measured, a second piece costs a CTA
// ~35% more time than its rows, and the head merge waits for the slowest
// contributor.
struct HeadCtas {
    int head, idx, n, first;  // this CTA is number idx of the n CTAs [first, first+n) of head
};
__device__ __forceinline__ HeadCtas head_ctas(int c, int G, int H) {
    const int base = G / H, extra = G % H, big = extra * (base + 1);
    HeadCtas r;
    if (c < big) {
        r.head = c / (base + 1);
        r.n = base + 1;
        r.first = r.head * (base + 1);
    } else {
        r.head = extra + (c - big) / base;
        r.n = base;
        r.first = big + (r.head - extra) * base;
    }
    r.idx = c - r.first;
    return r;
}

__device__ __forceinline__ AttnPlan plan_attention(int c, int G, int H, int S, int nuser) {
    const int cu = ctx_units(S), uu = (nuser + UNIT - 1) / UNIT, per = cu + uu;
    const HeadCtas hc = head_ctas(c, G, H);
    const int lo = hc.idx * per / hc.n, hi = (hc.idx + 1) * per / hc.n;  // units
    AttnPlan pl;
    pl.n = 0;
    if (lo < hi) {
        Piece pc;
        pc.head = hc.head;
        pc.c0 = min(lo, cu) * UNIT;
        pc.c1 = min(min(hi, cu) * UNIT, S);
        pc.u0 = max(lo - cu, 0) * UNIT;
        pc.u1 = min(max(hi - cu, 0) * UNIT, nuser);
        pc.slot = 0;
        pl.p[pl.n++] = pc;
    }
    return pl;
}

// One CTA's output-projection work for one head: rows [n0, n1) of W_o[:, head].
struct OPiece {
    int head, n0, n1;
};
struct OPlan {
    int n;
    OPiece p[2];
};
__device__ __forceinline__ OPlan plan_outproj(int c, int G, int H, int h) {
    const long long TW = (long long)H * h;
    const long long a = (long long)c * TW / G, b = (long long)(c + 1) * TW / G;
    OPlan pl;
    pl.n = 0;
    for (long long w = a; w < b;) {
        const int hd = (int)(w / h);
        const long long e = b < (long long)(hd + 1) * h ? b : (long long)(hd + 1) * h;
        pl.p[pl.n++] = OPiece{hd, (int)(w - (long long)hd * h), (int)(e - (long long)hd * h)};
        w = e;
    }
    return pl;
}

// virtual (head, part, d) QKV row -> physical row of W_qkv ([q | k | v] x h)
__device__ __forceinline__ int qkv_phys(int v, int D, int h) {
    const int head = v / (3 * D), rem = v - head * 3 * D, part = rem / D;
    return part * h + head * D + (rem - part * D);
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

// the same 16 bytes as EPL/2 packed fp32 pairs (consecutive elements)
template <int FMT>
__device__ __forceinline__ void expand16_2(const uint4& v, f2x* f) {
    const uint32_t w[4] = {v.x, v.y, v.z, v.w};
    if constexpr (FMT == 16) {
#pragma unroll
        for (int k = 0; k < 4; ++k) f[k] = bf16x2_to_f2(w[k]);
    } else if constexpr (FMT == 8) {
        const f2x bias = f2pack(-8388736.0f, -8388736.0f);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t u = w[k] ^ 0x80808080u;
            f[2 * k] = fadd2(f2pack(__uint_as_float(__byte_perm(u, 0x4B000000u, 0x7440)),
                                    __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7441))), bias);
            f[2 * k + 1] = fadd2(f2pack(__uint_as_float(__byte_perm(u, 0x4B000000u, 0x7442)),
                                        __uint_as_float(__byte_perm(u, 0x4B000000u, 0x7443))), bias);
        }
    } else {
        const f2x bias = f2pack(-8388616.0f, -8388616.0f);
#pragma unroll
        for (int k = 0; k < 4; ++k) {
            const uint32_t lo = (w[k] & 0x0F0F0F0Fu) ^ 0x08080808u;
            const uint32_t hi = ((w[k] >> 4) & 0x0F0F0F0Fu) ^ 0x08080808u;
#pragma unroll
            for (int b = 0; b < 4; ++b)
                f[4 * k + b] = fadd2(f2pack(__uint_as_float(__byte_perm(lo, 0x4B000000u, 0x7440 + b)),
                                            __uint_as_float(__byte_perm(hi, 0x4B000000u, 0x7440 + b))), bias);
        }
    }
}

// Online-softmax state of one lane group (the LPR lanes of one row subgroup).
template <int EPL>
struct OState {
    float m, l;
    f2x o[EPL / 2];  // output columns as packed pairs
};

template <int EPL>
__device__ __forceinline__ void ostate_init(OState<EPL>& s) {
    s.m = -CUDART_INF_F;
    s.l = 0.0f;
#pragma unroll
    for (int e = 0; e < EPL / 2; ++e) s.o[e] = 0ull;
}

template <int EPL>
__device__ __forceinline__ void ostate_merge_from(OState<EPL>& s, float m2, float l2, const f2x* o2) {
    const float mn = fmaxf(s.m, m2);
    if (mn == -CUDART_INF_F) return;
    const float a = exp2f((s.m - mn) * kLog2e), b = exp2f((m2 - mn) * kLog2e);
    s.l = s.l * a + l2 * b;
    const f2x a2 = f2pack(a, a), b2 = f2pack(b, b);
#pragma unroll
    for (int e = 0; e < EPL / 2; ++e) s.o[e] = ffma2(s.o[e], a2, fmul2(o2[e], b2));
    s.m = mn;
}

// ---------------------------------------------------------------------------
// Shared memory and diagnostics
// ---------------------------------------------------------------------------
template <int D>
struct Smem {
    uint8_t ring[NST][STAGE];
    uint64_t full[NST];
    uint64_t empty[NST];
    float xs[2048];               // phase input x (A) / per-head partial sums (R)
    float qs[2][D];               // q of the (<= 2) heads of this CTA's attention pieces
    uint16_t nk[2][D], nv[2][D];  // this step's user K/V row of those heads (bf16)
    float os[2][D];               // merged attention output of this CTA's W_o heads
    float ws_o[2][2][NCW][D];     // per (piece, context/user, warp) partial output
    float ws_m[2][2][NCW], ws_l[2][2][NCW];
    AttnPlan pl;                  // this CTA's attention pieces (shared: indexed at run time,
    OPlan op;                     // a per-thread copy would live in local memory)
    int hfirst[160], hlast[160];  // contributing CTA range of each head's attention
    int ch0[160];                 // first attention head of each CTA (-1: idle CTA)
    uint64_t qkv_bar, part_bar;   // CL: head cluster's q/k/v rows, attention partials arrived
    float cpart[8][D + 2];        // CL: (m, l, o) partial of each cluster CTA
    float kvf[2 * D];             // CL: this step's k | v row of the cluster's head (bf16 values)
    volatile long long prod_k[2]; // stages issued so far by each producer (for the prefetcher)
    int tphase;                   // diagnostics: phase of the ring waits being counted
    unsigned long long twait[3];  // diagnostics: ring-wait cycles of A, B, C (sum over warps)
};

// Diagnostics (TR): trace[(l*G + c)*16 + k], k = 0 layer start,
// 1 x ready, 2 A done, 3 q/k/v ready, 4 B done, 5 partials merged, 6 C done,
// 7 R done (%globaltimer ns); 8..10 = consumer ring-wait cycles in A, B, C.
// trace[(L*G + c)*16 + k]: 0 CTA start, 1/2 producer start/end (ns), 3 stages
// issued, 4 producer cycles waiting for free slots, 5 producer cycles total.
__device__ __forceinline__ void stamp(const MegaArgs& a, bool tr, int l, int k) {
    if (tr && threadIdx.x == 0) a.trace[((size_t)l * gridDim.x + blockIdx.x) * 16 + k] = gtimer();
}
template <class SM>
__device__ __forceinline__ void set_tphase(bool tr, SM& sm, int ph) {
    if (tr && threadIdx.x == 0) sm.tphase = ph;
}

// Per-piece schedule pieces that go through the ring: context rows [c0, c1) and
// the static user rows [u0, min(u1, ulen)) (written by earlier steps).
__device__ __forceinline__ int user_static_end(const Piece& pc, int ulen) { return min(pc.u1, ulen); }

// The producer: one thread walks the stage sequence the consumers use, as
// plain nested loops (layer -> QKV rows, attention pieces, W_o pieces), with
// every index in registers: per stage one wait for the slot, one expect_tx and
// 1-4 bulk copies (or one 2-D tensor box).
template <bool PF>
struct Prod {
    uint64_t* full;
    uint64_t* empty;
    uint8_t* ring;
    volatile long long* prod_k;
    const CUtensorMap* map;
    int sel = 0;          // producer: issues the stages with k % NPW == sel
    int dist = 0;         // prefetcher: stays at most `dist` stages ahead of the producers
    long long k = 0;      // global stage index
    long long waited = 0, count = 0;
    bool trace = false;

    __device__ __forceinline__ bool mine() const { return PF || (int)(k % NPW) == sel; }
    __device__ __forceinline__ uint8_t* acquire(uint32_t bytes) {
        if constexpr (PF) {
            const long long t0 = clock64();
            while (min(prod_k[0], prod_k[1]) + dist < k) {
                __nanosleep(64);
                if (clock64() - t0 > 4000000000ll) __trap();
            }
            return nullptr;
        } else {
            const int slot = (int)(k % NST);
            const uint32_t par = (uint32_t)((k / NST) & 1) ^ 1u;
            if (trace) {
                const long long w0 = clock64();
                mbar_wait(&empty[slot], par);
                waited += clock64() - w0;
                ++count;
            } else {
                mbar_wait(&empty[slot], par);
            }
            mbar_expect(&full[slot], bytes);
            return ring + (size_t)slot * STAGE;
        }
    }
    __device__ __forceinline__ void copy(uint8_t* dst, const void* src, uint32_t bytes) {
        if constexpr (PF) prefetch_l2(src, bytes);
        else bulk_g2s(dst, src, bytes, &full[k % NST]);
    }
    __device__ __forceinline__ void tile(uint8_t* dst, int x, int y) {
        if constexpr (PF) prefetch_tile_l2(map, x, y);
        else tma_2d(dst, map, x, y, &full[k % NST]);
    }
    __device__ __forceinline__ void advance() {
        if constexpr (!PF) {
            if ((int)(k % NPW) == sel) prod_k[sel] = k + 1;
        }
        ++k;
    }
};

template <int D, bool PF, bool TR>
__device__ void produce(const MegaArgs& a, Smem<D>& sm, int c, int G, int ulen, int sel) {
    const long long p0 = clock64();
    const unsigned long long g0 = gtimer();
    Prod<PF> pr;
    pr.prod_k = sm.prod_k;
    pr.map = &a.wo_map;
    pr.dist = a.prefetch_stages;
    pr.full = sm.full;
    pr.empty = sm.empty;
    pr.ring = &sm.ring[0][0];
    pr.trace = TR;
    pr.sel = sel;
    const int h = a.H * D;
    const Split q = rows_of(c, G, 3 * h);
    const AttnPlan& pl = sm.pl;
    const OPlan& op = sm.op;
    const int rpw = STAGE / (h * 2);
    const int ucap = att_stage_rows(D * 2, 0);
    constexpr int RPS = STAGE / (2 * D);
    #pragma unroll 1
    for (int l = 0; l < a.L; ++l) {
        const MegaLayer& ly = a.layer[l];
        // A: QKV rows in virtual head-major order; a stage never crosses more
        // than one (head, q|k|v) block boundary (rpw <= D for every supported shape)
        #pragma unroll 1
        for (int r = q.r0; r < q.r1; r += rpw) {
            if (pr.mine()) {
                const int n = min(rpw, q.r1 - r);
                uint8_t* dst = pr.acquire((uint32_t)n * h * 2);
                const int m = min(n, D - r % D);
                pr.copy(dst, ly.wqkv + (size_t)qkv_phys(r, D, h) * h, (uint32_t)m * h * 2);
                if (m < n)
                    pr.copy(dst + (size_t)m * h * 2, ly.wqkv + (size_t)qkv_phys(r + m, D, h) * h,
                            (uint32_t)(n - m) * h * 2);
            }
            pr.advance();
        }
        // B: context rows, then the static user rows, of each piece
        const int row_b = ly.fmt == 16 ? D * 2 : (ly.fmt == 8 ? D : D / 2);
        const int ng = ly.fmt == 16 ? 0 : D / ly.group;
        const int cap = att_stage_rows(row_b, ng);
        #pragma unroll 1
        for (int i = 0; i < pl.n; ++i) {
            const Piece& pc = pl.p[i];
            const uint8_t* ck = ly.ck + (size_t)pc.head * a.S * row_b;
            const uint8_t* cv = ly.cv + (size_t)pc.head * a.S * row_b;
            #pragma unroll 1
            for (int r = pc.c0; r < pc.c1; r += cap) {
                if (pr.mine() && (!PF || a.prefetch_ctx)) {
                    const int n = min(cap, pc.c1 - r);
                    const uint32_t kb = n * row_b, sb = n * ng * 4;
                    uint8_t* dst = pr.acquire(2 * kb + 2 * sb);
                    pr.copy(dst, ck + (size_t)r * row_b, kb);
                    pr.copy(dst + kb, cv + (size_t)r * row_b, kb);
                    if (ng) {
                        const size_t so = ((size_t)pc.head * a.S + r) * ng;
                        pr.copy(dst + 2 * kb, ly.cks + so, sb);
                        pr.copy(dst + 2 * kb + sb, ly.cvs + so, sb);
                    }
                }
                pr.advance();
            }
            const int ue = user_static_end(pc, ulen);
            #pragma unroll 1
            for (int r = pc.u0; r < ue; r += ucap) {
                if (pr.mine() && !PF) {  // (the user rows are L2-resident: written by earlier steps)
                    const int n = min(ucap, ue - r);
                    const size_t base = ((size_t)pc.head * a.cap + r) * D;
                    uint8_t* dst = pr.acquire((uint32_t)n * D * 4);
                    pr.copy(dst, ly.uk + base, (uint32_t)n * D * 2);
                    pr.copy(dst + (size_t)n * D * 2, ly.uv + base, (uint32_t)n * D * 2);
                }
                pr.advance();
            }
        }
        // C: W_o head column blocks, one 2-D box of RPS rows x D columns per stage
        const int row0 = a.wo_row0 + l * a.wo_layer_rows;
        #pragma unroll 1
        for (int i = 0; i < op.n; ++i) {
            #pragma unroll 1
            for (int r = op.p[i].n0; r < op.p[i].n1; r += RPS) {
                if (pr.mine()) {
                    uint8_t* dst = pr.acquire(STAGE);
                    pr.tile(dst, op.p[i].head * D, row0 + r);
                }
                pr.advance();
            }
        }
    }
    if (TR && sel == 0 && !PF) {
        unsigned long long* t = a.trace + ((size_t)a.L * G + c) * 16;
        t[1] = g0;
        t[2] = gtimer();
        t[3] = pr.count;
        t[4] = pr.waited;
        t[5] = clock64() - p0;
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
__device__ __forceinline__ const uint8_t* ring_acquire(Smem<D>& sm, long long k, bool tr = false) {
    if (tr) {
        const long long t0 = clock64();
        mbar_wait(&sm.full[k % NST], (uint32_t)((k / NST) & 1));
        if ((threadIdx.x & 31) == 0) atomicAdd(&sm.twait[sm.tphase], (unsigned long long)(clock64() - t0));
    } else {
        mbar_wait(&sm.full[k % NST], (uint32_t)((k / NST) & 1));
    }
    return sm.ring[k % NST];
}
template <int D>
__device__ __forceinline__ void ring_release(Smem<D>& sm, long long k) {
    __syncwarp();
    if ((threadIdx.x & 31) == 0) mbar_arrive(&sm.empty[k % NST]);
}
__device__ __forceinline__ int first_owned(const Cursor& cu) {
    return (int)(((threadIdx.x >> 5) - cu.k % NCW + NCW) % NCW);
}

// x lives in shared memory swizzled for proj_qkv's register load: lane l takes
// x[c*256 + l*8 .. +8] of every 256-chunk c as two 16-byte loads at lane stride
// 16 B (conflict-free), i.e. float4 index (c, half, l) -> c*64 + half*32 + l.
__device__ __forceinline__ int xs_idx4(int i4) {
    return ((i4 >> 6) << 6) | ((i4 & 1) << 5) | ((i4 & 63) >> 1);
}

// Layer input into shared memory.  Layer 0: the token input with the input
// transform (plain loads: written before the launch).  Later layers: the
// tagged words of R of the previous layer, every load in flight at once.
template <int D>
__device__ __forceinline__ void stage_x(const MegaArgs& a, Smem<D>& sm, int h, int l, uint32_t prev_tag,
                                        int ulen) {
    if (l == 0) {
        const uint16_t* pos_row = a.pos + (size_t)(a.S + ulen) * h;
        for (int i = threadIdx.x; i < h / 4; i += NCW * 32) {
            float4 v = reinterpret_cast<const float4*>(a.x)[i];
            const float4 g = reinterpret_cast<const float4*>(a.gamma)[i];
            const float4 b = reinterpret_cast<const float4*>(a.bias)[i];
            const uint2 p = reinterpret_cast<const uint2*>(pos_row)[i];
            v.x = g.x * (v.x + bf16_lo(p.x)) + b.x;
            v.y = g.y * (v.y + bf16_hi(p.x)) + b.y;
            v.z = g.z * (v.z + bf16_lo(p.y)) + b.z;
            v.w = g.w * (v.w + bf16_hi(p.y)) + b.w;
            reinterpret_cast<float4*>(sm.xs)[xs_idx4(i)] = v;
        }
    } else {
        constexpr int W = 2048 / (NCW * 32);  // words per thread at the largest h
        unsigned long long w[W];
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int i = k * NCW * 32 + threadIdx.x;
            if (i < h) w[k] = ll_ld(a.ll_x + i);
        }
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int i = k * NCW * 32 + threadIdx.x;
            if (i < h) sm.xs[xs_idx4(i >> 2) * 4 + (i & 3)] = ll_spin(a.ll_x + i, w[k], prev_tag);
        }
    }
    consumers_sync();
}

// A: y[v] = sum_k x[k] W_qkv[phys(v)][k] for the CTA's virtual rows, weights
// from the ring, x from shared memory into registers once (lane holds
// x[c*256 + lane*8 + e]).  q goes out as tagged words; k and v are rounded to
// bf16, appended to the user cache, and go out as tagged words too.
template <int D, int KC, bool TR, bool CL>
__device__ __forceinline__ void proj_qkv(const MegaArgs& a, const MegaLayer& ly, Smem<D>& sm, Cursor& cu,
                                         Split rows, int h, int ulen, uint32_t tag, uint32_t cs) {
    const int lane = threadIdx.x & 31;
    f2x xr[KC * 4];  // x pairs {x[2k], x[2k+1]} of this lane's 8 elements per chunk
#pragma unroll
    for (int c = 0; c < KC; ++c) {
        const float4 a0 = reinterpret_cast<const float4*>(sm.xs)[c * 64 + lane];
        const float4 a1 = reinterpret_cast<const float4*>(sm.xs)[c * 64 + 32 + lane];
        xr[c * 4 + 0] = f2pack(a0.x, a0.y); xr[c * 4 + 1] = f2pack(a0.z, a0.w);
        xr[c * 4 + 2] = f2pack(a1.x, a1.y); xr[c * 4 + 3] = f2pack(a1.z, a1.w);
    }
    constexpr int RG = 3;  // rows in flight per warp (independent FMA and shuffle chains)
    const int rows_per_w = STAGE / (h * 2);
    const int nst = (rows.r1 - rows.r0 + rows_per_w - 1) / rows_per_w;
    for (int j = first_owned(cu); j < nst; j += NCW) {
        const int r = rows.r0 + j * rows_per_w;
        const int n = min(rows_per_w, rows.r1 - r);
        const uint8_t* st = ring_acquire(sm, cu.k + j, TR);
        for (int i0 = 0; i0 < n; i0 += RG) {
            const uint8_t* wr[RG];
#pragma unroll
            for (int g = 0; g < RG; ++g) wr[g] = st + (size_t)min(i0 + g, n - 1) * h * 2 + lane * 16;
            f2x acc[RG];  // {even, odd} partial sums
#pragma unroll
            for (int g = 0; g < RG; ++g) acc[g] = 0ull;
            // software pipeline: chunk c+1 of every row is loaded before chunk c
            // is consumed (volatile loads keep their order)
            uint4 cur[RG], nxt[RG];
#pragma unroll
            for (int g = 0; g < RG; ++g) cur[g] = lds128(wr[g]);
#pragma unroll
            for (int c = 0; c < KC; ++c) {
                if (c + 1 < KC) {
#pragma unroll
                    for (int g = 0; g < RG; ++g) nxt[g] = lds128(wr[g] + (c + 1) * 512);
                }
#pragma unroll
                for (int g = 0; g < RG; ++g) {
                    const uint32_t ww[4] = {cur[g].x, cur[g].y, cur[g].z, cur[g].w};
#pragma unroll
                    for (int k = 0; k < 4; ++k) acc[g] = ffma2(bf16x2_to_f2(ww[k]), xr[c * 4 + k], acc[g]);
                }
                if (c + 1 < KC) {
#pragma unroll
                    for (int g = 0; g < RG; ++g) cur[g] = nxt[g];
                }
            }
            float y[RG];
#pragma unroll
            for (int g = 0; g < RG; ++g) y[g] = f2lo(acc[g]) + f2hi(acc[g]);
#pragma unroll
            for (int o = 16; o > 0; o >>= 1)
#pragma unroll
                for (int g = 0; g < RG; ++g) y[g] += __shfl_xor_sync(0xffffffffu, y[g], o);
            // lanes 0..RG-1 finish one row each
            const float yv = lane == 0 ? y[0] : (lane == 1 ? y[1] : y[2]);
            if (lane < RG && i0 + lane < n) {
                const int v = r + i0 + lane;
                const int head = v / (3 * D), rem = v - head * 3 * D, part = rem / D;
                if (part == 0) {
                    if constexpr (CL) {
                        const uint32_t dst = saddr(&sm.qs[0][rem]), bar = saddr(&sm.qkv_bar);
                        for (uint32_t rk = 0; rk < cs; ++rk) cl_st_async(cl_map(dst, rk), yv, cl_map(bar, rk));
                    } else {
                        ll_st(a.ll_qkv + v, yv, tag);
                    }
                } else {
                    const uint16_t b = f32_to_bf16_bits(yv);
                    uint16_t* dst = part == 1 ? ly.uk : ly.uv;
                    dst[((size_t)head * a.cap + ulen) * D + (rem - part * D)] = b;
                    if constexpr (CL) {
                        const uint32_t sd = saddr(&sm.kvf[rem - D]), bar = saddr(&sm.qkv_bar);
                        const float bv = __uint_as_float((uint32_t)b << 16);
                        for (uint32_t rk = 0; rk < cs; ++rk) cl_st_async(cl_map(sd, rk), bv, cl_map(bar, rk));
                    } else {
                        ll_st(a.ll_qkv + v, __uint_as_float((uint32_t)b << 16), tag);
                    }
                }
            }
        }
        ring_release(sm, cu.k + j);
    }
    cu.k += nst;
}

// Attention of q over n <= NPASS*RPP rows of a ring stage (or the shared-memory
// copy of this step's user row) owned by the calling warp, into this lane's
// state.  Branch-free: every lane group walks NPASS rows with the row index
// clamped to n-1 and masks the clamped rows out (probability 0), so the passes
// are straight-line code with independent load/FMA/shuffle chains.
// Pass 1 computes all logits, pass 2 does one rescale and one exp per row.
__host__ __device__ constexpr int att_rows_fit(int bytes_per_row) {
    return STAGE / bytes_per_row / UNIT * UNIT < ATT_ROWS ? STAGE / bytes_per_row / UNIT * UNIT : ATT_ROWS;
}
// passes covering the largest stage of a format (quantised: one scale group per
// row, the most rows att_stage_rows can give)
template <int D, int FMT>
__host__ __device__ constexpr int att_passes() {
    return (att_rows_fit(FMT == 16 ? 4 * D : 2 * (Fmt<D, FMT>::ROW + 4)) + Fmt<D, FMT>::RPP - 1) /
           Fmt<D, FMT>::RPP;
}

template <int D, int FMT, int NPASS>
__device__ __forceinline__ void attend_rows_mk(const uint8_t* kb, const uint8_t* vb, const float* ks,
                                               const float* vs, int ng, int group, int n,
                                               const f2x* qreg, OState<Fmt<D, FMT>::EPL>& st) {
    using F = Fmt<D, FMT>;
    constexpr int CP = NPASS < 4 ? NPASS : 4;  // passes per chunk (code size: one chunk body)
    const int lane = threadIdx.x & 31;
    const int sub = lane % F::LPR, rsub = lane / F::LPR;
    const int grp = FMT == 16 ? 0 : (sub * F::EPL) / group;
#pragma unroll 1
    for (int p0 = 0; p0 < NPASS && p0 * F::RPP < n; p0 += CP) {
        float lg[CP];
#pragma unroll
        for (int q = 0; q < CP; ++q) {
            const int row = min((p0 + q) * F::RPP + rsub, n - 1);
            const uint4 kv = *reinterpret_cast<const uint4*>(kb + row * F::ROW + sub * 16);
            f2x f[F::EPL / 2];
            expand16_2<FMT>(kv, f);
            f2x d2 = 0ull;
#pragma unroll
            for (int e = 0; e < F::EPL / 2; ++e) d2 = ffma2(qreg[e], f[e], d2);
            float dot = f2lo(d2) + f2hi(d2);
            if constexpr (FMT != 16) dot *= ks[row * ng + grp];
            lg[q] = dot;
        }
#pragma unroll
        for (int o = F::LPR >> 1; o > 0; o >>= 1)
#pragma unroll
            for (int q = 0; q < CP; ++q) lg[q] += __shfl_xor_sync(0xffffffffu, lg[q], o);
        float mx = -CUDART_INF_F;
#pragma unroll
        for (int q = 0; q < CP; ++q)
            if ((p0 + q) * F::RPP + rsub < n) mx = fmaxf(mx, lg[q]);
        if (mx != -CUDART_INF_F) {  // (no shuffles below: divergence is harmless)
            const float mn = fmaxf(st.m, mx);
            const float corr = exp2f((st.m - mn) * kLog2e);
            st.l *= corr;
            const f2x corr2 = f2pack(corr, corr);
#pragma unroll
            for (int e = 0; e < F::EPL / 2; ++e) st.o[e] = fmul2(st.o[e], corr2);
            st.m = mn;
#pragma unroll
            for (int q = 0; q < CP; ++q) {
                const int row = min((p0 + q) * F::RPP + rsub, n - 1);
                const float pr = (p0 + q) * F::RPP + rsub < n ? exp2f((lg[q] - mn) * kLog2e) : 0.0f;
                const uint4 vv = *reinterpret_cast<const uint4*>(vb + row * F::ROW + sub * 16);
                float vsc = 1.0f;
                if constexpr (FMT != 16) vsc = vs[row * ng + grp];
                f2x f[F::EPL / 2];
                expand16_2<FMT>(vv, f);
                st.l += pr;
                const float pv = pr * vsc;
                const f2x pv2 = f2pack(pv, pv);
#pragma unroll
                for (int e = 0; e < F::EPL / 2; ++e) st.o[e] = ffma2(pv2, f[e], st.o[e]);
            }
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
    if (__all_sync(0xffffffffu, st.m == -CUDART_INF_F)) {  // the warp saw no rows
        if (lane == 0) sm.ws_l[piece][kind][warp] = 0.0f;
        return;
    }
#pragma unroll
    for (int off = F::LPR; off < 32; off <<= 1) {
        f2x o2[F::EPL / 2];
        const float m2 = __shfl_xor_sync(0xffffffffu, st.m, off);
        const float l2 = __shfl_xor_sync(0xffffffffu, st.l, off);
#pragma unroll
        for (int e = 0; e < F::EPL / 2; ++e)
            o2[e] = f2pack(__shfl_xor_sync(0xffffffffu, f2lo(st.o[e]), off),
                           __shfl_xor_sync(0xffffffffu, f2hi(st.o[e]), off));
        ostate_merge_from<F::EPL>(st, m2, l2, o2);
    }
    if (lane < F::LPR) {
#pragma unroll
        for (int e = 0; e < F::EPL / 2; ++e) {
            sm.ws_o[piece][kind][warp][sub * F::EPL + 2 * e] = f2lo(st.o[e]);
            sm.ws_o[piece][kind][warp][sub * F::EPL + 2 * e + 1] = f2hi(st.o[e]);
        }
    }
    if (lane == 0) {
        sm.ws_m[piece][kind][warp] = st.m;
        sm.ws_l[piece][kind][warp] = st.l;
    }
}

// B: attention of the CTA's pieces.  q and this step's K/V row of each head
// arrive as tagged words from A; the context and earlier user rows come
// through the ring.  Ends with one tagged (m, l, o) partial per piece.
template <int D, int FMT, bool TR, bool CL>
__device__ __forceinline__ void attention_phase(const MegaArgs& a, const MegaLayer& ly, Smem<D>& sm,
                                                Cursor& cu, const AttnPlan& pl, int c, int ulen,
                                                int l, uint32_t tag, uint32_t cs) {
    using F = Fmt<D, FMT>;
    using FU = Fmt<D, 16>;
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const int ng = FMT == 16 ? 0 : D / ly.group;
    const int cap = att_stage_rows(F::ROW, ng);
    const int ucap = att_stage_rows(D * 2, 0);
    if constexpr (CL) {
        cl_wait(&sm.qkv_bar, (uint32_t)l & 1u);  // the head's q and k | v rows are in sm.qs / kvf
        if (threadIdx.x == 0 && l + 1 < a.L) mbar_expect(&sm.qkv_bar, 3 * D * 4);  // arm layer l+1
    } else {
        constexpr int W = (2 * 3 * D + NCW * 32 - 1) / (NCW * 32);
        unsigned long long w[W];
        const int nw = pl.n * 3 * D;
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int t = k * NCW * 32 + threadIdx.x;
            if (t < nw) w[k] = ll_ld(a.ll_qkv + (size_t)pl.p[t / (3 * D)].head * 3 * D + t % (3 * D));
        }
#pragma unroll
        for (int k = 0; k < W; ++k) {
            const int t = k * NCW * 32 + threadIdx.x;
            if (t < nw) {
                const int i = t / (3 * D), j = t % (3 * D);
                const float v =
                    ll_spin(a.ll_qkv + (size_t)pl.p[i].head * 3 * D + j, w[k], tag);
                if (j < D) sm.qs[i][j] = v;
                else if (j < 2 * D) sm.nk[i][j - D] = (uint16_t)(__float_as_uint(v) >> 16);
                else sm.nv[i][j - 2 * D] = (uint16_t)(__float_as_uint(v) >> 16);
            }
        }
        consumers_sync();
    }
    stamp(a, TR, l, 3);
    for (int i = 0; i < pl.n; ++i) {
        const Piece& pc = pl.p[i];
        {   // context rows (ring)
            f2x qreg[F::EPL / 2];
            const int sub = lane % F::LPR;
#pragma unroll
            for (int e = 0; e < F::EPL / 2; ++e)
                qreg[e] = f2pack(sm.qs[i][sub * F::EPL + 2 * e], sm.qs[i][sub * F::EPL + 2 * e + 1]);
            OState<F::EPL> st;
            ostate_init<F::EPL>(st);
            const int nst = (pc.c1 - pc.c0 + cap - 1) / cap;
            for (int j = first_owned(cu); j < nst; j += NCW) {
                const int r = pc.c0 + j * cap;
                const int n = min(cap, pc.c1 - r);
                const uint8_t* s = ring_acquire(sm, cu.k + j, TR);
                const int kbytes = n * F::ROW;
                attend_rows_mk<D, FMT, att_passes<D, FMT>()>(s, s + kbytes, (const float*)(s + 2 * kbytes),
                                       (const float*)(s + 2 * kbytes + n * ng * 4), ng, ly.group, n,
                                       qreg, st);
                ring_release(sm, cu.k + j);
            }
            cu.k += nst;
            if constexpr (FMT != 16) park_warp_state<D, FMT>(sm, st, i, 0);
            // user rows: earlier steps through the ring, this step's row from
            // shared memory; bf16 context shares the lane layout, so one state
            OState<FU::EPL> su;
            if constexpr (FMT == 16) {
                su = *reinterpret_cast<OState<FU::EPL>*>(&st);
            } else {
                ostate_init<FU::EPL>(su);
            }
            f2x qu[FU::EPL / 2];
            const int subu = lane % FU::LPR;
#pragma unroll
            for (int e = 0; e < FU::EPL / 2; ++e)
                qu[e] = f2pack(sm.qs[i][subu * FU::EPL + 2 * e], sm.qs[i][subu * FU::EPL + 2 * e + 1]);
            const int ue = user_static_end(pc, ulen);
            const int nsu = ue > pc.u0 ? (ue - pc.u0 + ucap - 1) / ucap : 0;
            for (int j = first_owned(cu); j < nsu; j += NCW) {
                const int r = pc.u0 + j * ucap;
                const int n = min(ucap, ue - r);
                const uint8_t* s = ring_acquire(sm, cu.k + j, TR);
                attend_rows_mk<D, 16, att_passes<D, 16>()>(s, s + n * D * 2, nullptr, nullptr, 0, D, n,
                                                            qu, su);
                ring_release(sm, cu.k + j);
            }
            cu.k += nsu;
            if (ulen >= pc.u0 && ulen < pc.u1 && warp == (int)((cu.k + i) % NCW)) {
                if constexpr (CL) {
                    for (int e = lane; e < D; e += 32) {
                        sm.nk[i][e] = (uint16_t)(__float_as_uint(sm.kvf[e]) >> 16);
                        sm.nv[i][e] = (uint16_t)(__float_as_uint(sm.kvf[D + e]) >> 16);
                    }
                    __syncwarp();
                }
                attend_rows_mk<D, 16, 1>((const uint8_t*)sm.nk[i], (const uint8_t*)sm.nv[i], nullptr,
                                         nullptr, 0, D, 1, qu, su);
            }
            park_warp_state<D, 16>(sm, su, i, FMT == 16 ? 0 : 1);
            if (FMT == 16 && lane == 0) sm.ws_l[i][1][warp] = 0.0f;
        }
    }
    consumers_sync();
    // CTA-level fold of every (piece, kind, warp) state -> this CTA's tagged
    // partials.  Each warp that owns 32 output columns (of one piece: 32 | D)
    // computes the 2*NCW rescale factors itself (one lane per state, shuffled to
    // every lane) -- no second block barrier, no serial warp-0 step.
    static_assert(2 * NCW <= 32, "one lane per (kind, warp) state");
    if constexpr (CL) {
        // one piece (or none: an empty partial, l = 0) into every cluster CTA's cpart[rank]
        static_assert(D <= NCW * 32, "one fold pass");
        if (warp * 32 < D) {
            const int cix = warp * 32 + lane;
            const int k = lane / NCW, w = lane % NCW;
            const bool on = pl.n > 0 && lane < 2 * NCW && sm.ws_l[0][k][w] > 0.0f;
            const float m = on ? sm.ws_m[0][k][w] : -CUDART_INF_F;
            const float M = warp_max(m);
            const float sc = on ? exp2f((m - M) * kLog2e) : 0.0f;
            const float Ls = warp_sum(on ? sm.ws_l[0][k][w] * sc : 0.0f);
            float o0 = 0.0f, o1 = 0.0f;
            if (pl.n > 0) {
#pragma unroll
                for (int ww = 0; ww < NCW; ++ww) {
                    o0 = fmaf(sm.ws_o[0][0][ww][cix], __shfl_sync(0xffffffffu, sc, ww), o0);
                    o1 = fmaf(sm.ws_o[0][1][ww][cix], __shfl_sync(0xffffffffu, sc, NCW + ww), o1);
                }
            }
            const uint32_t dst = saddr(&sm.cpart[cl_rank()][0]), bar = saddr(&sm.part_bar);
            for (uint32_t rk = 0; rk < cs; ++rk) {
                const uint32_t rd = cl_map(dst, rk), rb = cl_map(bar, rk);
                if (warp == 0 && lane == 0) {
                    cl_st_async(rd, M, rb);
                    cl_st_async(rd + 4, Ls, rb);
                }
                cl_st_async(rd + 4 * (2 + cix), o0 + o1, rb);
            }
        }
        return;
    }
    for (int t0 = warp * 32; t0 < pl.n * D; t0 += NCW * 32) {
        const int i = t0 / D, cix = t0 - i * D + lane;
        const int k = lane / NCW, w = lane % NCW;
        const bool on = lane < 2 * NCW && sm.ws_l[i][k][w] > 0.0f;
        const float m = on ? sm.ws_m[i][k][w] : -CUDART_INF_F;
        const float M = warp_max(m);
        const float sc = on ? exp2f((m - M) * kLog2e) : 0.0f;
        uint64_t* outp = a.ll_part + ((size_t)c * 2 + i) * (D + 2);
        if (t0 == i * D) {  // the first warp of the piece publishes (m, l)
            const float Ls = warp_sum(on ? sm.ws_l[i][k][w] * sc : 0.0f);
            if (lane == 0) {
                ll_st(outp, M, tag);
                ll_st(outp + 1, Ls, tag);
            }
        }
        float o0 = 0.0f, o1 = 0.0f;
#pragma unroll
        for (int ww = 0; ww < NCW; ++ww) {
            o0 = fmaf(sm.ws_o[i][0][ww][cix], __shfl_sync(0xffffffffu, sc, ww), o0);
            o1 = fmaf(sm.ws_o[i][1][ww][cix], __shfl_sync(0xffffffffu, sc, NCW + ww), o1);
        }
        ll_st(outp + 2 + cix, o0 + o1, tag);
    }
    // (the next consumers_sync is in the caller, before shared state is reused)
}

// C, part 1: merge of the partials of this CTA's W_o heads (Eq. 5 generalised
// to the CTAs that attended each head).  All consumer threads stage up to 8
// contributors per head at a time into shared memory (every tagged load in
// flight before any use), then one thread per (head, column) folds them
// online; the result is the normalised head output in sm.os[slot].
// Missing contributors are staged as (m = 0, l = 0): every staged value stays
// finite (the staging area is the fold's ws_o, which must stay finite).
template <int D>
__device__ __forceinline__ void merge_heads(const MegaArgs& a, Smem<D>& sm, const OPlan& op, uint32_t tag) {
    constexpr int MAXC = 8, W = D + 2;
    static_assert(2 * MAXC * W <= 2 * 2 * NCW * D, "staging fits the fold buffer");
    float* stage = &sm.ws_o[0][0][0][0];  // [2 slots][MAXC][D + 2]
    const int t = threadIdx.x;
    const int col = t % D, slot = t / D;
    const bool mine = t < op.n * D;
    float M = -CUDART_INF_F, Ls = 0.0f, O = 0.0f;
    int most = 0;
    for (int s2 = 0; s2 < op.n; ++s2) {
        const int hh = op.p[s2].head;
        most = max(most, sm.hlast[hh] - sm.hfirst[hh] + 1);
    }
    consumers_sync();  // the fold has finished reading ws_o
    for (int base = 0; base < most; base += MAXC) {
        constexpr int PER = (2 * MAXC * W + NCW * 32 - 1) / (NCW * 32);
        unsigned long long w[PER];
        const uint64_t* src[PER];
#pragma unroll
        for (int k = 0; k < PER; ++k) {
            const int idx = k * NCW * 32 + t;
            src[k] = nullptr;
            if (idx < op.n * MAXC * W) {
                const int s2 = idx / (MAXC * W), rem = idx - s2 * MAXC * W;
                const int j = rem / W, e = rem - j * W;
                const int hh = op.p[s2].head;
                const int cc = sm.hfirst[hh] + base + j;
                if (cc <= sm.hlast[hh] && sm.ch0[cc] >= 0) {
                    const int sl = sm.ch0[cc] == hh ? 0 : 1;
                    src[k] = a.ll_part + ((size_t)cc * 2 + sl) * W + e;
                    w[k] = ll_ld(src[k]);
                } else {
                    stage[idx] = 0.0f;  // (m, l, o) = 0: ignored (l == 0)
                }
            }
        }
#pragma unroll
        for (int k = 0; k < PER; ++k)
            if (src[k]) stage[k * NCW * 32 + t] = ll_spin(src[k], w[k], tag);
        consumers_sync();
        if (mine) {
            const float* st = stage + slot * MAXC * W;
            float Mn = M;
#pragma unroll
            for (int j = 0; j < MAXC; ++j)
                if (st[j * W + 1] > 0.0f) Mn = fmaxf(Mn, st[j * W]);
            const float corr = M == -CUDART_INF_F ? 0.0f : exp2f((M - Mn) * kLog2e);
            Ls *= corr;
            O *= corr;
#pragma unroll
            for (int j = 0; j < MAXC; ++j) {
                const float l = st[j * W + 1];
                const float sc = l > 0.0f ? exp2f((st[j * W] - Mn) * kLog2e) : 0.0f;
                Ls += l * sc;
                O += st[j * W + 2 + col] * sc;
            }
            M = Mn;
        }
        consumers_sync();
    }
    if (mine) sm.os[slot][col] = O / Ls;
}

// C, part 1 on a head cluster: the cs partials arrived in this CTA's cpart
// (every cluster CTA attends the cluster's head, and is this CTA's W_o head).
template <int D>
__device__ __forceinline__ void merge_cluster(Smem<D>& sm, int l, int L, uint32_t cs) {
    cl_wait(&sm.part_bar, (uint32_t)l & 1u);
    if (threadIdx.x == 0 && l + 1 < L) mbar_expect(&sm.part_bar, cs * (D + 2) * 4);  // arm layer l+1
    const int col = threadIdx.x;
    if (col < D) {
        float M = -CUDART_INF_F;
        for (uint32_t j = 0; j < cs; ++j)
            if (sm.cpart[j][1] > 0.0f) M = fmaxf(M, sm.cpart[j][0]);
        float Ls = 0.0f, O = 0.0f;
        for (uint32_t j = 0; j < cs; ++j) {
            const float lj = sm.cpart[j][1];
            const float sc = lj > 0.0f ? exp2f((sm.cpart[j][0] - M) * kLog2e) : 0.0f;
            Ls += lj * sc;
            O += sm.cpart[j][2 + col] * sc;
        }
        sm.os[0][col] = O / Ls;
    }
}

// C, part 2: rows [n0, n1) of W_o[:, head] (2-D boxes from the ring, RPS rows of
// D bf16 each) dotted with the merged head output -> tagged per-head partials.
template <int D, bool TR>
__device__ __forceinline__ void proj_wo(const MegaArgs& a, Smem<D>& sm, Cursor& cu, const OPiece& op,
                                        int slot, int h, uint32_t tag) {
    constexpr int LPR = D / 8;  // lanes per row, 8 bf16 each
    constexpr int RPP = 32 / LPR;
    constexpr int RPS = STAGE / (2 * D);
    const int lane = threadIdx.x & 31, sub = lane % LPR, rsub = lane / LPR;
    float o[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) o[e] = sm.os[slot][sub * 8 + e];
    uint64_t* out = a.ll_xpart + (size_t)op.head * h;
    const int nst = (op.n1 - op.n0 + RPS - 1) / RPS;
    for (int j = first_owned(cu); j < nst; j += NCW) {
        const int r = op.n0 + j * RPS;
        const int n = min(RPS, op.n1 - r);
        const uint8_t* st = ring_acquire(sm, cu.k + j, TR);
        constexpr int PB = 4;  // passes in flight
        static_assert((RPS / RPP) % PB == 0, "pass batching");
#pragma unroll 1
        for (int p0 = 0; p0 < RPS / RPP; p0 += PB) {
            float dot[PB];
#pragma unroll
            for (int b = 0; b < PB; ++b) {
                const int row = (p0 + b) * RPP + rsub;
                const uint4 w = *reinterpret_cast<const uint4*>(st + row * D * 2 + sub * 16);
                float d0 = bf16_lo(w.x) * o[0], d1 = bf16_hi(w.x) * o[1];
                d0 = fmaf(bf16_lo(w.y), o[2], d0);
                d1 = fmaf(bf16_hi(w.y), o[3], d1);
                d0 = fmaf(bf16_lo(w.z), o[4], d0);
                d1 = fmaf(bf16_hi(w.z), o[5], d1);
                d0 = fmaf(bf16_lo(w.w), o[6], d0);
                d1 = fmaf(bf16_hi(w.w), o[7], d1);
                dot[b] = d0 + d1;
            }
#pragma unroll
            for (int off = LPR >> 1; off > 0; off >>= 1)
#pragma unroll
                for (int b = 0; b < PB; ++b) dot[b] += __shfl_xor_sync(0xffffffffu, dot[b], off);
            if (sub == 0) {
#pragma unroll
                for (int b = 0; b < PB; ++b) {
                    const int row = (p0 + b) * RPP + rsub;
                    if (row < n) ll_st(out + r + row, dot[b], tag);
                }
            }
            if (p0 * RPP + PB * RPP >= n) break;
        }
        ring_release(sm, cu.k + j);
    }
    cu.k += nst;
}

// R: this CTA's output elements [e0, e1): the H per-head partials summed in
// head order.  Tagged for the next layer, or (last layer) the step output.
template <int D>
__device__ __forceinline__ void reduce_heads(const MegaArgs& a, Smem<D>& sm, Split el, int h, bool last,
                                             int step, uint32_t tag) {
    const int ne = el.r1 - el.r0, nw = a.H * ne;
    constexpr int W = 4;  // H * ne <= 64 * 14 < 4 * 256 for every supported shape
    unsigned long long w[W];
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int t = k * NCW * 32 + threadIdx.x;
        if (t < nw) w[k] = ll_ld(a.ll_xpart + (size_t)(t / ne) * h + el.r0 + t % ne);
    }
#pragma unroll
    for (int k = 0; k < W; ++k) {
        const int t = k * NCW * 32 + threadIdx.x;
        if (t < nw) sm.xs[t] = ll_spin(a.ll_xpart + (size_t)(t / ne) * h + el.r0 + t % ne, w[k], tag);
    }
    consumers_sync();
    if (threadIdx.x < ne) {
        float s = 0.0f;
        for (int hh = 0; hh < a.H; ++hh) s += sm.xs[hh * ne + threadIdx.x];
        const int e = el.r0 + threadIdx.x;
        if (last) {
            a.x[e] = s;
            a.hist[(size_t)step * h + e] = s;
        } else {
            ll_st(a.ll_x + e, s, tag);
        }
    }
    consumers_sync();
}

// Per-step merge topology (depends only on the step's user length): the first
// head of every CTA's unit range and the contiguous CTA range attending each head.
template <int D>
__device__ __forceinline__ void plan_merge(const MegaArgs& a, Smem<D>& sm, int G, int nuser) {
    const int per = ctx_units(a.S) + (nuser + UNIT - 1) / UNIT;
    for (int cc = threadIdx.x; cc < G; cc += NCW * 32) {
        const HeadCtas hc = head_ctas(cc, G, a.H);
        const bool busy = hc.idx * per / hc.n < (hc.idx + 1) * per / hc.n;
        sm.ch0[cc] = busy ? hc.head : -1;
        if (hc.idx == 0) {
            sm.hfirst[hc.head] = hc.first;
            sm.hlast[hc.head] = hc.first + hc.n - 1;
        }
    }
    consumers_sync();
}

template <int D, int KC, bool TR, bool CL>
__global__ void __launch_bounds__(THREADS, 1) decode_step_kernel(const __grid_constant__ MegaArgs a) {
    // (declared aligned and cast directly, so every access compiles to LDS/STS:
    // an integer round trip would lose the address space and give generic loads)
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    Smem<D>& sm = *reinterpret_cast<Smem<D>*>(smem_raw);
    const int c = blockIdx.x, G = gridDim.x;
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    const int h = a.H * D;
    const int ulen = a.state->user_len;  // user rows before this token
    const int step = a.state->step;
    const uint32_t epoch = *(volatile unsigned*)a.sync;
    if (TR && threadIdx.x == 0) a.trace[((size_t)a.L * G + c) * 16] = gtimer();  // start
    if (threadIdx.x == 0) {
        for (int i = 0; i < NST; ++i) {
            mbar_init(&sm.full[i], 1);
            mbar_init(&sm.empty[i], 1);
        }
        sm.prod_k[0] = sm.prod_k[1] = 0;
        sm.pl = plan_attention(c, G, a.H, a.S, ulen + 1);
        sm.op = plan_outproj(c, G, a.H, a.H * D);
        if (CL) {  // one arrival (the arming) + the layer's bytes
            mbar_init(&sm.qkv_bar, 1);
            mbar_init(&sm.part_bar, 1);
        }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
        if (CL) {
            mbar_expect(&sm.qkv_bar, 3 * D * 4);
            mbar_expect(&sm.part_bar, cl_size() * (D + 2) * 4);
        }
    }
    __syncthreads();
    if (CL) cl_sync_all();  // every cluster CTA's barriers exist before the first remote arrive
    if (warp >= NCW) {  // producers
        if (lane == 0) {
            if (warp < NCW + NPW) produce<D, false, TR>(a, sm, c, G, ulen, warp - NCW);
            else if (a.prefetch_stages > 0) produce<D, true, TR>(a, sm, c, G, ulen, 0);
        }
        return;
    }
    const uint32_t cs = CL ? cl_size() : 1u;
    Cursor cu;
    const Split qrows = rows_of(c, G, 3 * h), elems = rows_of(c, G, h);
    const AttnPlan& pl = sm.pl;
    const OPlan& op = sm.op;
    // the fold multiplies every parked state by its factor (0 for empty ones):
    // start from finite values
    for (int i = threadIdx.x; i < 2 * 2 * NCW * D; i += NCW * 32) (&sm.ws_o[0][0][0][0])[i] = 0.0f;
    plan_merge<D>(a, sm, G, ulen + 1);
    for (int l = 0; l < a.L; ++l) {
        const MegaLayer& ly = a.layer[l];
        const uint32_t tag = epoch * 128u + (uint32_t)l + 1u;
        stamp(a, TR, l, 0);
        if (TR && threadIdx.x == 0) sm.twait[0] = sm.twait[1] = sm.twait[2] = 0;
        set_tphase(TR, sm, 0);
        // ---- A: QKV (input transform fused at layer 0) ----
        stage_x<D>(a, sm, h, l, tag - 1u, ulen);
        stamp(a, TR, l, 1);
        proj_qkv<D, KC, TR, CL>(a, ly, sm, cu, qrows, h, ulen, tag, cs);
        stamp(a, TR, l, 2);
        set_tphase(TR, sm, 1);
        // ---- B: attention ----
        if (ly.fmt == 16) attention_phase<D, 16, TR, CL>(a, ly, sm, cu, pl, c, ulen, l, tag, cs);
        else if (ly.fmt == 8) attention_phase<D, 8, TR, CL>(a, ly, sm, cu, pl, c, ulen, l, tag, cs);
        else attention_phase<D, 4, TR, CL>(a, ly, sm, cu, pl, c, ulen, l, tag, cs);
        stamp(a, TR, l, 4);
        // ---- C: merge + output-projection column blocks of this CTA's heads ----
        if constexpr (CL) merge_cluster<D>(sm, l, a.L, cs);
        else merge_heads<D>(a, sm, op, tag);
        consumers_sync();
        stamp(a, TR, l, 5);
        set_tphase(TR, sm, 2);
        for (int i = 0; i < op.n; ++i) proj_wo<D, TR>(a, sm, cu, op.p[i], i, h, tag);
        stamp(a, TR, l, 6);
        // ---- R: sum over heads ----
        reduce_heads<D>(a, sm, elems, h, l == a.L - 1, step, tag);
        stamp(a, TR, l, 7);
        if (TR && threadIdx.x == 0)
            for (int i = 0; i < 3; ++i) a.trace[((size_t)l * G + c) * 16 + 8 + i] = sm.twait[i];
    }
    if (c == 0 && threadIdx.x == 0) {
        // every CTA read state/epoch before its first A, and this CTA's last R
        // needed every CTA's last A
        a.state->user_len = ulen + 1;
        a.state->step = step + 1;
        *(volatile unsigned*)a.sync = epoch + 1u;
    }
}

}  // namespace mk

size_t mega_smem_bytes(int D) {
    switch (D) {
        case 32: return sizeof(mk::Smem<32>);
        case 64: return sizeof(mk::Smem<64>);
        default: return sizeof(mk::Smem<128>);
    }
}

int mega_wo_box_rows(int D) { return mk::STAGE / (2 * D); }

bool mega_supported(int L, int H, int D, int S, int h) {
    if (L > kMegaMaxLayers || H > 64 || S % mk::UNIT != 0) return false;
    if (!(D == 32 || D == 64 || D == 128)) return false;
    if (h % 256 != 0 || h > 2048) return false;  // x held in registers (KC <= 8)
    if (mk::STAGE / (h * 2) < 1) return false;
    return true;
}

// Head clusters (the CL kernels): every head has cs = grid / H CTAs, cs in [2, 8],
// and the device can keep all grid / cs clusters resident at once (the dataflow
// spins on its peers, so a cluster that is not scheduled would hang the step).
static int mega_cluster(const void* fn, int grid, int H, size_t smem) {
    if (grid % H != 0) return 1;
    const int cs = grid / H;
    if (cs < 2 || cs > 8) return 1;
    if (const char* e = getenv("EKV_MEGA_CLUSTER"))  // experiments: 0 = off
        if (atoi(e) == 0) return 1;
    static std::mutex mu;
    static std::map<std::tuple<int, const void*, int>, int> fits;
    int dev = 0;
    EKV_CUDA(cudaGetDevice(&dev));
    std::lock_guard<std::mutex> lk(mu);
    auto key = std::make_tuple(dev, fn, cs * 1000 + grid);
    auto it = fits.find(key);
    if (it == fits.end()) {
        cudaLaunchConfig_t cfg{};
        cfg.gridDim = dim3(grid);
        cfg.blockDim = dim3(mk::THREADS);
        cfg.dynamicSmemBytes = smem;
        cudaLaunchAttribute at[1];
        at[0].id = cudaLaunchAttributeClusterDimension;
        at[0].val.clusterDim.x = cs;
        at[0].val.clusterDim.y = 1;
        at[0].val.clusterDim.z = 1;
        cfg.attrs = at;
        cfg.numAttrs = 1;
        int n = 0;
        if (cudaOccupancyMaxActiveClusters(&n, fn, &cfg) != cudaSuccess) {
            cudaGetLastError();
            n = 0;
        }
        it = fits.emplace(key, n * cs >= grid ? cs : 1).first;
    }
    return it->second;
}

template <int D, int KC, bool TR, bool CL>
static void launch_dkt(const MegaArgs& a, int grid, int cs, cudaStream_t st) {
    auto fn = mk::decode_step_kernel<D, KC, TR, CL>;
    const size_t smem = mega_smem_bytes(D);
    ensure_smem_attr((const void*)fn, (int)smem);
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = dim3(grid);
    cfg.blockDim = dim3(mk::THREADS);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    // Co-residency of every CTA (the dataflow spins on its peers): a cooperative launch
    // (with the head clusters' dimension when CL).  Nsight Compute's kernel replay fails
    // cooperative + cluster launches, so under the profiler (its injection environment)
    // the cluster launch goes alone: mega_cluster checked its grid against the clusters
    // the device keeps resident at once, and the profiler serialises kernels.
    static const bool profiled = getenv("NV_NSIGHT_INJECTION_TRANSPORT_TYPE") != nullptr;
    cudaLaunchAttribute at[2];
    at[0].id = cudaLaunchAttributeCooperative;
    at[0].val.cooperative = 1;
    at[1].id = cudaLaunchAttributeClusterDimension;
    at[1].val.clusterDim.x = CL ? cs : 1;
    at[1].val.clusterDim.y = 1;
    at[1].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = CL ? 2 : 1;
    if (CL && profiled) {
        cfg.attrs = at + 1;
        cfg.numAttrs = 1;
    }
    EKV_CUDA(cudaLaunchKernelEx(&cfg, fn, a));
}

// the diagnostics (phase stamps, ring counters) are compiled into a separate
// instantiation, so the production kernel carries none of their code
template <int D, int KC>
static void launch_dk(const MegaArgs& a, int grid, cudaStream_t st) {
    const size_t smem = mega_smem_bytes(D);
    ensure_smem_attr((const void*)mk::decode_step_kernel<D, KC, false, true>, (int)smem);  // (the query)
    const int cs = mega_cluster((const void*)mk::decode_step_kernel<D, KC, false, true>, grid, a.H, smem);
    if (cs > 1) {
        if (a.trace) launch_dkt<D, KC, true, true>(a, grid, cs, st);
        else launch_dkt<D, KC, false, true>(a, grid, cs, st);
    } else {
        if (a.trace) launch_dkt<D, KC, true, false>(a, grid, 1, st);
        else launch_dkt<D, KC, false, false>(a, grid, 1, st);
    }
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

// Grid = a multiple of the head count (every head gets the same number of attention
// CTAs, so no head's merge waits for a CTA that carries a larger share; C2, 32 heads:
// 128 CTAs = 3149 tok/s vs 148 CTAs = 2840), at most the SMs, and no more CTAs than the
// token's bytes need: below ~64 KB per CTA the dataflow's per-CTA synchronisation costs
// more than the extra bandwidth brings (configs[0], 4 layers h = 256, ~4 MB per token:
// 64 CTAs 30.3 k tok/s vs 144 CTAs 23.2 k).
int mega_grid(const MegaArgs& a, int num_sms) {
    const int H = a.H;
    int g = H <= num_sms ? num_sms / H * H : num_sms;
    double bytes = 0.0;
    const double h = (double)a.H * a.D;
    for (int l = 0; l < a.L; ++l) {
        const int f = a.layer[l].fmt;
        bytes += 8.0 * h * h + 2.0 * a.H * a.S * (f == 16 ? 2.0 * a.D : a.D * f / 8.0 + 4.0);
    }
    const int want = (int)std::ceil(bytes / (64.0 * 1024.0) / H) * H;
    if (H <= num_sms && want >= H && want < g) g = want;
    if (const char* e = getenv("EKV_MEGA_GRID")) {  // experiments
        const int v = atoi(e);
        if (v >= 1 && v <= num_sms) g = v;
    }
    return g;
}

void launch_decode_mega(const MegaArgs& a, int num_sms, cudaStream_t st) {
    num_sms = mega_grid(a, num_sms);
    require(num_sms <= 160, "decode megakernel: at most 160 SMs", EKV_EUNSUPPORTED);
    require(a.H * a.D >= num_sms, "decode megakernel: hidden size below the SM count", EKV_EUNSUPPORTED);
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
