/*
 * ekv_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement (plain C99, fp64) of the CE-LSLM cloud->edge KV-reuse hot
 * path of the reference artifact (/root/reference/proj), used as the parity
 * checker for the B200 kernels.  Only tests/, __graft_entry__.smoke() and
 * bench.py's cpu_baseline leg may load this library; the product
 * (paper_2505_14085_b200) never links or calls it.
 *
 * Every function cites the reference file:line it restates.  Pinning: the
 * restatement is checked bit-for-bit against the reference compiled from its
 * own sources (oracle/_ref, see oracle/Makefile) and against the reference's
 * golden values (model checksum fa0d3d12020757f7, from_lambda budgets,
 * tie-break rule, ...) in tests/test_oracle_pinned.py.
 *
 * The int8/int4 quantiser has NO reference (SPEC.md:281, 488 list cache
 * quantisation as a non-goal): its section below is this build's own contract
 * and is "parity unpinned vs reference".
 *
 * Build with -ffp-contract=off (no FMA contraction) so fp64 results are the
 * same bits as the reference built with g++ -O2 on x86-64.
 */
#include <math.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>

#define EKVO_EXPORT __attribute__((visibility("default")))

/* ------------------------------------------------------------------------ */
/* RNG: rng.hpp:13-45 (mt19937_64 + hand-mapped 53-bit uniform), rng.cpp    */
/* ------------------------------------------------------------------------ */

/* Rng::mix, rng.hpp:35-40 (splitmix64 finaliser of a + golden*(b+1)). */
EKVO_EXPORT uint64_t ekvo_mix(uint64_t a, uint64_t b) {
    uint64_t z = a + 0x9E3779B97F4A7C15ull * (b + 1);
    z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
    z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
    return z ^ (z >> 31);
}

typedef struct {
    uint64_t mt[312];
    int idx;
    uint64_t seed;
} mt64_t;

/* std::mt19937_64 (the standard fixes its output bit-for-bit). */
static void mt64_seed(mt64_t* g, uint64_t seed) {
    g->seed = seed;
    g->mt[0] = seed;
    for (int i = 1; i < 312; ++i)
        g->mt[i] = 6364136223846793005ull * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
    g->idx = 312;
}

static uint64_t mt64_next(mt64_t* g) {
    static const uint64_t UM = 0xFFFFFFFF80000000ull, LM = 0x7FFFFFFFull;
    if (g->idx >= 312) {
        for (int i = 0; i < 312; ++i) {
            uint64_t x = (g->mt[i] & UM) | (g->mt[(i + 1) % 312] & LM);
            uint64_t xa = x >> 1;
            if (x & 1ull) xa ^= 0xB5026F5AA96619E9ull;
            g->mt[i] = g->mt[(i + 156) % 312] ^ xa;
        }
        g->idx = 0;
    }
    uint64_t y = g->mt[g->idx++];
    y ^= (y >> 29) & 0x5555555555555555ull;
    y ^= (y << 17) & 0x71D67FFFEDA60000ull;
    y ^= (y << 37) & 0xFFF7EEE000000000ull;
    y ^= y >> 43;
    return y;
}

/* Rng::uniform(lo, hi), rng.hpp:22-24. */
static double mt64_uniform(mt64_t* g, double lo, double hi) {
    double u = (double)(mt64_next(g) >> 11) * 0x1.0p-53;
    return lo + (hi - lo) * u;
}

/* Rng::fork, rng.hpp:31. */
static void mt64_fork(const mt64_t* parent, uint64_t stream, mt64_t* child) {
    mt64_seed(child, ekvo_mix(parent->seed, stream));
}

/* fnv1a64, rng.cpp:7-15. */
EKVO_EXPORT uint64_t ekvo_fnv1a64(const void* data, size_t len, uint64_t h) {
    const unsigned char* p = (const unsigned char*)data;
    for (size_t i = 0; i < len; ++i) {
        h ^= p[i];
        h *= 1099511628211ull;
    }
    return h;
}

/* Raw mt19937_64 stream (pins the engine restatement against libstdc++). */
EKVO_EXPORT void ekvo_mt64_stream(uint64_t seed, int64_t n, uint64_t* out) {
    mt64_t g;
    mt64_seed(&g, seed);
    for (int64_t i = 0; i < n; ++i) out[i] = mt64_next(&g);
}

/* generate_embeddings, transformer.cpp:308-317: row i from Rng(seed).fork(i),
 * U[-1,1) per column, so row i at width h is a prefix of row i at h' > h. */
EKVO_EXPORT void ekvo_generate_embeddings(uint64_t seed, int n, int h, double* out) {
    mt64_t root, r;
    mt64_seed(&root, seed);
    for (int i = 0; i < n; ++i) {
        mt64_fork(&root, (uint64_t)i, &r);
        for (int c = 0; c < h; ++c) out[(size_t)i * h + c] = mt64_uniform(&r, -1.0, 1.0);
    }
}

/* init_model, transformer.cpp:82-115, written into the reference's own
 * layout: wq/wk/wv[l][hd] (h x d row-major), out_proj[l] (h x h),
 * pos (max_pos x h).  gamma = 1 and bias = 0 (transformer.cpp:111-112).
 * Returns Model::checksum (transformer.cpp:117-131). */
EKVO_EXPORT uint64_t ekvo_init_model(int L, int H, int d, int max_pos, uint64_t seed,
                                     double* wq, double* wk, double* wv, double* out_proj,
                                     double* pos) {
    const int h = H * d;
    mt64_t root, r;
    mt64_seed(&root, seed);
    uint64_t ck = 14695981039346656037ull;
    double* ones = (double*)malloc(sizeof(double) * (size_t)h);
    double* zeros = (double*)calloc((size_t)h, sizeof(double));
    for (int c = 0; c < h; ++c) ones[c] = 1.0;
    const size_t hd_sz = (size_t)h * d;
    for (int l = 0; l < L; ++l) {
        for (int hd = 0; hd < H; ++hd) {
            mt64_fork(&root, ekvo_mix((uint64_t)l, (uint64_t)hd), &r);
            double* q = wq + ((size_t)l * H + hd) * hd_sz;
            double* k = wk + ((size_t)l * H + hd) * hd_sz;
            double* v = wv + ((size_t)l * H + hd) * hd_sz;
            for (size_t i = 0; i < hd_sz; ++i) q[i] = mt64_uniform(&r, -0.1, 0.1);
            for (size_t i = 0; i < hd_sz; ++i) k[i] = mt64_uniform(&r, -0.1, 0.1);
            for (size_t i = 0; i < hd_sz; ++i) v[i] = mt64_uniform(&r, -0.1, 0.1);
            ck = ekvo_fnv1a64(q, hd_sz * 8, ck);
            ck = ekvo_fnv1a64(k, hd_sz * 8, ck);
            ck = ekvo_fnv1a64(v, hd_sz * 8, ck);
        }
        mt64_fork(&root, ekvo_mix(0x70726F6Aull, (uint64_t)l), &r);
        double* o = out_proj + (size_t)l * h * h;
        for (size_t i = 0; i < (size_t)h * h; ++i) o[i] = mt64_uniform(&r, -0.1, 0.1);
        ck = ekvo_fnv1a64(o, (size_t)h * h * 8, ck);
        ck = ekvo_fnv1a64(ones, (size_t)h * 8, ck);
        ck = ekvo_fnv1a64(zeros, (size_t)h * 8, ck);
    }
    mt64_fork(&root, 0x706F73ull, &r);
    for (size_t i = 0; i < (size_t)max_pos * h; ++i) pos[i] = mt64_uniform(&r, -0.1, 0.1);
    ck = ekvo_fnv1a64(pos, (size_t)max_pos * h * 8, ck);
    free(ones);
    free(zeros);
    return ck;
}

/* ------------------------------------------------------------------------ */
/* Counter-hash synthetic generator (this build's own; the GPU generator    */
/* ekv_fill_uniform_bf16 must reproduce it bit-for-bit).                    */
/* value(i) = bf16_rn(lo + (hi-lo) * ((mix(mix(seed,stream), i) >> 11)*2^-53)) */
/* ------------------------------------------------------------------------ */

static uint16_t f32_to_bf16_rn(float f) {
    uint32_t u;
    memcpy(&u, &f, 4);
    if ((u & 0x7F800000u) == 0x7F800000u && (u & 0x007FFFFFu)) return (uint16_t)((u >> 16) | 0x40);
    uint32_t lsb = (u >> 16) & 1u;
    u += 0x7FFFu + lsb;
    return (uint16_t)(u >> 16);
}

static float bf16_to_f32(uint16_t b) {
    uint32_t u = (uint32_t)b << 16;
    float f;
    memcpy(&f, &u, 4);
    return f;
}

/* double -> bf16, single rounding RN-even (matches __double2bfloat16). */
static uint16_t f64_to_bf16_rn(double x) {
    uint64_t u;
    memcpy(&u, &x, 8);
    uint64_t sign = u >> 63;
    double ax = fabs(x);
    if (isnan(x)) return 0x7FC0;
    if (ax == 0.0) return (uint16_t)(sign << 15);
    int e;
    double m = frexp(ax, &e); /* ax = m * 2^e, m in [0.5,1) */
    /* bf16 normal: 8 significant bits.  Exponent e-1 >= -126. */
    int ulp_exp = (e - 1) - 7;
    if (ulp_exp < -133) ulp_exp = -133; /* subnormal spacing 2^-133 */
    double scaled = ldexp(ax, -ulp_exp);
    double r = nearbyint(scaled); /* default RN-even */
    double v = ldexp(r, ulp_exp);
    float fv = (float)v; /* exact: v has <= 8 significant bits */
    uint16_t b = f32_to_bf16_rn(fv);
    return (uint16_t)(b | (sign << 15));
}

EKVO_EXPORT uint16_t ekvo_f32_to_bf16(float f) { return f32_to_bf16_rn(f); }
EKVO_EXPORT uint16_t ekvo_f64_to_bf16(double x) { return f64_to_bf16_rn(x); }

EKVO_EXPORT void ekvo_fill_uniform_bf16(uint64_t seed, uint64_t stream, int64_t n, double lo,
                                        double hi, uint16_t* out) {
    const uint64_t base = ekvo_mix(seed, stream);
    for (int64_t i = 0; i < n; ++i) {
        double u = (double)(ekvo_mix(base, (uint64_t)i) >> 11) * 0x1.0p-53;
        double x = lo + (hi - lo) * u;
        out[i] = f64_to_bf16_rn(x);
    }
}

/* ------------------------------------------------------------------------ */
/* a6: PruneSpec::from_lambda head_prune.cpp:14-22; select_channels         */
/* head_prune.cpp:83-108.                                                   */
/* ------------------------------------------------------------------------ */

EKVO_EXPORT int ekvo_prune_retained(double lambda, int head_dim) {
    return (int)floor((1.0 - lambda) * head_dim + 1e-9);
}

/* stable descending order by score (std::stable_sort with a > b), then the
 * first `retained` indices sorted ascending. Insertion sort is stable. */
static void rank_scores(const double* score, int d, int retained, int* kept) {
    int* order = (int*)malloc(sizeof(int) * (size_t)d);
    for (int i = 0; i < d; ++i) order[i] = i;
    for (int i = 1; i < d; ++i) {
        int v = order[i];
        int j = i - 1;
        while (j >= 0 && score[v] > score[order[j]]) {
            order[j + 1] = order[j];
            --j;
        }
        order[j + 1] = v;
    }
    for (int i = 0; i < retained; ++i) kept[i] = order[i];
    for (int i = 1; i < retained; ++i) { /* ascending */
        int v = kept[i];
        int j = i - 1;
        while (j >= 0 && kept[j] > v) {
            kept[j + 1] = kept[j];
            --j;
        }
        kept[j + 1] = v;
    }
    free(order);
}

/* Column sums of squares accumulated row by row (head_prune.cpp:92-96). */
EKVO_EXPORT void ekvo_colsq(const double* m, int64_t rows, int d, double* out) {
    for (int c = 0; c < d; ++c) {
        double acc = 0.0;
        for (int64_t i = 0; i < rows; ++i) acc += m[i * d + c] * m[i * d + c];
        out[c] = acc;
    }
}

/* select_channels on explicit stacked Q/K rows, head_prune.cpp:83-108. */
EKVO_EXPORT void ekvo_select_channels(const double* q, int64_t q_rows, const double* k,
                                      int64_t k_rows, int d, int retained, int* kept,
                                      double* score_out) {
    double* score = (double*)malloc(sizeof(double) * (size_t)d);
    for (int c = 0; c < d; ++c) {
        double qn = 0.0, kn = 0.0;
        for (int64_t i = 0; i < q_rows; ++i) qn += q[i * d + c] * q[i * d + c];
        for (int64_t j = 0; j < k_rows; ++j) kn += k[j * d + c] * k[j * d + c];
        score[c] = sqrt(qn) * sqrt(kn);
    }
    rank_scores(score, d, retained, kept);
    if (score_out) memcpy(score_out, score, sizeof(double) * (size_t)d);
    free(score);
}

/* The same rule on precomputed column sums of squares (what the GPU returns). */
EKVO_EXPORT void ekvo_rank_channels(const double* qsq, const double* ksq, int d, int retained,
                                    int* kept) {
    double* score = (double*)malloc(sizeof(double) * (size_t)d);
    for (int c = 0; c < d; ++c) score[c] = sqrt(qsq[c]) * sqrt(ksq[c]);
    rank_scores(score, d, retained, kept);
    free(score);
}

/* ------------------------------------------------------------------------ */
/* a7: prune_cache column slice, head_prune.cpp:170-197.                    */
/* ------------------------------------------------------------------------ */
EKVO_EXPORT void ekvo_prune_rows_f64(const double* src, int64_t rows, int d_c, const int* kept,
                                     int d_e, double* dst) {
    for (int64_t i = 0; i < rows; ++i)
        for (int c = 0; c < d_e; ++c) dst[i * d_e + c] = src[i * d_c + kept[c]];
}

EKVO_EXPORT void ekvo_prune_rows_bf16(const uint16_t* src, int64_t rows, int d_c,
                                      const int* kept, int d_e, uint16_t* dst) {
    for (int64_t i = 0; i < rows; ++i)
        for (int c = 0; c < d_e; ++c) dst[i * d_e + c] = src[i * d_c + kept[c]];
}

/* ------------------------------------------------------------------------ */
/* a8: quantise / pack / dequant.  NO REFERENCE.  This   */
/* is the build's own contract, restated here in the exact fp32 operation   */
/* order of kernel K3 (paper_2505_14085_b200/csrc/k_kvcodec.cu):            */
/*   per row (token, head) and group of g gathered channels:                */
/*   amax  = max |x| (fp32, x = bf16 input)                                 */
/*   amax < 2^-120: the group is all-zero (scale 0, codes 0)                */
/*   scale = RN(amax / Q), inv = RN(Q / amax), Q = 127 (int8) / 7 (int4)    */
/*   code  = round_half_even(RN(x * inv))   (|x*inv| <= Q(1+2^-22): no clamp) */
/*   int4: two's-complement nibbles, element 2j in the low nibble           */
/*   dequant: code * scale (exact in fp64); K6 materialises bf16_rn(fp32).  */
/* Layout: codes [rows][d_e*bits/8], scales [rows][d_e/g] fp32.             */
/* ------------------------------------------------------------------------ */
EKVO_EXPORT void ekvo_kv_compress(const uint16_t* src, int64_t rows, int d_c, const int* kept,
                                  int d_e, int bits, int group, uint8_t* codes, float* scales) {
    const float Q = bits == 8 ? 127.0f : 7.0f;
    const float tiny = 0x1.0p-120f;
    const int ng = d_e / group;
    const int row_bytes = d_e * bits / 8;
    float* x = (float*)malloc(sizeof(float) * (size_t)d_e);
    for (int64_t i = 0; i < rows; ++i) {
        for (int c = 0; c < d_e; ++c) x[c] = bf16_to_f32(src[i * d_c + kept[c]]);
        uint8_t* crow = codes + i * row_bytes;
        if (bits == 4) memset(crow, 0, (size_t)row_bytes);
        for (int gi = 0; gi < ng; ++gi) {
            float amax = 0.0f;
            for (int c = gi * group; c < (gi + 1) * group; ++c) {
                float a = fabsf(x[c]);
                if (a > amax) amax = a;
            }
            const int zero = !(amax >= tiny);
            volatile float scale = zero ? 0.0f : amax / Q;
            volatile float inv = zero ? 0.0f : Q / amax;
            scales[i * ng + gi] = scale;
            for (int c = gi * group; c < (gi + 1) * group; ++c) {
                int code = 0;
                if (!zero) {
                    volatile float t = x[c] * inv;
                    code = (int)nearbyintf(t);
                }
                if (bits == 8) {
                    crow[c] = (uint8_t)(int8_t)code;
                } else {
                    uint8_t nib = (uint8_t)(code & 0xF);
                    crow[c >> 1] |= (c & 1) ? (uint8_t)(nib << 4) : nib;
                }
            }
        }
    }
    free(x);
}

static int code_at(const uint8_t* crow, int c, int bits) {
    if (bits == 8) return (int)(int8_t)crow[c];
    int nib = (crow[c >> 1] >> ((c & 1) * 4)) & 0xF;
    return nib >= 8 ? nib - 16 : nib;
}

/* dequant to bf16 (K6 contract): bf16_rn(fp32(code) * scale). */
EKVO_EXPORT void ekvo_kv_dequant_bf16(const uint8_t* codes, const float* scales, int64_t rows,
                                      int d_e, int bits, int group, uint16_t* dst) {
    const int ng = d_e / group, row_bytes = d_e * bits / 8;
    for (int64_t i = 0; i < rows; ++i)
        for (int c = 0; c < d_e; ++c) {
            volatile float v = (float)code_at(codes + i * row_bytes, c, bits) * scales[i * ng + c / group];
            dst[i * d_e + c] = f32_to_bf16_rn(v);
        }
}

/* exact dequantised value code*scale as fp64 (what decode attention uses:  */
/* the product of an <=8-bit integer and an fp32 is exact in fp64).         */
EKVO_EXPORT void ekvo_kv_dequant_f64(const uint8_t* codes, const float* scales, int64_t rows,
                                     int d_e, int bits, int group, double* dst) {
    const int ng = d_e / group, row_bytes = d_e * bits / 8;
    for (int64_t i = 0; i < rows; ++i)
        for (int c = 0; c < d_e; ++c)
            dst[i * d_e + c] =
                (double)code_at(codes + i * row_bytes, c, bits) * (double)scales[i * ng + c / group];
}

/* ------------------------------------------------------------------------ */
/* a10/a11: segment_attention_prefix cache_merge.cpp:12-38 and              */
/* merge_attention cache_merge.cpp:59-80 (Eq. 5).         */
/* ------------------------------------------------------------------------ */
EKVO_EXPORT void ekvo_segment_attention(const double* q, const double* k, const double* v,
                                        int visible, int d, int vd, double* o, double* sigma,
                                        double* shift) {
    double* logits = (double*)malloc(sizeof(double) * (size_t)(visible > 0 ? visible : 1));
    for (int j = 0; j < visible; ++j) {
        double acc = 0.0;
        for (int c = 0; c < d; ++c) acc += q[c] * k[(size_t)j * d + c];
        logits[j] = acc;
    }
    double mx = logits[0];
    for (int j = 1; j < visible; ++j) mx = logits[j] > mx ? logits[j] : mx;
    double sig = 0.0;
    for (int c = 0; c < vd; ++c) o[c] = 0.0;
    for (int j = 0; j < visible; ++j) {
        const double w = exp(logits[j] - mx);
        sig += w;
        for (int c = 0; c < vd; ++c) o[c] += w * v[(size_t)j * vd + c];
    }
    for (int c = 0; c < vd; ++c) o[c] /= sig;
    *sigma = sig;
    *shift = mx;
    free(logits);
}

/* returns 0, or -1 for the reference's "non-positive or non-finite sigma". */
EKVO_EXPORT int ekvo_merge_attention(const double* o_c, double sigma_c, double shift_c,
                                     const double* o_u, double sigma_u, double shift_u, int d,
                                     double* o, double* alpha_ctx, double* alpha_user) {
    if (!(sigma_c > 0.0) || !(sigma_u > 0.0) || !isfinite(sigma_c) || !isfinite(sigma_u))
        return -1;
    const double m = shift_c > shift_u ? shift_c : shift_u;
    const double sc = sigma_c * exp(shift_c - m);
    const double su = sigma_u * exp(shift_u - m);
    const double ac = sc / (sc + su), au = su / (sc + su);
    for (int i = 0; i < d; ++i) o[i] = ac * o_c[i] + au * o_u[i];
    if (alpha_ctx) *alpha_ctx = ac;
    if (alpha_user) *alpha_user = au;
    return 0;
}

/* ------------------------------------------------------------------------ */
/* a2/a12: the edge forward with merged attention, merged_forward           */
/* cache_merge.cpp:156-226, and collaborative_decode :230-273.              */
/*                                                                          */
/* Weights are passed in the B200 layout:             */
/*   wqkvT[l]: (3h x h), row part*h + head*d + c  ==  W_part[l][head](:, c) */
/*   woT[l]:   (h x h),  woT[j][i] == out_proj[l](i, j)                     */
/* The arithmetic order is the reference's: every dot product runs over the */
/* input features left to right exactly as matmul (matrix.cpp:19-36).       */
/*                                                                          */
/* ctx_k/ctx_v: per layer [H][S][d] (already dequantised / gathered), or    */
/* NULL when S == 0.  Option user_kv_bf16 rounds the appended user K/V rows */
/* to bf16 (the B200 user-cache storage format); 0 = reference semantics.   */
/* ------------------------------------------------------------------------ */
typedef struct {
    int L, H, d, max_pos;
    const double* wqkvT; /* [L][3h][h] */
    const double* woT;   /* [L][h][h]  */
    const double* gamma; /* [h] (layer 0) */
    const double* bias;  /* [h] (layer 0) */
    const double* pos;   /* [max_pos][h] */
} ekvo_model_t;

typedef struct {
    int L, H, d, cap;   /* cap = max user rows */
    int len;            /* rows held */
    double* k;          /* [L][H][cap][d] */
    double* v;
} ekvo_ucache_t;

static void merged_forward(const ekvo_model_t* m, int S, const double* const* ctx_k,
                           const double* const* ctx_v, ekvo_ucache_t* uc, const double* emb,
                           int n, int user_kv_bf16, double* out_rows /* [n][h] */) {
    const int H = m->H, d = m->d, h = H * d;
    const int old = uc->len;
    double* x = (double*)malloc(sizeof(double) * (size_t)n * h);
    double* concat = (double*)malloc(sizeof(double) * (size_t)n * h);
    double* qkv = (double*)malloc(sizeof(double) * (size_t)n * 3 * h);
    double* o_u = (double*)malloc(sizeof(double) * (size_t)d);
    double* o_c = (double*)malloc(sizeof(double) * (size_t)d);
    double* merged = (double*)malloc(sizeof(double) * (size_t)d);
    for (int i = 0; i < n; ++i) {
        const double* p = m->pos + (size_t)(S + old + i) * h;
        for (int c = 0; c < h; ++c)
            x[(size_t)i * h + c] = m->gamma[c] * (emb[(size_t)i * h + c] + p[c]) + m->bias[c];
    }
    for (int l = 0; l < m->L; ++l) {
        const double* W = m->wqkvT + (size_t)l * 3 * h * h;
        for (int i = 0; i < n; ++i)
            for (int r = 0; r < 3 * h; ++r) {
                double acc = 0.0;
                const double* wr = W + (size_t)r * h;
                const double* xr = x + (size_t)i * h;
                for (int kk = 0; kk < h; ++kk) acc += xr[kk] * wr[kk];
                qkv[((size_t)i * 3 * h) + r] = acc;
            }
        for (int hd = 0; hd < H; ++hd) {
            double* uk = uc->k + (((size_t)l * H + hd) * uc->cap) * d;
            double* uv = uc->v + (((size_t)l * H + hd) * uc->cap) * d;
            for (int i = 0; i < n; ++i)
                for (int c = 0; c < d; ++c) {
                    double kv = qkv[(size_t)i * 3 * h + h + hd * d + c];
                    double vv = qkv[(size_t)i * 3 * h + 2 * h + hd * d + c];
                    if (user_kv_bf16) {
                        kv = (double)bf16_to_f32(f32_to_bf16_rn((float)kv));
                        vv = (double)bf16_to_f32(f32_to_bf16_rn((float)vv));
                    }
                    uk[(size_t)(old + i) * d + c] = kv;
                    uv[(size_t)(old + i) * d + c] = vv;
                }
            for (int i = 0; i < n; ++i) {
                const double* q = qkv + (size_t)i * 3 * h + hd * d;
                double su, hu;
                ekvo_segment_attention(q, uk, uv, old + i + 1, d, d, o_u, &su, &hu);
                const double* res = o_u;
                if (S > 0) {
                    double sc, hc;
                    const double* ck = ctx_k[l] + (size_t)hd * S * d;
                    const double* cv = ctx_v[l] + (size_t)hd * S * d;
                    ekvo_segment_attention(q, ck, cv, S, d, d, o_c, &sc, &hc);
                    ekvo_merge_attention(o_c, sc, hc, o_u, su, hu, d, merged, NULL, NULL);
                    res = merged;
                }
                for (int c = 0; c < d; ++c) concat[(size_t)i * h + hd * d + c] = res[c];
            }
        }
        const double* Wo = m->woT + (size_t)l * h * h;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < h; ++j) {
                double acc = 0.0;
                const double* wr = Wo + (size_t)j * h;
                const double* cr = concat + (size_t)i * h;
                for (int kk = 0; kk < h; ++kk) acc += cr[kk] * wr[kk];
                x[(size_t)i * h + j] = acc;
            }
    }
    uc->len += n;
    memcpy(out_rows, x, sizeof(double) * (size_t)n * h);
    free(x);
    free(concat);
    free(qkv);
    free(o_u);
    free(o_c);
    free(merged);
}

/* collaborative_decode, cache_merge.cpp:230-273.  teacher (optional,
 * [steps][h]) replaces the fed-back input row of step t with teacher[t]
 * (teacher forcing for per-step parity).  Returns 0 or negative on bad args. */
EKVO_EXPORT int ekvo_collaborative_decode(int L, int H, int d, int max_pos, const double* wqkvT,
                                          const double* woT, const double* gamma,
                                          const double* bias, const double* pos, int S,
                                          const double* ctx_k_all, const double* ctx_v_all,
                                          const double* user_emb, int U, int steps,
                                          const double* teacher, int user_kv_bf16,
                                          double* prefill_out, double* step_out) {
    if (steps < 1) return -1;
    const int h = H * d;
    if (S + U + steps > max_pos) return -2; /* "position overflow" */
    ekvo_model_t m = {L, H, d, max_pos, wqkvT, woT, gamma, bias, pos};
    ekvo_ucache_t uc;
    uc.L = L;
    uc.H = H;
    uc.d = d;
    uc.cap = U + steps;
    uc.len = 0;
    uc.k = (double*)calloc((size_t)L * H * uc.cap * d, sizeof(double));
    uc.v = (double*)calloc((size_t)L * H * uc.cap * d, sizeof(double));
    const double** ck = (const double**)malloc(sizeof(double*) * (size_t)L);
    const double** cv = (const double**)malloc(sizeof(double*) * (size_t)L);
    for (int l = 0; l < L; ++l) {
        ck[l] = S > 0 ? ctx_k_all + (size_t)l * H * S * d : NULL;
        cv[l] = S > 0 ? ctx_v_all + (size_t)l * H * S * d : NULL;
    }
    double* next = (double*)calloc((size_t)h, sizeof(double));
    if (U > 0) {
        merged_forward(&m, S, ck, cv, &uc, user_emb, U, user_kv_bf16, prefill_out);
        memcpy(next, prefill_out + (size_t)(U - 1) * h, sizeof(double) * (size_t)h);
    }
    for (int t = 0; t < steps; ++t) {
        if (teacher) memcpy(next, teacher + (size_t)t * h, sizeof(double) * (size_t)h);
        merged_forward(&m, S, ck, cv, &uc, next, 1, user_kv_bf16, step_out + (size_t)t * h);
        memcpy(next, step_out + (size_t)t * h, sizeof(double) * (size_t)h);
    }
    free(uc.k);
    free(uc.v);
    free(ck);
    free(cv);
    free(next);
    return 0;
}

/* forward_rows over an empty cache == prefill (transformer.cpp:175-251) in the
 * same B200 weight layout: returns per-layer outputs [L][n][h] and the K/V
 * cache [L][H][n][d].  Used to make the inputs of the alignment stage (the
 * cloud hidden states X_lc and the cloud K/V) in small end-to-end tests. */
/* kv_bf16 = 1 rounds the cached K/V rows to bf16 before they are attended (and
 * returned): the B200 prefill keeps its KV cache in bf16 (ekv_prefill). */
EKVO_EXPORT void ekvo_prefill_ex(int L, int H, int d, int max_pos, const double* wqkvT,
                                 const double* woT, const double* gamma, const double* bias,
                                 const double* pos, const double* emb, int n, int kv_bf16,
                                 double* layer_out, double* k_out, double* v_out) {
    (void)max_pos;
    const int h = H * d;
    double* x = (double*)malloc(sizeof(double) * (size_t)n * h);
    double* concat = (double*)malloc(sizeof(double) * (size_t)n * h);
    double* qkv = (double*)malloc(sizeof(double) * (size_t)n * 3 * h);
    double* o = (double*)malloc(sizeof(double) * (size_t)d);
    double* kb = (double*)malloc(sizeof(double) * (size_t)n * d);
    double* vb = (double*)malloc(sizeof(double) * (size_t)n * d);
    for (int i = 0; i < n; ++i)
        for (int c = 0; c < h; ++c)
            x[(size_t)i * h + c] = gamma[c] * (emb[(size_t)i * h + c] + pos[(size_t)i * h + c]) + bias[c];
    for (int l = 0; l < L; ++l) {
        const double* W = wqkvT + (size_t)l * 3 * h * h;
        for (int i = 0; i < n; ++i)
            for (int r = 0; r < 3 * h; ++r) {
                double acc = 0.0;
                for (int kk = 0; kk < h; ++kk) acc += x[(size_t)i * h + kk] * W[(size_t)r * h + kk];
                qkv[(size_t)i * 3 * h + r] = acc;
            }
        for (int hd = 0; hd < H; ++hd) {
            for (int i = 0; i < n; ++i)
                for (int c = 0; c < d; ++c) {
                    double kv = qkv[(size_t)i * 3 * h + h + hd * d + c];
                    double vv = qkv[(size_t)i * 3 * h + 2 * h + hd * d + c];
                    if (kv_bf16) {
                        kv = (double)bf16_to_f32(f32_to_bf16_rn((float)kv));
                        vv = (double)bf16_to_f32(f32_to_bf16_rn((float)vv));
                    }
                    kb[(size_t)i * d + c] = kv;
                    vb[(size_t)i * d + c] = vv;
                }
            if (k_out) memcpy(k_out + (((size_t)l * H + hd) * n) * d, kb, sizeof(double) * (size_t)n * d);
            if (v_out) memcpy(v_out + (((size_t)l * H + hd) * n) * d, vb, sizeof(double) * (size_t)n * d);
            for (int i = 0; i < n; ++i) {
                double s, sh;
                ekvo_segment_attention(qkv + (size_t)i * 3 * h + hd * d, kb, vb, i + 1, d, d, o, &s, &sh);
                for (int c = 0; c < d; ++c) concat[(size_t)i * h + hd * d + c] = o[c];
            }
        }
        const double* Wo = woT + (size_t)l * h * h;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < h; ++j) {
                double acc = 0.0;
                for (int kk = 0; kk < h; ++kk) acc += concat[(size_t)i * h + kk] * Wo[(size_t)j * h + kk];
                x[(size_t)i * h + j] = acc;
            }
        memcpy(layer_out + (size_t)l * n * h, x, sizeof(double) * (size_t)n * h);
    }
    free(x);
    free(concat);
    free(qkv);
    free(o);
    free(kb);
    free(vb);
}

EKVO_EXPORT void ekvo_prefill(int L, int H, int d, int max_pos, const double* wqkvT,
                              const double* woT, const double* gamma, const double* bias,
                              const double* pos, const double* emb, int n, double* layer_out,
                              double* k_out, double* v_out) {
    ekvo_prefill_ex(L, H, d, max_pos, wqkvT, woT, gamma, bias, pos, emb, n, 0, layer_out, k_out,
                    v_out);
}

/* Q = X * W_Q for one cloud layer in the B200 layout (wqT [H*d_c][h_c]) and
 * its per-column sums of squares over all rows: the alignment projection of
 * build_deep_kv (sim.cpp:240-253, project_qkv transformer.cpp:133-152) fused
 * with the column-norm loop of select_channels (head_prune.cpp:92-97).
 * colsq_out[n] for n in [0, H*d_c); the stacked-over-heads channel sums are
 * sum_h colsq_out[h*d_c + c]. */
EKVO_EXPORT void ekvo_align_qnorm(const double* X, int S, int h_c, const double* wqT, int n_cols,
                                  double* colsq_out) {
    for (int n = 0; n < n_cols; ++n) colsq_out[n] = 0.0;
    for (int i = 0; i < S; ++i)
        for (int n = 0; n < n_cols; ++n) {
            double acc = 0.0;
            for (int kk = 0; kk < h_c; ++kk) acc += X[(size_t)i * h_c + kk] * wqT[(size_t)n * h_c + kk];
            colsq_out[n] += acc * acc;
        }
}

/* ------------------------------------------------------------------------ */
/* a3: layer matching, layer_match.cpp:25-228 (+ pearson_corr matrix.cpp:64-93) */
/* ------------------------------------------------------------------------ */
static void rsm_(const double* o, int n, int c, double* s) { /* layer_match.cpp:25-41 */
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double acc = 0.0;
            for (int k = 0; k < c; ++k) acc += o[(size_t)i * c + k] * o[(size_t)j * c + k];
            s[(size_t)i * n + j] = acc;
        }
}

static void double_center_(const double* s, int n, double* out) { /* :46-69 */
    double* rm = (double*)calloc((size_t)n, sizeof(double));
    double* cm = (double*)calloc((size_t)n, sizeof(double));
    double total = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            rm[i] += s[(size_t)i * n + j];
            cm[j] += s[(size_t)i * n + j];
            total += s[(size_t)i * n + j];
        }
    for (int i = 0; i < n; ++i) {
        rm[i] /= (double)n;
        cm[i] /= (double)n;
    }
    total /= (double)((size_t)n * n);
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) out[(size_t)i * n + j] = s[(size_t)i * n + j] - rm[i] - cm[j] + total;
    free(rm);
    free(cm);
}

static double hsic_(const double* se, const double* sc, int n, double* scratch) { /* :119-138 */
    double_center_(se, n, scratch);
    double tr = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) tr += scratch[(size_t)i * n + j] * sc[(size_t)j * n + i];
    return tr / ((double)(n - 1) * (double)(n - 1));
}

/* returns 0 ok, -1 "degenerate representation" (layer_match.cpp:150) */
EKVO_EXPORT int ekvo_cka(const double* oe, int ce, const double* oc, int cc, int n, double* out) {
    double* se = (double*)malloc(sizeof(double) * (size_t)n * n);
    double* sc = (double*)malloc(sizeof(double) * (size_t)n * n);
    double* tmp = (double*)malloc(sizeof(double) * (size_t)n * n);
    rsm_(oe, n, ce, se);
    rsm_(oc, n, cc, sc);
    const double self_e = hsic_(se, se, n, tmp);
    const double self_c = hsic_(sc, sc, n, tmp);
    int rc = 0;
    if (self_e < 1e-15 || self_c < 1e-15) rc = -1;
    else *out = hsic_(se, sc, n, tmp) / sqrt(self_e * self_c);
    free(se);
    free(sc);
    free(tmp);
    return rc;
}

/* pearson_corr matrix.cpp:64-93; returns -1 on "zero variance" */
static int pearson_(const double* x, const double* y, size_t n, double* out) {
    double mx = 0.0, my = 0.0;
    for (size_t i = 0; i < n; ++i) {
        mx += x[i];
        my += y[i];
    }
    mx /= (double)n;
    my /= (double)n;
    double sxy = 0.0, sxx = 0.0, syy = 0.0;
    for (size_t i = 0; i < n; ++i) {
        const double dx = x[i] - mx, dy = y[i] - my;
        sxy += dx * dy;
        sxx += dx * dx;
        syy += dy * dy;
    }
    if (sxx == 0.0 || syy == 0.0) return -1;
    double r = sxy / sqrt(sxx * syy);
    if (r < -1.0) r = -1.0;
    if (r > 1.0) r = 1.0;
    *out = r;
    return 0;
}

/* cosine_matrix + strict_lower_flat, layer_match.cpp:71-103; returns -(row+2)
 * for "zero-norm row N" */
static int cos_lower_(const double* o, int n, int c, double* flat) {
    double* norms = (double*)malloc(sizeof(double) * (size_t)n);
    for (int i = 0; i < n; ++i) {
        double acc = 0.0;
        for (int k = 0; k < c; ++k) acc += o[(size_t)i * c + k] * o[(size_t)i * c + k];
        norms[i] = sqrt(acc);
        if (norms[i] == 0.0) {
            free(norms);
            return -(i + 2);
        }
    }
    size_t idx = 0;
    for (int i = 1; i < n; ++i)
        for (int j = 0; j < i; ++j) {
            double acc = 0.0;
            for (int k = 0; k < c; ++k) acc += o[(size_t)i * c + k] * o[(size_t)j * c + k];
            flat[idx++] = acc / (norms[i] * norms[j]);
        }
    free(norms);
    return 0;
}

/* rsa, layer_match.cpp:155-164.  0 ok; -1 zero variance; -(row+2) zero-norm row */
EKVO_EXPORT int ekvo_rsa(const double* oe, int ce, const double* oc, int cc, int n, double* out) {
    const size_t m = (size_t)n * (n - 1) / 2;
    double* fe = (double*)malloc(sizeof(double) * m);
    double* fc = (double*)malloc(sizeof(double) * m);
    int rc = cos_lower_(oe, n, ce, fe);
    if (rc == 0) rc = cos_lower_(oc, n, cc, fc);
    if (rc == 0) rc = pearson_(fe, fc, m, out);
    free(fe);
    free(fc);
    return rc;
}

/* scale_normalize, layer_match.cpp:105-115 (Frobenius norm -> sqrt(N)). */
static void scale_normalize_(const double* o, int n, int c, double* out) {
    double f = 0.0;
    for (size_t i = 0; i < (size_t)n * c; ++i) f += o[i] * o[i];
    f = sqrt(f);
    if (f == 0.0) {
        memcpy(out, o, sizeof(double) * (size_t)n * c);
        return;
    }
    const double target = sqrt((double)n);
    for (size_t i = 0; i < (size_t)n * c; ++i) out[i] = o[i] * (target / f);
}

/* match_layers, layer_match.cpp:166-228.  edge_outs [me][n][ce], cloud_outs
 * [nc][n][cc]; best[le] = cloud layer or -1.  Returns 0 or the first error. */
EKVO_EXPORT int ekvo_match_layers(const double* edge_outs, int me, int ce, const double* cloud_outs,
                                  int nc, int cc, int n, double theta_cka, double theta_rsa,
                                  double* cka_out, double* rsa_out, int* best) {
    double* en = (double*)malloc(sizeof(double) * (size_t)me * n * ce);
    double* cn = (double*)malloc(sizeof(double) * (size_t)nc * n * cc);
    for (int l = 0; l < me; ++l)
        scale_normalize_(edge_outs + (size_t)l * n * ce, n, ce, en + (size_t)l * n * ce);
    for (int l = 0; l < nc; ++l)
        scale_normalize_(cloud_outs + (size_t)l * n * cc, n, cc, cn + (size_t)l * n * cc);
    int rc = 0;
    for (int le = 0; le < me && rc == 0; ++le) {
        int best_lc = -1;
        double best_cka = 0.0;
        for (int lc = 0; lc < nc; ++lc) {
            double c = 0.0, r = 0.0;
            rc = ekvo_cka(en + (size_t)le * n * ce, ce, cn + (size_t)lc * n * cc, cc, n, &c);
            if (rc) break;
            rc = ekvo_rsa(en + (size_t)le * n * ce, ce, cn + (size_t)lc * n * cc, cc, n, &r);
            if (rc) break;
            cka_out[(size_t)le * nc + lc] = c;
            rsa_out[(size_t)le * nc + lc] = r;
            if (c >= theta_cka && r >= theta_rsa) {
                if (best_lc < 0 || c > best_cka) {
                    best_lc = lc;
                    best_cka = c;
                }
            }
        }
        best[le] = best_lc;
    }
    free(en);
    free(cn);
    return rc;
}

/* ------------------------------------------------------------------------ */
/* a13: cache_source cost_model.cpp:64-71; pipeline_schedule :73-100.       */
/* ------------------------------------------------------------------------ */
/* 0 local, 1 peer, 2 cloud; -1 layer out of range */
EKVO_EXPORT int ekvo_cache_source(int layer, double cost_local, double cost_peer, int boundary,
                                  int m) {
    if (layer < 1 || layer > m) return -1;
    if (layer > boundary) return 2;
    return cost_local <= cost_peer ? 0 : 1;
}

/* t_pip[l] = max(t_comm[l], t_comp[l-1]), t_comp[-1] = 0; totals. */
EKVO_EXPORT int ekvo_pipeline_schedule(const double* t_comm, const double* t_comp, int n,
                                       double* t_pip, double* sequential_total,
                                       double* pipelined_total) {
    if (n < 1) return -1;
    for (int l = 0; l < n; ++l)
        if (t_comm[l] < 0.0 || t_comp[l] < 0.0) return -2;
    double prev = 0.0, pip = 0.0, seq = 0.0;
    for (int l = 0; l < n; ++l) {
        t_pip[l] = t_comm[l] > prev ? t_comm[l] : prev;
        pip += t_pip[l];
        prev = t_comp[l];
    }
    for (int l = 0; l < n; ++l) seq += t_comm[l] + t_comp[l];
    *pipelined_total = pip + t_comp[n - 1];
    *sequential_total = seq;
    return 0;
}
