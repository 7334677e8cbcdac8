// K7: the layer map on the device (match_layers, layer_match.cpp:166-228).
//
// Inputs are the probe-prefill outputs of every edge and cloud layer (fp64,
// [layers][n][c], n = N_probe).  Everything is fp64 with the reference's exact
// operation order (no FMA contraction, sequential sums in the reference's loop
// order), so the CKA / RSA matrices are bit-identical to the reference run on
// the same outputs and the argmax (ties -> smaller cloud layer) cannot differ:
//   scale_normalize (:105-115)  one thread per layer: sequential Frobenius sum
//   rsm / gram (:25-41)         one thread per (layer, i, j): sequential k-sum of
//                               the normalised products, k-chunks staged in smem
//   double_center + self HSIC (:46-69, :119-138), cosine lower triangle
//   (:71-103)                   one block per layer
//   HSIC(e, c) and Pearson of the cosine triangles (:140-164, matrix.cpp:64-93)
//                               one thread per (edge layer, cloud layer) pair
// The work is tiny (tens of microseconds at the C2 shapes); it runs once per
// model pair, off the decode path.
#include "ekv_common.cuh"
#include "ekv_kernels.h"

namespace ekv {

namespace k7 {

constexpr int KC = 32;  // k-chunk of the Gram tile

// scale = sqrt(n) / ||O||_F (0 -> 1: the reference leaves a zero matrix as is)
__global__ void frob_scale_kernel(const double* __restrict__ outs, int n, int c, double* __restrict__ scale) {
    if (threadIdx.x != 0) return;
    const double* o = outs + (size_t)blockIdx.x * n * c;
    double f = 0.0;
    for (size_t i = 0; i < (size_t)n * c; ++i) f = __dadd_rn(f, __dmul_rn(o[i], o[i]));
    f = sqrt(f);
    scale[blockIdx.x] = f == 0.0 ? 0.0 : __ddiv_rn(sqrt((double)n), f);  // 0: "not scaled"
}

// S[l][i][j] = sum_k (o_ik * s)(o_jk * s), k ascending.  Block (l, i0): rows
// i0..i0+3, all j; 4 x n threads.
__global__ void gram_kernel(const double* __restrict__ outs, int n, int c, const double* __restrict__ scale,
                            double* __restrict__ gram) {
    extern __shared__ double tile[];  // [n][KC + 1]
    const int l = blockIdx.y;
    const double s = scale[l];
    const double* o = outs + (size_t)l * n * c;
    const int j = threadIdx.x % n, ii = threadIdx.x / n, i = blockIdx.x * 4 + ii;
    double acc = 0.0;
    for (int k0 = 0; k0 < c; k0 += KC) {
        const int kn = min(KC, c - k0);
        for (int t = threadIdx.x; t < n * KC; t += blockDim.x) {
            const int r = t / KC, kk = t % KC;
            if (kk < kn) {
                const double v = o[(size_t)r * c + k0 + kk];
                tile[r * (KC + 1) + kk] = s == 0.0 ? v : __dmul_rn(v, s);
            }
        }
        __syncthreads();
        if (i < n)
            for (int kk = 0; kk < kn; ++kk)
                acc = __dadd_rn(acc, __dmul_rn(tile[i * (KC + 1) + kk], tile[j * (KC + 1) + kk]));
        __syncthreads();
    }
    if (i < n) gram[((size_t)l * n + i) * n + j] = acc;
}

// Per layer: double-centred Gram (the reference's loop order), self HSIC, and the
// strict lower triangle of the cosine matrix.  One block per layer.
__global__ void layer_stats_kernel(const double* __restrict__ gram, int n, double* __restrict__ centred,
                                   double* __restrict__ self_hsic, double* __restrict__ cosflat,
                                   int* __restrict__ zero_row) {
    extern __shared__ double sh[];  // rm[n], cm[n], norms[n], total
    double* rm = sh;
    double* cm = sh + n;
    double* nr = sh + 2 * n;
    const int l = blockIdx.x;
    const double* s = gram + (size_t)l * n * n;
    // row sums (j ascending), column sums (i ascending), total (row-major), norms
    for (int t = threadIdx.x; t < n; t += blockDim.x) {
        double r = 0.0, cc = 0.0;
        for (int q = 0; q < n; ++q) {
            r = __dadd_rn(r, s[(size_t)t * n + q]);
            cc = __dadd_rn(cc, s[(size_t)q * n + t]);
        }
        rm[t] = __ddiv_rn(r, (double)n);
        cm[t] = __ddiv_rn(cc, (double)n);
        nr[t] = sqrt(s[(size_t)t * n + t]);
    }
    if (threadIdx.x == 0) {
        double tot = 0.0;
        for (int q = 0; q < n * n; ++q) tot = __dadd_rn(tot, s[q]);
        sh[3 * n] = __ddiv_rn(tot, (double)n * (double)n);
        int z = -1;
        for (int q = 0; q < n; ++q)
            if (z < 0 && s[(size_t)q * n + q] == 0.0) z = q;
        zero_row[l] = z;
    }
    __syncthreads();
    const double tot = sh[3 * n];
    double* cen = centred + (size_t)l * n * n;
    for (int t = threadIdx.x; t < n * n; t += blockDim.x) {
        const int i = t / n, j = t % n;
        cen[t] = __dadd_rn(__dsub_rn(__dsub_rn(s[t], rm[i]), cm[j]), tot);
    }
    const size_t m = (size_t)n * (n - 1) / 2;
    for (size_t t = threadIdx.x; t < m; t += blockDim.x) {
        // t -> (i, j), i > j, row-major over the strict lower triangle
        int i = (int)((1.0 + sqrt(1.0 + 8.0 * (double)t)) / 2.0);
        while ((size_t)i * (i - 1) / 2 > t) --i;
        while ((size_t)(i + 1) * i / 2 <= t) ++i;
        const int j = (int)(t - (size_t)i * (i - 1) / 2);
        cosflat[(size_t)l * m + t] = __ddiv_rn(s[(size_t)i * n + j], __dmul_rn(nr[i], nr[j]));
    }
    __syncthreads();
    if (threadIdx.x == 0) {
        double tr = 0.0;
        for (int i = 0; i < n; ++i)
            for (int j = 0; j < n; ++j) tr = __dadd_rn(tr, __dmul_rn(cen[(size_t)i * n + j], s[(size_t)j * n + i]));
        self_hsic[l] = __ddiv_rn(tr, __dmul_rn((double)(n - 1), (double)(n - 1)));
    }
}

// One thread per (edge layer, cloud layer): HSIC(e, c) and the Pearson
// correlation of the two cosine triangles.  Layers [0, me) are edge, [me, me+nc)
// cloud in the per-layer buffers.
__global__ void pair_kernel(const double* __restrict__ gram, const double* __restrict__ centred,
                            const double* __restrict__ cosflat, int me, int nc, int n,
                            double* __restrict__ hsic, double* __restrict__ corr, int* __restrict__ zero_var) {
    const int p = blockIdx.x * blockDim.x + threadIdx.x;
    if (p >= me * nc) return;
    const int le = p / nc, lc = me + p % nc;
    const double* ce = centred + (size_t)le * n * n;
    const double* sc = gram + (size_t)lc * n * n;
    double tr = 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) tr = __dadd_rn(tr, __dmul_rn(ce[(size_t)i * n + j], sc[(size_t)j * n + i]));
    hsic[p] = __ddiv_rn(tr, __dmul_rn((double)(n - 1), (double)(n - 1)));
    const size_t m = (size_t)n * (n - 1) / 2;
    const double* x = cosflat + (size_t)le * m;
    const double* y = cosflat + (size_t)lc * m;
    double mx = 0.0, my = 0.0;
    for (size_t i = 0; i < m; ++i) {
        mx = __dadd_rn(mx, x[i]);
        my = __dadd_rn(my, y[i]);
    }
    mx = __ddiv_rn(mx, (double)m);
    my = __ddiv_rn(my, (double)m);
    double sxy = 0.0, sxx = 0.0, syy = 0.0;
    for (size_t i = 0; i < m; ++i) {
        const double dx = __dsub_rn(x[i], mx), dy = __dsub_rn(y[i], my);
        sxy = __dadd_rn(sxy, __dmul_rn(dx, dy));
        sxx = __dadd_rn(sxx, __dmul_rn(dx, dx));
        syy = __dadd_rn(syy, __dmul_rn(dy, dy));
    }
    zero_var[p] = (sxx == 0.0 || syy == 0.0);
    double r = (sxx == 0.0 || syy == 0.0) ? 0.0 : __ddiv_rn(sxy, sqrt(__dmul_rn(sxx, syy)));
    corr[p] = r < -1.0 ? -1.0 : (r > 1.0 ? 1.0 : r);
}

}  // namespace k7

// outs: [me + nc] layers packed as edge [me][n][ce] then cloud [nc][n][cc] (two
// buffers); work buffers are allocated by the caller (see ekv_capi.cu).
void launch_layer_match(const double* edge_outs, int me, int ce, const double* cloud_outs, int nc, int cc,
                        int n, double* scale, double* gram, double* centred, double* self_hsic,
                        double* cosflat, int* zero_row, double* hsic, double* corr, int* zero_var,
                        cudaStream_t st) {
    using namespace k7;
    const int L = me + nc;
    frob_scale_kernel<<<me, 32, 0, st>>>(edge_outs, n, ce, scale);
    frob_scale_kernel<<<nc, 32, 0, st>>>(cloud_outs, n, cc, scale + me);
    const size_t tile = sizeof(double) * (size_t)n * (KC + 1);
    gram_kernel<<<dim3((n + 3) / 4, me), 4 * n, tile, st>>>(edge_outs, n, ce, scale, gram);
    gram_kernel<<<dim3((n + 3) / 4, nc), 4 * n, tile, st>>>(cloud_outs, n, cc, scale + me,
                                                            gram + (size_t)me * n * n);
    layer_stats_kernel<<<L, 256, sizeof(double) * (3 * n + 1), st>>>(gram, n, centred, self_hsic, cosflat,
                                                                       zero_row);
    pair_kernel<<<(me * nc + 127) / 128, 128, 0, st>>>(gram, centred, cosflat, me, nc, n, hsic, corr, zero_var);
    EKV_CUDA(cudaGetLastError());
    count_launches(6);
}

}  // namespace ekv
