"""GPU parity: every kernel on the hot path against the CPU oracle (oracle/ekv_oracle.c,
pinned to the reference in test_oracle_pinned.py), called through the C ABI.

Bars:
* integer / byte / index work (generator, gather, codes, scales, channel masks,
  layer maps): bit-exact;
* floating point: normwise  max|gpu - ref| / max|ref|  <= 1e-3 with fp32 outputs,
  the oracle fed the identical bf16 / dequantised inputs.
"""
import ctypes

import numpy as np
import pytest
import torch

from oracle import bf16_to_f64, f32_to_bf16_bits

pytestmark = pytest.mark.gpu

TOL = 1e-3


def normwise(got, want):
    got = np.asarray(got, dtype=np.float64)
    want = np.asarray(want, dtype=np.float64)
    return float(np.max(np.abs(got - want)) / max(np.max(np.abs(want)), 1e-30))


@pytest.fixture(scope="module")
def ek():
    from paper_2505_14085_b200 import build
    build.build()
    from paper_2505_14085_b200 import edgekv
    return edgekv


@pytest.fixture(scope="module")
def ctx(ek):
    return ek.Context(0)


def rand_bf16(ctx, shape, seed, stream, lo=-1.0, hi=1.0):
    t = torch.empty(shape, dtype=torch.bfloat16, device="cuda")
    ctx.fill_uniform_bf16(t, seed, stream, lo, hi)
    ctx.synchronize()
    return t


def bits(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


# ----------------------------------------------------------------- generator
def test_counter_hash_generator_bit_exact(ctx, oracle):
    for n, seed, stream, lo, hi in [(1, 1, 0, -1, 1), (100003, 42, 7, -0.05, 0.05),
                                    (4096, 2**63 + 9, 2**40, -3.0, 0.5)]:
        t = rand_bf16(ctx, (n,), seed, stream, lo, hi)
        assert np.array_equal(bits(t), oracle.fill_uniform_bf16(seed, stream, n, lo, hi))


# ------------------------------------------------------ stage 2: gather/compress
SHAPES = [  # (rows, d_c, d_e, bits, group)  fast paths + generic path + edge cases
    (4096, 128, 64, 8, 64), (4096, 128, 64, 4, 32), (1023, 64, 32, 8, 32), (1023, 64, 32, 4, 32),
    (777, 128, 128, 8, 128), (64, 128, 128, 4, 32), (33, 64, 64, 8, 16), (5, 6, 4, 8, 4),
    (7, 6, 4, 4, 2), (1, 128, 64, 8, 64), (300, 256, 128, 8, 128), (300, 80, 64, 8, 64),
    (129, 128, 64, 8, 16), (129, 128, 64, 4, 64),
]


@pytest.mark.parametrize("rows,d_c,d_e,nbits,group", SHAPES)
def test_kv_compress_codes_and_scales_bit_exact(ek, ctx, oracle, rows, d_c, d_e, nbits, group):
    rng = np.random.default_rng(rows * 7 + d_c)
    src = rand_bf16(ctx, (rows, d_c), rows, d_c, -4.0, 4.0)
    src[rows // 2] = 0  # an all-zero row: scale 0, codes 0
    if rows > 3:
        src[1, :] = 1e-30  # denormal-range row
    kept = np.sort(rng.choice(d_c, d_e, replace=False)).astype(np.int32)
    codes, scales = ek.kv_compress(ctx, src, kept, nbits, group)
    want_c, want_s = oracle.kv_compress(bits(src), kept, nbits, group)
    assert np.array_equal(codes.cpu().numpy(), want_c)
    assert np.array_equal(scales.cpu().numpy().view(np.uint32), want_s.view(np.uint32))
    # K6 dequant, bit-exact
    deq = ek.kv_dequant(ctx, codes, scales, d_e, nbits, group)
    assert np.array_equal(bits(deq), oracle.kv_dequant_bf16(want_c, want_s, d_e, nbits, group))
    # gather == prune_cache slice
    g = ek.prune_cache(ctx, src, kept)
    assert np.array_equal(bits(g), oracle.prune_rows_bf16(bits(src), kept))


def test_quantisation_fidelity_bounds(ek, ctx, oracle):
    """|x - code*scale| <= scale/2 per element (round-to-nearest of the fp32 quotient,
    so up to one quotient ulp, Q*2^-23*scale, beyond), reported separately from
    parity (tolerance definition)."""
    src = rand_bf16(ctx, (2048, 128), 5, 5)
    kept = np.arange(0, 128, 2, dtype=np.int32)
    for nbits, group in [(8, 64), (4, 32)]:
        codes, scales = ek.kv_compress(ctx, src, kept, nbits, group)
        deq = oracle.kv_dequant_f64(codes.cpu().numpy(), scales.cpu().numpy(), 64, nbits, group)
        x = bf16_to_f64(bits(src))[:, kept]
        s = np.repeat(scales.cpu().numpy().astype(np.float64), group, axis=1)
        assert np.all(np.abs(x - deq) <= s * (0.5 + 128 * 2.0**-23))


def test_kv_colnorm_matches_fp64(ek, ctx):
    for rows, d in [(65536, 128), (1000, 64), (17, 6)]:
        K = rand_bf16(ctx, (rows, d), rows, d)
        got = ek.kv_colnorm(ctx, K).cpu().numpy()
        x = bf16_to_f64(bits(K))
        want = (x * x).sum(axis=0)
        assert np.max(np.abs(got - want) / want) < 1e-5


# ---------------------------------------------------------- stage 1: K1 + mask
@pytest.mark.parametrize("m,S,hc,n", [(1, 128, 64, 256), (2, 256, 512, 512), (1, 512, 512, 512),
                                      (3, 384, 1024, 768)])
def test_align_qnorm_tcgen05_matches_fp64(ek, ctx, m, S, hc, n):
    X = rand_bf16(ctx, (m, S, hc), 11, S)
    W = rand_bf16(ctx, (m, n, hc), 12, n, -0.1, 0.1)
    got = ek.align_qnorm(ctx, X, W).cpu().numpy()
    x = bf16_to_f64(bits(X)).reshape(m, S, hc)
    w = bf16_to_f64(bits(W)).reshape(m, n, hc)
    want = np.stack([((x[i] @ w[i].T) ** 2).sum(axis=0) for i in range(m)])
    assert np.max(np.abs(got - want) / want) < 1e-4


def test_channel_mask_bit_exact_vs_reference_rule(ek, ctx, oracle):
    """select_channels over stacked Q/K of 2 matched layers x 8 heads: the GPU mask
    equals the oracle's select_channels on the identical bf16 X, W_Q and K."""
    m, S, H, dc = 2, 256, 8, 64
    hc = H * dc
    rng = np.random.default_rng(3)
    # heterogeneous channel importance (the regime channel pruning targets)
    X = rand_bf16(ctx, (m, S, hc), 21, 0)
    W = rand_bf16(ctx, (m, H * dc, hc), 22, 0, -0.05, 0.05)
    Wn = bf16_to_f64(bits(W)).reshape(m, H * dc, hc)
    colscale = np.exp(rng.uniform(-1.0, 1.0, dc))
    Wn = Wn * np.tile(colscale, H)[None, :, None]
    W = torch.from_numpy(f32_to_bf16_bits(Wn.astype(np.float32)).view(np.int16)).view(torch.bfloat16).cuda()
    Kc = rand_bf16(ctx, (m, H, S, dc), 23, 0)
    kept, margin, q_c, k_c = ek.select_channels(ctx, X, W, Kc, 0.5, dc)
    x = bf16_to_f64(bits(X)).reshape(m, S, hc)
    w = bf16_to_f64(bits(W)).reshape(m, H * dc, hc)
    q_stack = np.concatenate([(x[i] @ w[i].T).reshape(S, H, dc).transpose(1, 0, 2).reshape(-1, dc)
                              for i in range(m)])
    k_stack = bf16_to_f64(bits(Kc)).reshape(-1, dc)
    want, _ = oracle.select_channels(q_stack, k_stack, oracle.prune_retained(0.5, dc))
    assert margin > 1e-6, "near-tie at the cut: mask parity not decidable at fp32"
    assert kept.tolist() == want.tolist()


# ------------------------------------------------------- stage 3: attention
def _segments(ek, ctx, oracle, fmt, H, S, d, seed):
    """A context segment in the given format and its exact fp64 dequantised values."""
    k = rand_bf16(ctx, (H, S, d), seed, 1)
    v = rand_bf16(ctx, (H, S, d), seed, 2)
    if fmt == ek.EKV_KV_BF16 or S == 0:
        return (ek.Segment(ek.EKV_KV_BF16, S, k, v, group=d),
                bf16_to_f64(bits(k)).reshape(H, S, d), bf16_to_f64(bits(v)).reshape(H, S, d))
    nb = 8 if fmt == ek.EKV_KV_INT8 else 4
    g = d if nb == 8 else 32
    ident = np.arange(d, dtype=np.int32)
    kc, ks = ek.kv_compress(ctx, k, ident, nb, g)
    vc, vs = ek.kv_compress(ctx, v, ident, nb, g)
    kd = oracle.kv_dequant_f64(kc.reshape(H * S, -1).cpu().numpy(), ks.reshape(H * S, -1).cpu().numpy(), d, nb, g)
    vd = oracle.kv_dequant_f64(vc.reshape(H * S, -1).cpu().numpy(), vs.reshape(H * S, -1).cpu().numpy(), d, nb, g)
    return (ek.Segment(fmt, S, kc, vc, ks, vs, group=g), kd.reshape(H, S, d), vd.reshape(H, S, d))


@pytest.mark.parametrize("fmt", [16, 8, 4])
@pytest.mark.parametrize("d", [32, 64, 128])
@pytest.mark.parametrize("R,S,base", [(1, 2048, 15), (3, 300, 0), (1, 0, 4), (2, 129, 40)])
def test_decode_attention_vs_segment_merge(ek, ctx, oracle, fmt, d, R, S, base):
    H, cap = 4, 64
    seg, kd, vd = _segments(ek, ctx, oracle, fmt, H, S, d, seed=S + d)
    q = torch.randn((R, H, d), device="cuda", dtype=torch.float32) * 0.5
    uk = rand_bf16(ctx, (H, cap, d), 91, d)
    uv = rand_bf16(ctx, (H, cap, d), 92, d)
    out, lse = ek.decode_attention(ctx, q, seg, uk, uv, base, want_lse=True)
    qn = q.double().cpu().numpy()
    ukn = bf16_to_f64(bits(uk)).reshape(H, cap, d)
    uvn = bf16_to_f64(bits(uv)).reshape(H, cap, d)
    want = np.zeros((R, H, d))
    want_lse = np.zeros((R, H))
    for r in range(R):
        for h in range(H):
            u = oracle.segment_attention(qn[r, h], ukn[h], uvn[h], visible=base + r + 1)
            if S == 0:  # degenerate merge (cache_merge.cpp:209-210)
                want[r, h] = u[0]
                want_lse[r, h] = np.log(u[1]) + u[2]
            else:
                c = oracle.segment_attention(qn[r, h], kd[h], vd[h])
                want[r, h] = oracle.merge_attention(c, u)[0]
                want_lse[r, h] = np.logaddexp(np.log(c[1]) + c[2], np.log(u[1]) + u[2])
    assert normwise(out.cpu().numpy(), want) <= TOL
    assert np.max(np.abs(lse.cpu().numpy() - want_lse)) < 1e-3


def test_decode_attention_rejects_bad_arguments(ek, ctx):
    H, d = 2, 64
    seg = ek.Segment(ek.EKV_KV_BF16, 0, group=d)
    uk = torch.zeros((H, 4, d), dtype=torch.bfloat16, device="cuda")
    q = torch.zeros((1, H, d), device="cuda")
    with pytest.raises(ek.EkvError, match="empty segment"):
        ek.decode_attention(ctx, q, seg, uk, uk, 4)
    with pytest.raises(ek.EkvError, match="head_dim"):
        ek.decode_attention(ctx, torch.zeros((1, H, 48), device="cuda"), seg,
                            torch.zeros((H, 4, 48), dtype=torch.bfloat16, device="cuda"),
                            torch.zeros((H, 4, 48), dtype=torch.bfloat16, device="cuda"), 0)


@pytest.mark.parametrize("n_jobs,rows,nbits,group", [
    (22, 32 * 2048, 8, 64),   # the bench's C2 launch: K and V of 11 deep layers, 32 heads x 2048 tokens
    (16, 32 * 2048, 4, 32),   # configs[4] int4
    (5, 1003, 8, 64),         # ragged: rows not a multiple of the 32-row tile
    (3, 17, 4, 32),           # fewer rows than one tile
])
def test_kv_compress_batched_launch_bit_exact(ek, ctx, oracle, n_jobs, rows, nbits, group):
    """K3's multi-job persistent launch (`ekv_kv_compress_batched`, the launch bench.py times)
    at full C2 size: every job's codes and scales equal the oracle's."""
    d_c, d_e = 128, 64
    srcs = [rand_bf16(ctx, (rows, d_c), 900 + j, rows, -2.0, 2.0) for j in range(n_jobs)]
    srcs[0][rows // 3] = 0
    rng = np.random.default_rng(n_jobs * rows)
    kept = np.sort(rng.choice(d_c, d_e, replace=False)).astype(np.int32)
    kept_t = torch.from_numpy(kept).cuda()
    cw = d_e * nbits // 8
    codes = [torch.empty((rows, cw), dtype=torch.uint8, device="cuda") for _ in range(n_jobs)]
    scales = [torch.empty((rows, d_e // group), dtype=torch.float32, device="cuda") for _ in range(n_jobs)]
    P = ctypes.c_void_p * n_jobs
    ek.compress_batched(ctx, n_jobs, P(*[s.data_ptr() for s in srcs]), rows, d_c, kept_t, d_e, nbits,
                        group, P(*[c.data_ptr() for c in codes]), P(*[s.data_ptr() for s in scales]))
    ctx.synchronize()
    for j in range(n_jobs):
        want_c, want_s = oracle.kv_compress(bits(srcs[j]), kept, nbits, group)
        assert np.array_equal(codes[j].cpu().numpy(), want_c), j
        assert np.array_equal(scales[j].cpu().numpy().view(np.uint32), want_s.view(np.uint32)), j
