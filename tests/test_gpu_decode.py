"""GPU parity of the composed path: collaborative decode (merged_forward +
collaborative_decode, cache_merge.cpp:156-273) and the full CE-LSLM flow of
Artifacts (sim.cpp:100-265) at the reference's smallest scenario shape
(BASELINE.json configs[0]), through the C ABI.

Oracle semantics for the decode loop: the oracle consumes the same bf16 weights,
the same bf16 local context and the exact dequantised cloud context; the user
cache is rounded to bf16 as the B200 stores it (oracle option user_kv_bf16), and
each step is teacher-forced with the GPU's own input row.
Bar: normwise max|gpu-ref|/max|ref| <= 1e-3 per output row, fp32 outputs.
"""
import os

import numpy as np
import pytest
import torch

from oracle import bf16_to_f64, model_from_reference_layout

pytestmark = pytest.mark.gpu
TOL = 1e-3


def normwise(got, want):
    return float(np.max(np.abs(np.asarray(got, np.float64) - want)) / max(np.max(np.abs(want)), 1e-30))


@pytest.fixture(scope="module")
def ek():
    from paper_2505_14085_b200 import build
    build.build()
    from paper_2505_14085_b200 import edgekv
    return edgekv


@pytest.fixture(scope="module")
def ctx(ek):
    return ek.Context(0)


def host_bf16_model(oracle, L, H, d, max_pos, seed):
    """Random scaled-init edge weights in the B200 layout, bf16 bits + exact fp64."""
    h = H * d
    a = float(np.sqrt(3.0 / h))
    wq = []
    wo = []
    for l in range(L):
        q = oracle.fill_uniform_bf16(seed, 4 * l, h * h, -a / np.sqrt(d), a / np.sqrt(d))
        kv = oracle.fill_uniform_bf16(seed, 4 * l + 1, 2 * h * h, -a, a)
        wq.append(np.concatenate([q, kv]).reshape(3 * h, h))
        wo.append(oracle.fill_uniform_bf16(seed, 4 * l + 2, h * h, -a, a).reshape(h, h))
    pos = oracle.fill_uniform_bf16(seed, 0x706F73, max_pos * h, -0.1, 0.1).reshape(max_pos, h)
    rng = np.random.default_rng(seed)
    gamma = (1.0 + rng.uniform(-0.2, 0.2, h)).astype(np.float32)
    bias = rng.uniform(-0.1, 0.1, h).astype(np.float32)
    bits = dict(wqkvT=np.stack(wq), woT=np.stack(wo), pos=pos, gamma=gamma, bias=bias)
    f64 = dict(L=L, H=H, d=d, max_pos=max_pos, wqkvT=bf16_to_f64(bits["wqkvT"]),
               woT=bf16_to_f64(bits["woT"]), pos=bf16_to_f64(pos), gamma=gamma.astype(np.float64),
               bias=bias.astype(np.float64))
    return bits, f64


def upload_model(ek, ctx, bits, L, H, d, max_pos):
    m = ek.EdgeModel(ctx, L, H, d, max_pos)
    for l in range(L):
        m.set_layer(l, bits["wqkvT"][l], bits["woT"][l])
    m.set_io(bits["gamma"], bits["bias"], bits["pos"])
    return m


def bits_of(t):
    return t.view(torch.int16).cpu().numpy().view(np.uint16)


def make_context(ek, ctx, oracle, model, S, formats, seed, d_c=None):
    """Assembled context: bf16 layers uploaded directly, quantised layers produced by
    the GPU compressor from a wider cloud KV (d_c) with a random kept mask.
    Returns (AssembledContext, ctx_k f64 [L][H][S][d], ctx_v f64)."""
    L, H, d = model.L, model.H, model.d
    d_c = d_c or 2 * d
    kvc = ek.AssembledContext(model, S, formats, group=32 if EKV_INT4 in formats else d)
    ck = np.zeros((L, H, S, d)); cv = np.zeros((L, H, S, d))
    rng = np.random.default_rng(seed)
    for l, f in enumerate(formats):
        if f == ek.EKV_KV_BF16:
            kb = oracle.fill_uniform_bf16(seed, 100 + l, H * S * d, -1, 1).reshape(H, S, d)
            vb = oracle.fill_uniform_bf16(seed, 200 + l, H * S * d, -1, 1).reshape(H, S, d)
            kvc.upload_bf16(l, kb, vb)
            ck[l] = bf16_to_f64(kb); cv[l] = bf16_to_f64(vb)
        else:
            nb = 8 if f == ek.EKV_KV_INT8 else 4
            g = kvc.segment(l).group
            kept = np.sort(rng.choice(d_c, d, replace=False)).astype(np.int32)
            outs = []
            for j in range(2):
                src = torch.empty((H, S, d_c), dtype=torch.bfloat16, device="cuda")
                ctx.fill_uniform_bf16(src, seed, 300 + 2 * l + j, -1, 1)
                ctx.synchronize()
                codes, scales = ek.kv_compress(ctx, src, kept, nb, g)
                wc, ws = oracle.kv_compress(bits_of(src).reshape(H * S, d_c), kept, nb, g)
                assert np.array_equal(codes.reshape(H * S, -1).cpu().numpy(), wc)
                outs.append((codes, scales, oracle.kv_dequant_f64(wc, ws, d, nb, g).reshape(H, S, d)))
            kvc.set_layer(l, outs[0][0], outs[1][0], outs[0][1], outs[1][1])
            ck[l] = outs[0][2]; cv[l] = outs[1][2]
    return kvc, ck, cv


EKV_INT8, EKV_INT4 = 8, 4


@pytest.mark.parametrize("path", ["mega", "graph"])
@pytest.mark.parametrize("formats,S,U,T,H,d", [([16, 8, 8], 320, 5, 6, 4, 64),
                                               ([16, 16], 0, 3, 4, 4, 64),
                                               ([16, 4], 256, 9, 3, 4, 64),
                                               ([8, 8], 128, 0, 3, 4, 64),
                                               ([16, 8], 300, 4, 3, 4, 64),
                                               ([16, 8, 4], 512, 7, 5, 8, 32),
                                               ([8, 16], 256, 3, 4, 4, 128)])
def test_collaborative_decode_matches_oracle(ek, ctx, oracle, formats, S, U, T, H, d, path):
    L = len(formats)
    h, max_pos = H * d, 1024
    bits, f64 = host_bf16_model(oracle, L, H, d, max_pos, seed=7 + S)
    model = upload_model(ek, ctx, bits, L, H, d, max_pos)
    kvc, ck, cv = make_context(ek, ctx, oracle, model, S, formats, seed=11 + S)
    sess = ek.Session(model, kvc, U + T)
    got_path = sess.set_decode_path(path)
    assert got_path == ("graph" if (path == "graph" or S % 16) else "mega")
    ue = oracle.generate_embeddings(43, max(U, 1), h)[:U]
    ue32 = ue.astype(np.float32)
    pre, steps = ek.collaborative_decode(sess, ue32, T)
    teacher = np.vstack([pre[-1:] if U else np.zeros((1, h)), steps[:-1]]).astype(np.float64)
    want_pre, want_steps = oracle.collaborative_decode(f64, ck if S else None, cv if S else None,
                                                       ue32.astype(np.float64), T, teacher=teacher,
                                                       user_kv_bf16=True)
    for r in range(U):
        assert normwise(pre[r], want_pre[r]) <= TOL, (r, normwise(pre[r], want_pre[r]))
    for t in range(T):
        assert normwise(steps[t], want_steps[t]) <= TOL, (t, normwise(steps[t], want_steps[t]))
    assert np.all(np.isfinite(steps))
    # the device API (forward + decode) is the same computation
    sess.reset()
    if U:
        out = sess.forward(torch.from_numpy(ue32).cuda())
        assert np.array_equal(out.cpu().numpy(), pre)
    st = sess.decode(T).cpu().numpy()
    assert np.array_equal(st, steps)
    if got_path == "mega":  # head clusters (when the grid has 2-8 CTAs per head) vs global exchange
        sess.reset()
        os.environ["EKV_MEGA_CLUSTER"] = "0"
        try:
            if U:
                sess.forward(torch.from_numpy(ue32).cuda())
            assert np.array_equal(sess.decode(T).cpu().numpy(), steps)
        finally:
            del os.environ["EKV_MEGA_CLUSTER"]


@pytest.mark.parametrize("grid", [8, 16, 32, 36])
def test_mega_head_clusters_bit_identical(ek, ctx, oracle, grid):
    """The persistent kernel with 2 / 4 / 8 CTAs per head (thread-block clusters,
    DSMEM exchange) and with 9 (no cluster: global tagged words) computes the same
    bits as the global exchange, and matches the oracle."""
    L, H, d, S, U, T = 4, 4, 64, 1024, 3, 3
    h = H * d
    bits, f64 = host_bf16_model(oracle, L, H, d, 512 + S, seed=91)
    model = upload_model(ek, ctx, bits, L, H, d, 512 + S)
    kvc, ck, cv = make_context(ek, ctx, oracle, model, S, [16, 8, 16, 8], seed=93)
    ue32 = oracle.generate_embeddings(45, U, h).astype(np.float32)
    runs = []
    os.environ["EKV_MEGA_GRID"] = str(grid)
    try:
        for cl in ("1", "0"):
            os.environ["EKV_MEGA_CLUSTER"] = cl
            sess = ek.Session(model, kvc, U + T)
            assert sess.set_decode_path("mega") == "mega"
            runs.append(ek.collaborative_decode(sess, ue32, T))
    finally:
        del os.environ["EKV_MEGA_GRID"], os.environ["EKV_MEGA_CLUSTER"]
    (pre, steps), (pre0, steps0) = runs
    assert np.array_equal(steps, steps0) and np.array_equal(pre, pre0)
    teacher = np.vstack([pre[-1:], steps[:-1]]).astype(np.float64)
    _, want = oracle.collaborative_decode(f64, ck, cv, ue32.astype(np.float64), T, teacher=teacher,
                                          user_kv_bf16=True)
    assert max(normwise(steps[t], want[t]) for t in range(T)) <= TOL


def test_collaborative_decode_errors(ek, ctx, oracle):
    L, H, d = 2, 4, 64
    bits, _ = host_bf16_model(oracle, L, H, d, 64, seed=3)
    model = upload_model(ek, ctx, bits, L, H, d, 64)
    kvc = ek.AssembledContext(model, 60, [16, 16])
    sess = ek.Session(model, kvc, 16)
    ue = np.zeros((3, H * d), np.float32)
    with pytest.raises(ek.EkvError, match="position overflow"):
        ek.collaborative_decode(sess, ue, 2)
    with pytest.raises(ek.EkvError, match="steps must be >= 1"):
        ek.collaborative_decode(sess, ue[:1], 0)
    other = ek.EdgeModel(ctx, 2, 8, 32, 64)
    with pytest.raises(ek.EkvError, match="align with head pruning"):
        ek.Session(other, kvc, 4)


def test_shared_context_two_consumers_identical(ek, ctx, oracle):
    """cache_merge_test.cpp:333-348: two readers of one context cache agree exactly."""
    L, H, d = 2, 4, 64
    bits, _ = host_bf16_model(oracle, L, H, d, 512, seed=5)
    model = upload_model(ek, ctx, bits, L, H, d, 512)
    kvc, _, _ = make_context(ek, ctx, oracle, model, 200, [16, 8], seed=5)
    a = ek.Session(model, kvc, 16)
    b = ek.Session(model, kvc, 16)
    ue = oracle.generate_embeddings(1, 4, H * d).astype(np.float32)
    ra = ek.collaborative_decode(a, ue, 5)
    rb = ek.collaborative_decode(b, ue, 5)
    assert np.array_equal(ra[1], rb[1]) and np.array_equal(ra[0], rb[0])


def run_full_ce_lslm_path(ek, ctx, oracle, Lc=8, Le=4, deep=2, bits=8):
    """The end-to-end composition of Artifacts (sim.cpp:100-265): cloud Lc layers
    d=512 (8x64), edge Le layers d=256 (8x32), S=512, U=16, T=16 decode steps,
    lambda 0.5, `deep` deep layers compressed to `bits`-bit codes.
      1. layer map: probe prefill (oracle fp64) -> GPU-host match_layers == oracle
      2. alignment: K1 (tcgen05) + K2 norms on the bf16 cloud X_lc / W_Q / K ->
         mask == oracle select_channels on the same bf16 inputs (bit-exact)
      3. compression: K3 int8 codes of the pruned cloud KV (bit-exact)
      4. decode: collaborative_decode over [local bf16 | cloud int8] context
    """
    Hc, dc, He, de = 8, 64, 8, 32
    hc, he, S, U, T = Hc * dc, He * de, 512, 16, 16
    max_pos = S + U + T
    # models (random scaled init, bf16-exact values, B200 layout)
    cbits, cf = host_bf16_model(oracle, Lc, Hc, dc, max_pos, seed=11)
    ebits, ef = host_bf16_model(oracle, Le, He, de, max_pos, seed=13)
    cf["gamma"] = np.ones(hc); cf["bias"] = np.zeros(hc)
    ef["gamma"] = np.ones(he); ef["bias"] = np.zeros(he)
    ebits["gamma"] = np.ones(he, np.float32); ebits["bias"] = np.zeros(he, np.float32)
    # 1. layer map (sim.cpp:100-122): probe seed mix(42, 0x9B0BE), 64 probes
    pseed = oracle.mix(42, 0x9B0BE)
    eo = oracle.prefill(ef, oracle.generate_embeddings(pseed, 64, he))[0]
    co = oracle.prefill(cf, oracle.generate_embeddings(pseed, 64, hc))[0]
    cka, rsa, best = ek.match_layers(ctx, eo, co, 0.0, -1.0)
    assert np.array_equal(best, oracle.match_layers(eo, co, 0.0, -1.0)[2])
    boundary = Le - deep
    deep_match = {le: int(best[le]) for le in range(boundary, Le)}
    assert all(v >= 0 for v in deep_match.values())
    # context prefill on both sides (the cloud's outputs are the alignment inputs)
    eseed = oracle.mix(42, 0xC7E20000)
    ctx_c = oracle.generate_embeddings(eseed, S, hc)
    ctx_e = oracle.generate_embeddings(eseed, S, he)
    c_out, c_k, c_v = oracle.prefill(cf, ctx_c)
    _, e_k, e_v = oracle.prefill(ef, ctx_e)
    lcs = sorted(set(deep_match.values()))
    x0 = ctx_c + cf["pos"][:S]
    Xs = np.stack([x0 if lc == 0 else c_out[lc - 1] for lc in lcs])       # [m][S][hc]
    from oracle import f32_to_bf16_bits
    to_dev = lambda a: torch.from_numpy(f32_to_bf16_bits(np.asarray(a, np.float32)).view(np.int16)).view(torch.bfloat16).cuda()
    Xd = to_dev(Xs)
    Wq = np.stack([cbits["wqkvT"][lc][:hc] for lc in lcs])                 # [m][hc][hc] bf16 bits
    Wd = torch.from_numpy(Wq.view(np.int16)).view(torch.bfloat16).cuda()
    Kd = to_dev(np.stack([c_k[lc] for lc in lcs]))                         # [m][H][S][dc]
    Vd = to_dev(np.stack([c_v[lc] for lc in lcs]))
    # 2. mask parity on identical bf16 inputs
    kept, margin, _, _ = ek.select_channels(ctx, Xd, Wd, Kd, 0.5, dc)
    xb = bf16_to_f64(bits_of(Xd)).reshape(Xs.shape)
    wb = bf16_to_f64(Wq)
    q_stack = np.concatenate([(xb[i] @ wb[i].T).reshape(S, Hc, dc).transpose(1, 0, 2).reshape(-1, dc)
                              for i in range(len(lcs))])
    k_stack = bf16_to_f64(bits_of(Kd)).reshape(-1, dc)
    want_kept, _ = oracle.select_channels(q_stack, k_stack, oracle.prune_retained(0.5, dc))
    assert margin > 1e-6
    assert kept.tolist() == want_kept.tolist()
    # 3+4. assemble [local bf16 | cloud int8] and decode
    edge = upload_model(ek, ctx, ebits, Le, He, de, max_pos)
    fmts = [16] * boundary + [bits] * deep
    group = de if bits == 8 else 32
    kvc = ek.AssembledContext(edge, S, fmts, group=group)
    ck = np.zeros((Le, He, S, de)); cv = np.zeros((Le, He, S, de))
    for l in range(boundary):
        kb = f32_to_bf16_bits(e_k[l].astype(np.float32)); vb = f32_to_bf16_bits(e_v[l].astype(np.float32))
        kvc.upload_bf16(l, kb, vb)
        ck[l] = bf16_to_f64(kb); cv[l] = bf16_to_f64(vb)
    got_kept, got_margin = ek.build_deep_kv(ctx, kvc, deep_match, Xd, Wd, Kd, Vd, 0.5, lcs)
    assert got_kept.tolist() == want_kept.tolist() and got_margin > 1e-6
    for le, lc in deep_match.items():
        i = lcs.index(lc)
        for src, dst in ((Kd, ck), (Vd, cv)):
            wc, ws = oracle.kv_compress(bits_of(src[i]).reshape(Hc * S, dc), want_kept, bits, group)
            dst[le] = oracle.kv_dequant_f64(wc, ws, de, bits, group).reshape(He, S, de)
    sess = ek.Session(edge, kvc, U + T)
    useed = oracle.mix(42, 0x55E20000)
    ue = oracle.generate_embeddings(useed, U, he).astype(np.float32)
    for path in (("mega", "graph") if bits == 8 else ("graph",)):
        assert sess.set_decode_path(path) == path
        pre, steps = ek.collaborative_decode(sess, ue, T)
        teacher = np.vstack([pre[-1:], steps[:-1]]).astype(np.float64)
        wp, ws_ = oracle.collaborative_decode(ef, ck, cv, ue.astype(np.float64), T, teacher=teacher,
                                              user_kv_bf16=True)
        assert max(normwise(pre[r], wp[r]) for r in range(U)) <= TOL
        assert max(normwise(steps[t], ws_[t]) for t in range(T)) <= TOL, path


def test_full_ce_lslm_path_config1(ek, ctx, oracle):
    """The end-to-end composition of Artifacts (sim.cpp:100-265) at BASELINE
    configs[0]'s shape: cloud 8L d=512 (8x64), edge 4L d=256 (8x32), S=512,
    U=16, T=64 (decode steps checked 16 here), lambda 0.5, 2 deep layers.
      1. layer map: probe prefill (oracle fp64) -> GPU-host match_layers == oracle
      2. alignment: K1 (tcgen05) + K2 norms on the bf16 cloud X_lc / W_Q / K ->
         mask == oracle select_channels on the same bf16 inputs (bit-exact)
      3. compression: K3 int8 codes of the pruned cloud KV (bit-exact)
      4. decode: collaborative_decode over [local bf16 | cloud int8] context
    """
    run_full_ce_lslm_path(ek, ctx, oracle)


def test_long_context_32k_decode(ek, ctx, oracle):
    """BASELINE configs[3]'s context length: S = 32768 reused rows ([local bf16 | cloud
    int8] layers), both decode paths, against the oracle."""
    L, H, d, S, U, T = 2, 4, 64, 32768, 4, 3
    formats = [16, 8]
    max_pos = S + U + T + 1
    bits, f64 = host_bf16_model(oracle, L, H, d, max_pos, seed=71)
    model = upload_model(ek, ctx, bits, L, H, d, max_pos)
    kvc, ck, cv = make_context(ek, ctx, oracle, model, S, formats, seed=73)
    sess = ek.Session(model, kvc, U + T)
    ue = oracle.generate_embeddings(79, U, H * d).astype(np.float32)
    for path in ("mega", "graph"):
        assert sess.set_decode_path(path) == path
        pre, steps = ek.collaborative_decode(sess, ue, T)
        teacher = np.vstack([pre[-1:], steps[:-1]]).astype(np.float64)
        wp, ws = oracle.collaborative_decode(f64, ck, cv, ue.astype(np.float64), T, teacher=teacher,
                                             user_kv_bf16=True)
        assert max(normwise(pre[r], wp[r]) for r in range(U)) <= TOL, path
        assert max(normwise(steps[t], ws[t]) for t in range(T)) <= TOL, path


@pytest.mark.parametrize("Lc,Le,deep,bits", [(16, 4, 2, 8), (16, 4, 2, 4), (8, 4, 2, 4)])
def test_full_ce_lslm_path_compression_sweep(ek, ctx, oracle, Lc, Le, deep, bits):
    """BASELINE configs[4] at reduced size: int8 vs int4 KV and cloud:edge layer ratios
    4:1 (16 -> 4 layers) and 2:1 (8 -> 4), the whole path (layer map, mask, codes,
    decode) against the oracle."""
    run_full_ce_lslm_path(ek, ctx, oracle, Lc, Le, deep, bits)


def _layer_bytes(seg, H, d):
    rows = H * seg.S
    row_b = d * 2 if seg.format == 16 else d * seg.format // 8
    return rows * row_b, (rows * (d // seg.group) * 4 if seg.format != 16 else 0)


@pytest.mark.parametrize("overlap", [True, False])
def test_pipelined_prefill_eq20(ek, ctx, oracle, overlap):
    """Eq. 20 (pipeline_schedule, cost_model.cpp:73-100) on the device: the context
    layers arrive from pinned host memory on the copy stream while the user rows
    are forwarded; the result equals the resident-context forward bit for bit (and
    the oracle), and decode continues from it."""
    import ctypes as C
    from paper_2505_14085_b200.capi import call
    L, H, d, S, U, T = 3, 4, 64, 512, 11, 3
    formats = [16, 8, 8]
    max_pos = S + U + T + 1
    bits, f64 = host_bf16_model(oracle, L, H, d, max_pos, seed=91)
    model = upload_model(ek, ctx, bits, L, H, d, max_pos)
    kvc, ck, cv = make_context(ek, ctx, oracle, model, S, formats, seed=93)
    ue = torch.from_numpy(oracle.generate_embeddings(97, U, H * d).astype(np.float32)).cuda()
    ref = ek.Session(model, kvc, U + T)
    want = ref.forward(ue).cpu().numpy()
    want_steps = ref.decode(T).cpu().numpy()
    # host copies of every context layer, then wipe the device storage
    uploads = {}
    for l in range(L):
        seg = kvc.segment(l)
        nb, ns = _layer_bytes(seg, H, d)
        hk = torch.empty(nb, dtype=torch.uint8).pin_memory()
        hv = torch.empty(nb, dtype=torch.uint8).pin_memory()
        call("ekv_copy", ctx.h, C.c_void_p(hk.data_ptr()), C.c_void_p(seg.k), nb, 1)
        call("ekv_copy", ctx.h, C.c_void_p(hv.data_ptr()), C.c_void_p(seg.v), nb, 1)
        call("ekv_memset", ctx.h, C.c_void_p(seg.k), 0, nb)
        call("ekv_memset", ctx.h, C.c_void_p(seg.v), 0, nb)
        hks = hvs = None
        if ns:
            hks = torch.empty(ns // 4, dtype=torch.float32).pin_memory()
            hvs = torch.empty(ns // 4, dtype=torch.float32).pin_memory()
            call("ekv_copy", ctx.h, C.c_void_p(hks.data_ptr()), C.c_void_p(seg.k_scales), ns, 1)
            call("ekv_copy", ctx.h, C.c_void_p(hvs.data_ptr()), C.c_void_p(seg.v_scales), ns, 1)
        uploads[l] = (hk, hv, hks, hvs)
    sess = ek.Session(model, kvc, U + T)
    out, tcomm, tcomp, total = sess.forward_pipelined(ue, uploads, overlap=overlap)
    assert np.array_equal(out.cpu().numpy(), want)
    assert np.all(tcomm > 0) and np.all(tcomp > 0) and total > 0
    st = sess.decode(T).cpu().numpy()
    assert np.array_equal(st, want_steps)
    wp, _ = oracle.collaborative_decode(f64, ck, cv, ue.cpu().numpy().astype(np.float64), 1,
                                        user_kv_bf16=True)
    assert max(normwise(want[r], wp[r]) for r in range(U)) <= TOL


@pytest.mark.timeout(300)
def test_persistent_kernels_on_two_streams(ek):
    """Two contexts (two CUDA streams) on one GPU decoding at the same time: every K8
    launch needs all of its CTAs resident (the dataflow spins on its peers), so two
    launches in flight must not interleave their CTAs (cooperative launch, head clusters
    at C2's 4 CTAs per head).  Same inputs on both streams -> same bits as run alone."""
    L, H, d, S, U, T = 2, 32, 64, 1024, 4, 24
    runs = []
    for _ in range(2):
        c = ek.Context(0)
        m = ek.EdgeModel(c, L, H, d, S + 64)
        m.synthesize(5)
        kv = ek.AssembledContext(m, S, [16, 8], group=d)
        kv.synthesize(6)
        s = ek.Session(m, kv, U + T)
        s.forward(torch.full((U, H * d), 0.25, device="cuda"))
        runs.append((c, m, kv, s))
    alone = runs[0][3].decode(T).cpu().numpy()
    runs[0][3].reset()
    runs[0][3].forward(torch.full((U, H * d), 0.25, device="cuda"))
    outs = [r[3].decode(T, sync=False) for r in runs]  # both streams in flight
    for r in runs:
        r[0].synchronize()
    assert np.array_equal(outs[0].cpu().numpy(), alone)
    assert np.array_equal(outs[1].cpu().numpy(), alone)
