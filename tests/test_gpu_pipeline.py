"""GPU parity of the whole-operation stage 1+2 entry points (ekv_pipeline.cu):

* ekv_prefill        prefill / forward_rows (transformer.cpp:175-251): per-layer
                     outputs, x0 and the KV cache vs the oracle's prefill (KV rows
                     rounded to bf16 as the device stores them);
* ekv_match_layers   match_layers from host buffers on K7 (layer_match.cpp:166-228);
* ekv_deep_match     Artifacts::deep_match (sim.cpp:100-122): probe prefill of both
                     models on the device + K7, its map and its error;
* ekv_build_deep_kv  Artifacts::build_deep_kv (sim.cpp:217-265): mask vs the
                     oracle's select_channels, codes bit-exact;
* ekv_prompt_context Artifacts::prompt + build_deep_kv + assembled_context on the
                     device at BASELINE configs[0]'s shape, then collaborative
                     decode over the result vs the oracle.
Bars: normwise max|gpu-ref|/max|ref| <= 1e-3 per row for fp32 outputs; bf16-stored
KV rows within that bar plus one bf16 ulp of the oracle's bf16-rounded rows; masks, maps
and codes exact.
"""
import numpy as np
import pytest
import torch

from oracle import bf16_to_f64, f32_to_bf16_bits, model_from_reference_layout
from test_gpu_decode import TOL, bits_of, host_bf16_model, normwise, upload_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ek():
    from paper_2505_14085_b200 import build
    build.build()
    from paper_2505_14085_b200 import edgekv
    return edgekv


@pytest.fixture(scope="module")
def ctx(ek):
    return ek.Context(0)


def within_bf16_ulp(got, want):
    """bf16-stored rows vs the oracle's bf16-rounded rows: the rows are projections of
    hidden states that carry the fp32 path's error (normwise <= 1e-3, the output bar), then
    round to bf16, where the two roundings may land one bf16 ulp (<= 2^-7 relative) apart."""
    tol = 2.0 ** -7 * np.abs(want) + TOL * np.max(np.abs(want))
    return bool(np.all(np.abs(got - want) <= tol))


def dev32(a):
    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.float32)).cuda()


def test_prefill_matches_oracle(ek, ctx, oracle):
    L, H, d, n = 3, 4, 64, 37
    h = H * d
    bits, f64 = host_bf16_model(oracle, L, H, d, 64, seed=3)
    model = upload_model(ek, ctx, bits, L, H, d, 64)
    emb = oracle.generate_embeddings(5, n, h).astype(np.float32)
    lo, x0, k, v = ek.prefill(model, dev32(emb), want_x0=True, want_kv=True)
    wlo, wk, wv = oracle.prefill(f64, emb.astype(np.float64), kv_bf16=True)
    lo = lo.cpu().numpy()
    for l in range(L):
        for r in range(n):
            assert normwise(lo[l, r], wlo[l, r]) <= TOL, (l, r)
    want_x0 = f64["gamma"] * (emb.astype(np.float64) + f64["pos"][:n]) + f64["bias"]
    assert normwise(x0.cpu().numpy(), want_x0) <= 1e-6
    kb = bf16_to_f64(bits_of(k)).reshape(L, H, n, d)
    vb = bf16_to_f64(bits_of(v)).reshape(L, H, n, d)
    for l in range(L):
        assert within_bf16_ulp(kb[l], wk[l]) and within_bf16_ulp(vb[l], wv[l]), l
    with pytest.raises(ek.EkvError, match="position overflow"):
        ek.prefill(model, dev32(np.zeros((65, h))))


def test_match_layers_host_buffers_on_k7(ek, ctx, oracle):
    """The heterogeneous pair of layer_match_test.cpp:286-329 (3L 2x6 vs 5L 4x6)."""
    e = model_from_reference_layout(oracle.init_model(3, 2, 6, 64, 41), 3, 2, 6, 64)
    c = model_from_reference_layout(oracle.init_model(5, 4, 6, 64, 43), 5, 4, 6, 64)
    eo = oracle.prefill(e, oracle.generate_embeddings(9, 16, 12))[0]
    co = oracle.prefill(c, oracle.generate_embeddings(9, 16, 24))[0]
    a = ek.match_layers(ctx, eo, co, 0.5, 0.3)
    b = oracle.match_layers(eo, co, 0.5, 0.3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


def c1_models(ek, ctx, oracle, max_pos):
    """BASELINE configs[0]: cloud 8L 8x64 (h=512), edge 4L 8x32 (h=256)."""
    cbits, cf = host_bf16_model(oracle, 8, 8, 64, max_pos, seed=11)
    ebits, ef = host_bf16_model(oracle, 4, 8, 32, max_pos, seed=13)
    cloud = upload_model(ek, ctx, cbits, 8, 8, 64, max_pos)
    edge = upload_model(ek, ctx, ebits, 4, 8, 32, max_pos)
    return edge, ebits, ef, cloud, cbits, cf


def test_deep_match_on_device(ek, ctx, oracle):
    edge, _, ef, cloud, _, cf = c1_models(ek, ctx, oracle, 600)
    pseed = oracle.mix(42, 0x9B0BE)
    pe = oracle.generate_embeddings(pseed, 64, edge.h)
    pc = oracle.generate_embeddings(pseed, 64, cloud.h)
    dm, cka, rsa, best = ek.deep_match(edge, cloud, dev32(pe), dev32(pc), 2, 0.0, -1.0)
    # K7 on the device's own probe outputs == the oracle's match_layers on them, bit for bit
    eo = ek.prefill(edge, dev32(pe))[0].double().cpu().numpy()
    co = ek.prefill(cloud, dev32(pc))[0].double().cpu().numpy()
    w = oracle.match_layers(eo, co, 0.0, -1.0)
    assert np.array_equal(cka, w[0]) and np.array_equal(rsa, w[1]) and best.tolist() == w[2].tolist()
    # the map equals the one from the fp64 oracle prefill (argmax margins are percent-level)
    wf = oracle.match_layers(oracle.prefill(ef, pe)[0], oracle.prefill(cf, pc)[0], 0.0, -1.0)
    assert best.tolist() == wf[2].tolist()
    assert dm == {2: int(best[2]), 3: int(best[3])}
    with pytest.raises(ek.EkvError, match="edge layer 2 has no matched cloud layer"):
        ek.deep_match(edge, cloud, dev32(pe), dev32(pc), 2, 1.5, -1.0)


def test_prompt_context_full_path_config1(ek, ctx, oracle):
    """Artifacts (sim.cpp:100-265) end to end on the device at configs[0]'s shape: layer
    map, edge + cloud context prefill, K1/K2 mask, K3 codes into the assembled context,
    then collaborative decode (U = 16, T = 16) -- every stage against the oracle."""
    S, U, T, deep = 512, 16, 16, 2
    max_pos = S + U + T
    edge, ebits, ef, cloud, cbits, cf = c1_models(ek, ctx, oracle, max_pos)
    pseed = oracle.mix(42, 0x9B0BE)
    pe = dev32(oracle.generate_embeddings(pseed, 64, edge.h))
    pc = dev32(oracle.generate_embeddings(pseed, 64, cloud.h))
    dmap = ek.deep_match(edge, cloud, pe, pc, deep, 0.0, -1.0)[0]
    eseed = oracle.mix(42, 0xC7E20000)
    emb_e = oracle.generate_embeddings(eseed, S, edge.h).astype(np.float32)
    emb_c = oracle.generate_embeddings(eseed, S, cloud.h).astype(np.float32)
    kvc = ek.AssembledContext(edge, S, [16, 16, 8, 8], group=32)
    kept, margin = ek.prompt_context(edge, cloud, dev32(emb_e), dev32(emb_c), dmap, 0.5, kvc)
    # the same device prefills, re-run: the inputs the alignment consumed (deterministic)
    _, _, e_k, e_v = ek.prefill(edge, dev32(emb_e), want_kv=True)
    c_lo, c_x0, c_k, c_v = ek.prefill(cloud, dev32(emb_c), want_x0=True, want_kv=True)
    lcs = sorted(set(dmap.values()))
    X = np.stack([(c_x0 if lc == 0 else c_lo[lc - 1]).cpu().numpy() for lc in lcs])
    xb = bf16_to_f64(f32_to_bf16_bits(X))                                   # [m][S][hc]
    wq = bf16_to_f64(np.stack([cbits["wqkvT"][lc][:cloud.h] for lc in lcs]))
    q_stack = np.concatenate([(xb[i] @ wq[i].T).reshape(S, 8, 64).transpose(1, 0, 2).reshape(-1, 64)
                              for i in range(len(lcs))])
    ckb = bf16_to_f64(bits_of(c_k)).reshape(8, 8, S, 64)
    k_stack = np.concatenate([ckb[lc].reshape(-1, 64) for lc in lcs])
    want_kept, _ = oracle.select_channels(q_stack, k_stack, oracle.prune_retained(0.5, 64))
    assert margin > 1e-6
    assert kept.tolist() == want_kept.tolist()
    # the cloud prefill itself vs the fp64 oracle (the alignment's inputs are right)
    wlo, wk, _ = oracle.prefill(cf, emb_c.astype(np.float64), kv_bf16=True)
    for lc in lcs:
        assert within_bf16_ulp(ckb[lc], wk[lc])
        if lc:
            assert normwise(c_lo[lc - 1].cpu().numpy(), wlo[lc - 1]) <= TOL
    # assembled context: local layers = edge prefill KV; deep layers = codes of the cloud KV
    ck = np.zeros((4, 8, S, 32)); cv = np.zeros((4, 8, S, 32))
    ekb = bf16_to_f64(bits_of(e_k)).reshape(4, 8, S, 32)
    evb = bf16_to_f64(bits_of(e_v)).reshape(4, 8, S, 32)
    cvb = bf16_to_f64(bits_of(c_v)).reshape(8, 8, S, 64)
    import ctypes as C
    from paper_2505_14085_b200.capi import call
    for l in range(4):
        seg = kvc.segment(l)
        if l < 2:
            got = np.zeros((8 * S * 32,), np.uint16)
            call("ekv_copy", ctx.h, got.ctypes.data_as(C.c_void_p), C.c_void_p(seg.k), got.nbytes, 1)
            assert np.array_equal(got.reshape(8, S, 32), bits_of(e_k[l]).reshape(8, S, 32))
            ck[l] = ekb[l]; cv[l] = evb[l]
        else:
            lc = dmap[l]
            for src, dst, ptr, sptr in ((c_k, ck, seg.k, seg.k_scales), (c_v, cv, seg.v, seg.v_scales)):
                wc, ws = oracle.kv_compress(bits_of(src[lc]).reshape(8 * S, 64), want_kept, 8, 32)
                got = np.zeros_like(wc)
                call("ekv_copy", ctx.h, got.ctypes.data_as(C.c_void_p), C.c_void_p(ptr), got.nbytes, 1)
                assert np.array_equal(got, wc), ("codes", l)
                dst[l] = oracle.kv_dequant_f64(wc, ws, 32, 8, 32).reshape(8, S, 32)
    sess = ek.Session(edge, kvc, U + T)
    ue = oracle.generate_embeddings(oracle.mix(42, 0x55E20000), U, edge.h).astype(np.float32)
    pre, steps = ek.collaborative_decode(sess, ue, T)
    teacher = np.vstack([pre[-1:], steps[:-1]]).astype(np.float64)
    wp, ws_ = oracle.collaborative_decode(ef, ck, cv, ue.astype(np.float64), T, teacher=teacher,
                                          user_kv_bf16=True)
    assert max(normwise(pre[r], wp[r]) for r in range(U)) <= TOL
    assert max(normwise(steps[t], ws_[t]) for t in range(T)) <= TOL


def test_build_deep_kv_full_mask_and_errors(ek, ctx, oracle):
    """lambda = 0: ChannelMask::full (sim.cpp:255-256) -- the codes are the unpruned
    cloud KV; and the assemble_context errors for mismatched geometry."""
    H, S, d = 4, 128, 64
    bits, _ = host_bf16_model(oracle, 2, H, d, S + 8, seed=21)
    model = upload_model(ek, ctx, bits, 2, H, d, S + 8)
    kvc = ek.AssembledContext(model, S, [16, 8], group=d)
    X = torch.empty((1, S, H * d), dtype=torch.bfloat16, device="cuda")
    W = torch.empty((1, H * d, H * d), dtype=torch.bfloat16, device="cuda")
    K = torch.empty((1, H, S, d), dtype=torch.bfloat16, device="cuda")
    V = torch.empty_like(K)
    for i, t in enumerate((X, W, K, V)):
        ctx.fill_uniform_bf16(t, 31, i, -1, 1)
    ctx.synchronize()
    kept, margin = ek.build_deep_kv(ctx, kvc, {1: 5}, X, W, K, V, 0.0, [5])
    assert kept.tolist() == list(range(d)) and margin == float("inf")
    wc, _ = oracle.kv_compress(bits_of(K[0]).reshape(H * S, d), np.arange(d, dtype=np.int32), 8, d)
    import ctypes as C
    from paper_2505_14085_b200.capi import call
    got = np.zeros_like(wc)
    call("ekv_copy", ctx.h, got.ctypes.data_as(C.c_void_p), C.c_void_p(kvc.segment(1).k), got.nbytes, 1)
    assert np.array_equal(got, wc)
    with pytest.raises(ValueError, match="align with head pruning"):
        ek.build_deep_kv(ctx, kvc, {1: 5}, X, W, K, V, 0.5, [5])
    K8 = torch.empty((1, 8, S // 2, d), dtype=torch.bfloat16, device="cuda")
    with pytest.raises(ValueError, match="head count mismatch"):
        ek.build_deep_kv(ctx, kvc, {1: 5}, X, W, K8, K8, 0.0, [5])
    with pytest.raises(ek.EkvError, match="not a quantised"):
        ek.build_deep_kv(ctx, kvc, {0: 5}, X, W, K, V, 0.0, [5])


def test_long_prefill_tensor_core_attention(ek, ctx, oracle):
    """A 200-row user prefill over a bf16 + int8 context: one layer-major chunk whose
    context attention runs on K10 with two 128-row session tiles, then K11's causal
    user segment; vs the split-KV kernel K4 (EKV_PREFILL_K4=1) and the oracle."""
    import os
    from test_gpu_decode import make_context
    L, H, d, S, U = 2, 4, 64, 384, 200
    h = H * d
    bits, f64 = host_bf16_model(oracle, L, H, d, S + U + 8, seed=61)
    model = upload_model(ek, ctx, bits, L, H, d, S + U + 8)
    kvc, ck, cv = make_context(ek, ctx, oracle, model, S, [16, 8], seed=63)
    ue = oracle.generate_embeddings(65, U, h).astype(np.float32)
    out = ek.Session(model, kvc, U + 4).forward(dev32(ue)).cpu().numpy()
    os.environ["EKV_PREFILL_K4"] = "1"
    try:
        out4 = ek.Session(model, kvc, U + 4).forward(dev32(ue)).cpu().numpy()
    finally:
        del os.environ["EKV_PREFILL_K4"]
    assert max(normwise(out[r], out4[r].astype(np.float64)) for r in range(U)) <= 1e-4
    want, _ = oracle.collaborative_decode(f64, ck, cv, ue.astype(np.float64), 1, user_kv_bf16=True)
    for r in (0, 1, 127, 128, 129, U - 1):
        assert normwise(out[r], want[r]) <= TOL, r
