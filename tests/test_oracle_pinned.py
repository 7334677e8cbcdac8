"""Pin the C restatement (oracle/ekv_oracle.c) before trusting it.

Two anchors, both CPU-only:
* the reference's own golden values and known-answer tests (cited per test);
* bit-for-bit agreement with the UNMODIFIED reference compiled from its sources
  (oracle/_ref, built by oracle/Makefile), on seeded random inputs.
"""
import math

import numpy as np
import pytest

from oracle import model_from_reference_layout


def _rng(seed):
    return np.random.default_rng(seed)


# --------------------------------------------------------------------------- RNG
def test_mix_and_mt19937_match_reference(oracle, ref):
    for a, b in [(0, 0), (42, 0x9B0BE), (2**63 + 5, 17), (12345, 2**64 - 1)]:
        assert oracle.mix(a, b) == ref.mix(a, b)
    for seed in (0, 1, 42, 2**40 + 3):
        assert np.array_equal(oracle.mt64_stream(seed, 2000), ref.mt64_stream(seed, 2000))


def test_std_mt19937_64_known_answer(oracle):
    # The C++ standard fixes the 10000th output of a default-seeded
    # mt19937_64 (seed 5489) at 9981545732273789042 ([rand.predef]).
    assert int(oracle.mt64_stream(5489, 10000)[-1]) == 9981545732273789042


def test_model_checksum_golden(oracle, ref):
    # transformer_test.cpp:301-310: (2L, 2H, d4, max_pos 32, seed 12345)
    got = oracle.init_model(2, 2, 4, 32, 12345)
    assert f"{got['checksum']:016x}" == "fa0d3d12020757f7"
    want = ref.init_model(2, 2, 4, 32, 12345)
    assert want["checksum"] == got["checksum"]
    for key in ("wq", "wk", "wv", "out_proj", "pos"):
        assert np.array_equal(got[key], want[key]), key


def test_generate_embeddings_matches_and_is_width_stable(oracle, ref):
    a = oracle.generate_embeddings(99, 5, 12)
    assert np.array_equal(a, ref.generate_embeddings(99, 5, 12))
    # transformer_test.cpp:345-350: row i at width 4 is a prefix of width 8
    narrow = oracle.generate_embeddings(99, 3, 4)
    wide = oracle.generate_embeddings(99, 3, 8)
    assert np.array_equal(narrow, wide[:, :4])


# ---------------------------------------------------------- a6: select_channels
@pytest.mark.parametrize("lam,d,want", [(0.2, 80, 64), (0.0, 7, 7), (1.0, 7, 0),
                                        (1.0 / 3.0, 6, 4), (0.5, 7, 3), (0.5, 128, 64)])
def test_from_lambda_budgets(oracle, ref, lam, d, want):
    # head_prune_test.cpp:66-81
    assert oracle.prune_retained(lam, d) == want
    assert ref.prune_retained(lam, d) == want


def test_select_channels_tie_break_golden(oracle, ref):
    # head_prune_test.cpp:160-167: identical scores keep the lower indices
    q = np.array([[1, 1, 1], [0, 0, 0]], dtype=float)
    kept, _ = oracle.select_channels(q, q, oracle.prune_retained(1.0 / 3.0, 3))
    assert kept.tolist() == [0, 1]
    assert ref.select_channels(q, q, 1.0 / 3.0).tolist() == [0, 1]


def test_select_channels_matches_reference(oracle, ref):
    rng = _rng(3)
    for trial in range(40):
        d = int(rng.integers(2, 65))
        rows = int(rng.integers(1, 40))
        lam = float(rng.choice([0.0, 0.25, 1 / 3, 0.5, 0.75, 1.0]))
        scale = np.exp(rng.uniform(-1.5, 1.5, size=d))
        q = rng.uniform(-1, 1, (rows, d)) * scale
        k = rng.uniform(-1, 1, (rows + 3, d)) * scale[::-1]
        if trial % 7 == 0:  # exact ties
            q[:, : d // 2] = 1.0
            k[:, : d // 2] = 1.0
        retained = oracle.prune_retained(lam, d)
        kept, _ = oracle.select_channels(q, k, retained)
        assert kept.tolist() == ref.select_channels(q, k, lam).tolist()
        # ranking from column sums of squares (the GPU's interface) is the same rule
        assert oracle.rank_channels(oracle.colsq(q), oracle.colsq(k), retained).tolist() == kept.tolist()


# --------------------------------------------------------------- a7: prune_cache
def test_prune_cache_slice_matches_reference(oracle, ref):
    rng = _rng(5)
    L, H, S, dc = 2, 3, 7, 8
    keys = rng.uniform(-1, 1, (L, H, S, dc))
    vals = rng.uniform(-1, 1, (L, H, S, dc))
    kept = np.array([0, 2, 4, 5])
    rk, rv = ref.prune_cache(keys, vals, kept)
    # head_prune_test.cpp:247: out.keys[0][0](2,1) == in(2,2)
    assert rk[0, 0, 2, 1] == keys[0, 0, 2, 2]
    assert np.array_equal(rk, keys[..., kept]) and np.array_equal(rv, vals[..., kept])
    u16 = (rng.integers(0, 2**16, (L * H * S, dc))).astype(np.uint16)
    assert np.array_equal(oracle.prune_rows_bf16(u16, kept), u16[:, kept])


# ------------------------------------------------- a10/a11: segment + merge (Eq. 5)
def test_segment_and_merge_bit_identical_to_reference(oracle, ref):
    rng = _rng(7)
    for trial in range(200):
        d = int(rng.integers(1, 17))
        n = int(rng.integers(1, 40))
        s = 3.0 if trial % 5 == 0 else 1.0
        q = rng.uniform(-s, s, d)
        k = rng.uniform(-s, s, (n, d))
        v = rng.uniform(-s, s, (n, d))
        a = oracle.segment_attention(q, k, v)
        b = ref.segment_attention(q, k, v)
        assert np.array_equal(a[0], b[0]) and a[1] == b[1] and a[2] == b[2]
        k2 = rng.uniform(-s, s, (5, d))
        v2 = rng.uniform(-s, s, (5, d))
        u = oracle.segment_attention(q, k2, v2)
        m1 = oracle.merge_attention(a, u)
        m2 = ref.merge_attention(b, ref.segment_attention(q, k2, v2))
        assert np.array_equal(m1[0], m2[0]) and m1[1] == m2[1] and m1[2] == m2[2]


def test_merge_identity_over_random_splits(oracle):
    # cache_merge_test.cpp:153-176 / acceptance criterion 1 (<1e-12 / 1e-9)
    rng = _rng(11)
    worst = 0.0
    for trial in range(1000):
        d = int(rng.integers(1, 9))
        total = int(rng.integers(2, 16))
        split = int(rng.integers(1, total))
        s = 3.0 if trial % 3 == 0 else 1.0
        q = rng.uniform(-s, s, d)
        k = rng.uniform(-s, s, (total, d))
        v = rng.uniform(-s, s, (total, d))
        o, ac, au = oracle.merge_attention(oracle.segment_attention(q, k[:split], v[:split]),
                                           oracle.segment_attention(q, k[split:], v[split:]))
        assert abs(ac + au - 1.0) < 1e-12
        want, _, _ = oracle.segment_attention(q, k, v)
        worst = max(worst, float(np.max(np.abs(o - want))))
    assert worst < 1e-12


def test_merge_hot_cold_segments_golden(oracle):
    # cache_merge_test.cpp:178-200: logits ~+400 vs ~-50 merge exactly
    q = np.array([20.0, 0.0])
    kh = np.array([[20.0, 1.0], [19.5, -1.0]]); vh = np.array([[1.0, 2.0], [3.0, 4.0]])
    kc = np.array([[-2.5, 0.3], [-2.4, 0.1], [-2.6, 0.2]])
    vc = np.array([[5.0, 6.0], [7.0, 8.0], [9.0, 10.0]])
    o, ac, _ = oracle.merge_attention(oracle.segment_attention(q, kh, vh),
                                      oracle.segment_attention(q, kc, vc))
    assert math.isfinite(o[0]) and abs(ac - 1.0) < 1e-12
    want, _, _ = oracle.segment_attention(q, np.vstack([kh, kc]), np.vstack([vh, vc]))
    assert np.max(np.abs(o - want)) < 1e-12


def test_merge_rejects_bad_sigma(oracle):
    with pytest.raises(ValueError, match="non-positive or non-finite sigma"):
        oracle.merge_attention((np.ones(2), 0.0, 0.0), (np.ones(2), 1.0, 0.0))


# ------------------------------------------- a2/a12: prefill + collaborative_decode
def _ref_init_model(ref, L, H, d, max_pos, seed):
    m = ref.init_model(L, H, d, max_pos, seed)
    return model_from_reference_layout(m, L, H, d, max_pos)


def test_prefill_bit_identical_to_reference(oracle, ref):
    m = _ref_init_model(ref, 3, 2, 4, 32, 23)
    emb = oracle.generate_embeddings(41, 9, 8)
    a = oracle.prefill(m, emb)
    b = ref.prefill(m, emb)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)


@pytest.mark.parametrize("S,U,steps", [(0, 3, 2), (5, 3, 1), (6, 4, 5), (5, 0, 3)])
def test_collaborative_decode_bit_identical_to_reference(oracle, ref, S, U, steps):
    L, H, d = 4, 2, 3
    m = _ref_init_model(ref, L, H, d, 64, 5)
    h = H * d
    rng = _rng(S * 100 + U)
    ck = rng.uniform(-1, 1, (L, H, S, d)) if S else None
    cv = rng.uniform(-1, 1, (L, H, S, d)) if S else None
    ue = oracle.generate_embeddings(43, U, h)
    if U == 0:
        ue = np.zeros((0, h))
    p1, s1 = oracle.collaborative_decode(m, ck, cv, ue, steps)
    p2, s2 = ref.collaborative_decode(m, ck, cv, ue, steps, boundary=2)
    assert np.array_equal(p1, p2) and np.array_equal(s1, s2)


def test_context_from_same_model_reproduces_monolithic_prefill(oracle):
    # cache_merge_test.cpp:297-326 on the restatement
    o = oracle
    ref_like = o.init_model(3, 2, 4, 64, 23)
    m = model_from_reference_layout(ref_like, 3, 2, 4, 64)
    ctx_emb = o.generate_embeddings(41, 5, 8)
    user = o.generate_embeddings(43, 3, 8)
    _, k, v = o.prefill(m, ctx_emb)
    pre, _ = o.collaborative_decode(m, k, v, user, 1)
    lo, _, _ = o.prefill(m, np.vstack([ctx_emb, user]))
    assert np.max(np.abs(pre[-1] - lo[-1, -1])) < 1e-9


# ------------------------------------------------------------- a3: layer matching
def test_cka_rsa_match_layers_bit_identical(oracle, ref):
    rng = _rng(21)
    oe = rng.uniform(-1, 1, (16, 8))
    oc = rng.uniform(-1, 1, (16, 12))
    assert oracle.cka(oe, oc) == ref.cka(oe, oc)
    assert oracle.rsa(oe, oc) == ref.rsa(oe, oc)
    edge = _ref_init_model(ref, 3, 2, 6, 64, 41)
    cloud = _ref_init_model(ref, 5, 4, 6, 64, 43)
    pe = oracle.generate_embeddings(9, 16, 12)
    pc = oracle.generate_embeddings(9, 16, 24)
    eo = oracle.prefill(edge, pe)[0]
    co = oracle.prefill(cloud, pc)[0]
    a = oracle.match_layers(eo, co, 0.5, 0.3)
    b = ref.match_layers(eo, co, 0.5, 0.3)
    for x, y in zip(a, b):
        assert np.array_equal(x, y)
    # exhaustive-scan oracle, layer_match_test.cpp:286-329
    cka, rsa, best = a
    for le in range(3):
        ok = [lc for lc in range(5) if cka[le, lc] >= 0.5 and rsa[le, lc] >= 0.3]
        want = -1 if not ok else max(ok, key=lambda lc: (cka[le, lc], -lc))
        assert best[le] == want


def test_self_match_diagonal(oracle):
    # acceptance criterion 4 / layer_match_test.cpp:249-272
    m = model_from_reference_layout(oracle.init_model(5, 2, 8, 64, 2029), 5, 2, 8, 64)
    outs = oracle.prefill(m, oracle.generate_embeddings(404, 24, 16))[0]
    cka, _, best = oracle.match_layers(outs, outs, 0.5, 0.0)
    assert best.tolist() == [0, 1, 2, 3, 4]
    assert np.max(np.abs(np.diag(cka) - 1.0)) <= 1e-9


def test_layer_match_errors(oracle):
    with pytest.raises(ValueError, match="degenerate"):
        oracle.cka(np.ones((6, 3)), np.random.default_rng(0).uniform(-1, 1, (6, 3)))
    o = np.random.default_rng(1).uniform(-1, 1, (5, 3))
    o[2] = 0.0
    with pytest.raises(ValueError, match="row 2"):
        oracle.rsa(o, o)


# -------------------------------------------------------- a13: scheduler interface
def test_cache_source_and_pipeline_schedule(oracle, ref):
    # cost_model_test.cpp:92-114
    cases = [(5, 0.1, 99.0, 4, 6), (6, 0.0, 0.0, 4, 6), (2, 1.0, 2.0, 4, 6), (2, 3.0, 2.0, 4, 6),
             (1, 2.0, 2.0, 4, 6)]
    for c in cases:
        assert oracle.cache_source(*c) == ref.cache_source(*c)
    assert [oracle.cache_source(*c) for c in cases] == [2, 2, 0, 1, 0]
    assert oracle.cache_source(0, 1, 1, 4, 6) == -1
    pip, seq, tot = oracle.pipeline_schedule([2, 1, 4], [3, 2, 5])
    assert pip.tolist() == [2.0, 3.0, 4.0] and tot == 14.0 and seq == 17.0
    rng = _rng(7)
    for _ in range(200):
        n = int(rng.integers(1, 13))
        a = rng.uniform(0, 10, n); b = rng.uniform(0, 10, n)
        x = oracle.pipeline_schedule(a, b)
        y = ref.pipeline_schedule(a, b)
        assert np.array_equal(x[0], y[0]) and x[1] == y[1] and x[2] == y[2]
        assert x[2] <= x[1] + 1e-12 and x[2] >= max(a.sum(), b.sum()) - 1e-12


# --------------------------------------- alignment projection (Q colsq) restated
def test_align_qnorm_matches_direct_projection(oracle):
    rng = _rng(31)
    X = rng.uniform(-1, 1, (20, 16))
    wqT = rng.uniform(-1, 1, (24, 16))
    got = oracle.align_qnorm(X, wqT)
    want = ((X @ wqT.T) ** 2).sum(axis=0)
    assert np.allclose(got, want, rtol=1e-13, atol=0)
