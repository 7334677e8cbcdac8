"""GPU parity of the batched-session decode (k_batch.cu, BASELINE configs[2]):
B concurrent sessions over one shared assembled context, advanced in lock-step
through the C ABI.  Each session must equal the reference's collaborative_decode
(cache_merge.cpp:230-273) on its own user prompt -- the oracle is run per
session, teacher-forced with that session's own GPU input rows (as in
test_gpu_decode.py), with the user cache rounded to bf16 as stored.
Bar: normwise max|gpu-ref|/max|ref| <= 1e-3 per output row, fp32 outputs.
"""
import numpy as np
import pytest
import torch

from test_gpu_decode import TOL, host_bf16_model, make_context, normwise, upload_model

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


def check_sessions(oracle, f64, ck, cv, ue, pre, steps, which):
    U, T = ue.shape[1], steps.shape[0]
    h = ue.shape[2]
    worst = 0.0
    for b in which:
        teacher = np.vstack([pre[-1:, b] if U else np.zeros((1, h)), steps[:-1, b]]).astype(np.float64)
        wp, ws = oracle.collaborative_decode(f64, ck, cv, ue[b].astype(np.float64), T, teacher=teacher,
                                             user_kv_bf16=True)
        for r in range(U):
            e = normwise(pre[r, b], wp[r]); worst = max(worst, e)
            assert e <= TOL, (b, "prefill", r, e)
        for t in range(T):
            e = normwise(steps[t, b], ws[t]); worst = max(worst, e)
            assert e <= TOL, (b, "step", t, e)
    return worst


@pytest.mark.parametrize("B,fmts,H,S,U,T", [(5, [16, 16], 4, 320, 3, 4),    # ragged last chunk
                                            (5, [16, 8], 4, 320, 3, 4),     # [local bf16 | cloud int8]
                                            (3, [16, 16], 4, 0, 2, 3),      # empty context (s = 0 bypass)
                                            (8, [8, 16, 8], 4, 128, 0, 3),  # no user prompt
                                            (33, [8], 4, 1000, 2, 2),       # BN = 64, many chunks
                                            (2, [16, 8], 8, 2048, 2, 2),    # C2 context length
                                            (3, [16, 8], 4, 32768, 2, 2)])  # C4 context length
def test_batch_matches_oracle_per_session(ek, ctx, oracle, B, fmts, H, S, U, T):
    L = len(fmts)
    d = 64
    h, max_pos = H * d, S + U + T + 8
    bits, f64 = host_bf16_model(oracle, L, H, d, max_pos, seed=17 + S)
    model = upload_model(ek, ctx, bits, L, H, d, max_pos)
    kvc, ck, cv = make_context(ek, ctx, oracle, model, S, fmts, seed=19 + S)
    batch = ek.SessionBatch(model, kvc, B, U + T)
    ue = np.stack([oracle.generate_embeddings(1000 + b, max(U, 1), h)[:U] for b in range(B)]).astype(np.float32)
    pre, steps = ek.collaborative_decode_batch(batch, ue, T)
    assert np.all(np.isfinite(steps))
    check_sessions(oracle, f64, ck if S else None, cv if S else None, ue, pre, steps, range(B))
    # the device API (forward + decode) is the same computation, bit for bit
    batch.reset()
    if U:
        out = batch.forward(torch.from_numpy(ue).cuda())
        assert np.array_equal(out.cpu().numpy(), pre)
    st = batch.decode(T).cpu().numpy()
    assert np.array_equal(st, steps)


def test_batch_two_tiles_and_single_session_agreement(ek, ctx, oracle):
    """B = 130 > 128 sessions (two tensor-core session tiles); spot-check sessions against
    the oracle and every session against the batch-1 engine on the same inputs."""
    B, L, H, d, S, U, T = 130, 1, 4, 64, 256, 2, 2
    h, max_pos = H * d, 512
    bits, f64 = host_bf16_model(oracle, L, H, d, max_pos, seed=23)
    model = upload_model(ek, ctx, bits, L, H, d, max_pos)
    kvc, ck, cv = make_context(ek, ctx, oracle, model, S, [8] * L, seed=29)
    batch = ek.SessionBatch(model, kvc, B, U + T)
    ue = np.stack([oracle.generate_embeddings(2000 + b, U, h) for b in range(B)]).astype(np.float32)
    pre, steps = ek.collaborative_decode_batch(batch, ue, T)
    check_sessions(oracle, f64, ck, cv, ue, pre, steps, [0, 1, 64, 127, 128, 129])
    sess = ek.Session(model, kvc, U + T)
    for b in (0, 77, 129):
        p1, s1 = ek.collaborative_decode(sess, ue[b], T)
        assert max(normwise(p1[r], pre[r, b]) for r in range(U)) <= TOL
        assert max(normwise(s1[t], steps[t, b]) for t in range(T)) <= TOL


def test_batch_sessions_are_independent(ek, ctx, oracle):
    """Permuting the sessions permutes the outputs exactly (no cross-session leakage)."""
    B, L, H, d, S, U, T = 6, 2, 4, 64, 192, 2, 3
    h, max_pos = H * d, 512
    bits, _ = host_bf16_model(oracle, L, H, d, max_pos, seed=31)
    model = upload_model(ek, ctx, bits, L, H, d, max_pos)
    kvc, _, _ = make_context(ek, ctx, oracle, model, S, [16, 8], seed=37)
    batch = ek.SessionBatch(model, kvc, B, U + T)
    ue = np.stack([oracle.generate_embeddings(3000 + b, U, h) for b in range(B)]).astype(np.float32)
    _, s1 = ek.collaborative_decode_batch(batch, ue, T)
    perm = np.array([3, 0, 5, 1, 4, 2])
    _, s2 = ek.collaborative_decode_batch(batch, ue[perm], T)
    assert np.array_equal(s2, s1[:, perm])


def test_batch_errors(ek, ctx, oracle):
    L, H, d = 2, 4, 64
    bits, _ = host_bf16_model(oracle, L, H, d, 64, seed=3)
    model = upload_model(ek, ctx, bits, L, H, d, 64)
    kvc = ek.AssembledContext(model, 60, [16, 16])
    batch = ek.SessionBatch(model, kvc, 4, 16)
    ue = np.zeros((4, 3, H * d), np.float32)
    with pytest.raises(ek.EkvError, match="position overflow"):
        ek.collaborative_decode_batch(batch, ue, 2)
    with pytest.raises(ek.EkvError, match="steps must be >= 1"):
        ek.collaborative_decode_batch(batch, ue[:, :1], 0)
    other = ek.EdgeModel(ctx, 2, 8, 32, 64)
    with pytest.raises(ek.EkvError, match="align with head pruning"):
        ek.SessionBatch(other, kvc, 2, 4)
    kv4 = ek.AssembledContext(model, 64, [16, 4], group=32)
    with pytest.raises(ek.EkvError, match="not supported"):
        ek.SessionBatch(model, kv4, 2, 4)
