"""Pin the oracle restatement against golden vectors emitted by the UNMODIFIED
reference (tests/golden/make_golden.py, committed fixtures).  Runs on any host,
including ones where the reference library cannot be built."""
import os

import numpy as np
import pytest

from oracle import model_from_reference_layout

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def g():
    return np.load(G)


def test_rng_golden(oracle, g):
    assert np.array_equal(oracle.mt64_stream(int(g["mt_seed"][0]), 64), g["mt_stream"])
    for (a, b), want in zip(g["mix_in"], g["mix_out"]):
        assert oracle.mix(int(a), int(b)) == int(want)
    assert np.array_equal(oracle.generate_embeddings(99, 5, 12), g["embeddings"])


def test_model_golden(oracle, g):
    m = oracle.init_model(2, 2, 4, 32, 12345)
    assert m["checksum"] == int(g["model_checksum"][0])
    assert f"{m['checksum']:016x}" == "fa0d3d12020757f7"  # transformer_test.cpp:301-310
    for k in ("wq", "wk", "wv", "out_proj", "pos"):
        assert np.array_equal(m[k], g["model_" + k])


def test_prune_golden(oracle, g):
    for (lam, d), want in zip(g["from_lambda_in"], g["from_lambda_out"]):
        assert oracle.prune_retained(float(lam), int(d)) == int(want)
    kept, _ = oracle.select_channels(g["sel_q"], g["sel_k"], oracle.prune_retained(0.5, 16))
    assert kept.tolist() == g["sel_kept"].tolist()


def test_merge_golden(oracle, g):
    q, k, v = g["seg_q"], g["seg_k"], g["seg_v"]
    c = oracle.segment_attention(q, k[:6], v[:6])
    u = oracle.segment_attention(q, k[6:], v[6:])
    assert np.array_equal(np.concatenate([c[0], [c[1], c[2]]]), g["seg_ctx"])
    assert np.array_equal(np.concatenate([u[0], [u[1], u[2]]]), g["seg_user"])
    mo = oracle.merge_attention(c, u)
    assert np.array_equal(np.concatenate([mo[0], [mo[1], mo[2]]]), g["merge_out"])


def test_collaborative_decode_golden(oracle, g):
    m = model_from_reference_layout(
        {k: g["model_" + k] for k in ("wq", "wk", "wv", "out_proj", "pos")}, 2, 2, 4, 32)
    _, ck, cv = oracle.prefill(m, g["cd_ctx_emb"])
    pre, steps = oracle.collaborative_decode(m, ck, cv, g["cd_user"], 4)
    assert np.array_equal(pre, g["cd_prefill"]) and np.array_equal(steps, g["cd_steps"])


def test_match_layers_golden(oracle, g):
    cka, rsa, best = oracle.match_layers(g["ml_edge"], g["ml_cloud"], 0.5, 0.3)
    assert np.array_equal(cka, g["ml_cka"]) and np.array_equal(rsa, g["ml_rsa"])
    assert best.tolist() == g["ml_best"].tolist()


def test_scheduler_golden(oracle, g):
    for c, want in zip(g["cs_in"], g["cs_out"]):
        assert oracle.cache_source(int(c[0]), c[1], c[2], int(c[3]), int(c[4])) == int(want)
    pip, seq, tot = oracle.pipeline_schedule(g["ps_comm"], g["ps_comp"])
    assert np.array_equal(pip, g["ps_pip"]) and [seq, tot] == g["ps_tot"].tolist()
