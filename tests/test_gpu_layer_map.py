"""K7: the layer map (match_layers, layer_match.cpp:166-228) on the device.

The kernel computes in fp64 with the reference's operation order, so the CKA /
RSA matrices must be bit-identical to the oracle restatement (itself pinned
bit-identical to the reference, test_oracle_pinned.py) and the argmax equal.
"""
import os

import numpy as np
import pytest
import torch

from oracle import model_from_reference_layout

pytestmark = pytest.mark.gpu

G = os.path.join(os.path.dirname(os.path.abspath(__file__)), "golden", "reference_vectors.npz")


@pytest.fixture(scope="module")
def ctx():
    from paper_2505_14085_b200 import edgekv as ek
    return ek.Context(0)


def _dev(ctx, edge, cloud, t_cka, t_rsa):
    from paper_2505_14085_b200 import edgekv as ek
    e = torch.from_numpy(np.ascontiguousarray(edge, dtype=np.float64)).cuda()
    c = torch.from_numpy(np.ascontiguousarray(cloud, dtype=np.float64)).cuda()
    return ek.match_layers_dev(ctx, e, c, t_cka, t_rsa)


def _same(a, b):
    for x, y in zip(a, b):
        assert np.array_equal(x, y), (x, y)


def test_golden_fixture(ctx, oracle):
    g = np.load(G)
    got = _dev(ctx, g["ml_edge"], g["ml_cloud"], 0.5, 0.3)
    assert np.array_equal(got[0], g["ml_cka"]) and np.array_equal(got[1], g["ml_rsa"])
    assert got[2].tolist() == g["ml_best"].tolist()


@pytest.mark.parametrize("me,nc,n,ce,cc", [(3, 5, 16, 12, 24), (4, 8, 64, 256, 512),
                                          (8, 12, 64, 2048, 4096), (2, 3, 3, 5, 7)])
def test_random_outputs_bit_identical(ctx, oracle, me, nc, n, ce, cc):
    rng = np.random.default_rng(me * 100 + nc)
    edge = rng.uniform(-1, 1, (me, n, ce))
    cloud = rng.uniform(-1, 1, (nc, n, cc))
    # correlate some layers so the argmax is non-trivial
    for le in range(me):
        lc = (le * nc) // me
        w = min(ce, cc)
        cloud[lc, :, :w] += 2.0 * edge[le, :, :w]
    for tc, tr in [(0.0, -1.0), (0.5, 0.3), (0.9, 0.9)]:
        _same(_dev(ctx, edge, cloud, tc, tr), oracle.match_layers(edge, cloud, tc, tr))


def test_probe_prefill_outputs(ctx, oracle):
    # the real use: probe prefill of two reference-initialised models
    m = model_from_reference_layout(oracle.init_model(4, 2, 8, 64, 7), 4, 2, 8, 64)
    mc = model_from_reference_layout(oracle.init_model(6, 2, 16, 64, 9), 6, 2, 16, 64)
    eo = oracle.prefill(m, oracle.generate_embeddings(5, 32, 16))[0]
    co = oracle.prefill(mc, oracle.generate_embeddings(5, 32, 32))[0]
    _same(_dev(ctx, eo, co, 0.0, -1.0), oracle.match_layers(eo, co, 0.0, -1.0))
    # self match: diagonal (acceptance criterion 4)
    cka, _, best = _dev(ctx, eo, eo, 0.5, 0.0)
    assert best.tolist() == [0, 1, 2, 3]
    assert np.max(np.abs(np.diag(cka) - 1.0)) <= 1e-9


def test_ties_pick_smaller_cloud_layer(ctx, oracle):
    rng = np.random.default_rng(3)
    edge = rng.uniform(-1, 1, (2, 8, 6))
    cloud = np.stack([edge[0], edge[0], edge[1], edge[1]])
    _, _, best = _dev(ctx, edge, cloud, 0.0, -1.0)
    assert best.tolist() == [0, 2]


def test_errors_match_reference_messages(ctx):
    from paper_2505_14085_b200.capi import EkvError
    rng = np.random.default_rng(4)
    edge = rng.uniform(-1, 1, (2, 8, 6))
    cloud = rng.uniform(-1, 1, (3, 8, 10))
    bad = cloud.copy()
    bad[1, 5, :] = 0.0
    with pytest.raises(EkvError, match="zero-norm row 5"):
        _dev(ctx, edge, bad, 0.0, -1.0)
    with pytest.raises(EkvError, match="degenerate representation"):
        _dev(ctx, np.zeros_like(edge), cloud, 0.0, -1.0)
    with pytest.raises(EkvError, match="theta_cka"):
        _dev(ctx, edge, cloud, -0.1, 0.0)
