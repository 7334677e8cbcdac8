"""Context-layer sources (paper_2505_14085_b200/sources.py, ekv_kvctx_copy_layers):
Eq. 19 local-vs-peer for the shallow layers (cost_model.cpp:64-71), peer sharing over
NVLink (sim.cpp:757-786), the cloud pack over the link and the historical-cache
fallback when the link is down (sim.cpp:816-820, 885-895)."""
import ctypes as C

import numpy as np
import pytest
import torch

from test_gpu_decode import host_bf16_model, make_context, upload_model

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ek():
    from paper_2505_14085_b200 import build
    build.build()
    from paper_2505_14085_b200 import edgekv
    return edgekv


def layer_bytes(ctx, seg, H, d):
    from paper_2505_14085_b200.capi import call
    rows = H * seg.S
    nb = rows * d * seg.format // 8
    out = []
    for p in (seg.k, seg.v):
        a = np.zeros(nb, np.uint8)
        call("ekv_copy", ctx.h, C.c_void_p(a.ctypes.data), C.c_void_p(p), nb, 1)
        out.append(a)
    return out


def test_sources_peer_cloud_and_historical_cache(ek, oracle):
    from paper_2505_14085_b200 import sources
    ctx = ek.Context(0)
    L, H, d, S = 4, 4, 64, 256
    formats = [16, 16, 8, 8]
    bits, _ = host_bf16_model(oracle, L, H, d, S + 8, seed=81)
    model = upload_model(ek, ctx, bits, L, H, d, S + 8)
    cloud_side, _, _ = make_context(ek, ctx, oracle, model, S, formats, seed=83)   # holds the deep codes
    peer, _, _ = make_context(ek, ctx, oracle, model, S, formats, seed=85)         # a peer holding the prompt
    pack = ek.kvpack_export(cloud_side, [2, 3], [5, 7], list(range(0, 128, 2)), 128)
    fetched = []

    def cloud():
        fetched.append(1)
        return pack

    hist = sources.HistoricalCache()
    mine = ek.AssembledContext(model, S, formats, group=d)
    calls = []
    src = sources.prepare_context(mine, 7, 2, local=calls.append, peer=peer, cost_local=2.0, cost_peer=1.0,
                                  cloud=cloud, history=hist)
    assert src == {0: "peer", 1: "peer", 2: "cloud", 3: "cloud"} and not calls and len(fetched) == 1
    for l in range(4):
        want = peer if l < 2 else cloud_side
        assert all(np.array_equal(a, b) for a, b in zip(layer_bytes(ctx, mine.segment(l), H, d),
                                                        layer_bytes(ctx, want.segment(l), H, d)))
    # the link goes down: the same prompt is served from the historical cache ...
    again = ek.AssembledContext(model, S, formats, group=d)
    src = sources.prepare_context(again, 7, 2, local=calls.append, peer=None, cloud=cloud, link_up=False,
                                  history=hist)
    assert src[2] == src[3] == "historical" and len(fetched) == 1 and calls == [[0, 1]]
    assert np.array_equal(layer_bytes(ctx, again.segment(3), H, d)[1],
                          layer_bytes(ctx, cloud_side.segment(3), H, d)[1])
    # ... and a prompt it never saw fails like the reference
    with pytest.raises(sources.CloudUnreachable, match="cloud unreachable"):
        sources.prepare_context(again, 8, 2, local=calls.append, cloud=cloud, link_up=False, history=hist)
    # Eq. 19: equal cost keeps the layer local (cost_model_test.cpp:92-103)
    assert sources.shallow_sources(2, 4, 1.0, 1.0) == ["local", "local"]


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (gpurun --gpus 2)")
def test_peer_sharing_across_gpus_over_nvlink(ek, oracle):
    """A context on GPU 1 takes its shallow layers from the peer context on GPU 0."""
    L, H, d, S = 2, 4, 64, 512
    bits, _ = host_bf16_model(oracle, L, H, d, S + 8, seed=87)
    c0, c1 = ek.Context(0), ek.Context(1)
    m0 = upload_model(ek, c0, bits, L, H, d, S + 8)
    m1 = upload_model(ek, c1, bits, L, H, d, S + 8)
    a = ek.AssembledContext(m0, S, [16, 16])
    a.synthesize(89)
    b = ek.AssembledContext(m1, S, [16, 16])
    b.copy_layers_from(a, [0, 1])
    for l in range(2):
        assert all(np.array_equal(x, y) for x, y in zip(layer_bytes(c1, b.segment(l), H, d),
                                                        layer_bytes(c0, a.segment(l), H, d)))
    # the copied context decodes exactly like the peer's own
    ue = oracle.generate_embeddings(3, 4, H * d).astype(np.float32)
    r0 = ek.collaborative_decode(ek.Session(m0, a, 8), ue, 4)
    torch.cuda.set_device(1)
    r1 = ek.collaborative_decode(ek.Session(m1, b, 8), ue, 4)
    torch.cuda.set_device(0)
    assert np.array_equal(r0[1], r1[1])
