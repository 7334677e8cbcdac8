"""Packed-KV wire format on the device path: the compressed cloud layers of an
assembled context exported as one EKVPACK1 stream, imported into a fresh
context, give bit-identical storage and an identical collaborative decode."""
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


@pytest.fixture(scope="module")
def ctx(ek):
    return ek.Context(0)


def dev_bytes(ctx, ptr, n):
    from paper_2505_14085_b200.capi import call
    out = np.zeros(n, np.uint8)
    call("ekv_copy", ctx.h, C.c_void_p(out.ctypes.data), C.c_void_p(ptr), n, 1)
    return out


@pytest.mark.parametrize("fmt", [8, 4])
def test_kvpack_round_trip(ek, ctx, oracle, fmt):
    L, H, d, S, U, T = 3, 4, 64, 256, 3, 3
    formats = [16, fmt, fmt]
    bits, _ = host_bf16_model(oracle, L, H, d, S + U + T + 1, seed=61)
    model = upload_model(ek, ctx, bits, L, H, d, S + U + T + 1)
    kvc, _, _ = make_context(ek, ctx, oracle, model, S, formats, seed=63)
    kept = list(range(0, 2 * d, 2))
    pack = ek.kvpack_export(kvc, [1, 2], [5, 7], kept, 2 * d)
    info = ek.kvpack_parse(pack)
    assert info["layers"] == [1, 2] and info["cloud_layers"] == [5, 7] and info["kept"] == kept
    assert info["bits"] == fmt and info["S"] == S and info["bytes"] == pack.numel()
    # a fresh context: same local layer, cloud layers only from the pack
    kv2 = ek.AssembledContext(model, S, formats, group=kvc.segment(1).group)
    s0 = kvc.segment(0)
    kv2.upload_bf16(0, dev_bytes(ctx, s0.k, H * S * d * 2).view(np.uint16),
                    dev_bytes(ctx, s0.v, H * S * d * 2).view(np.uint16))
    ek.kvpack_import(kv2, pack)
    for l in (1, 2):
        a, b = kvc.segment(l), kv2.segment(l)
        nb = H * S * d * fmt // 8
        ns = H * S * (d // a.group) * 4
        assert np.array_equal(dev_bytes(ctx, a.k, nb), dev_bytes(ctx, b.k, nb))
        assert np.array_equal(dev_bytes(ctx, a.v_scales, ns), dev_bytes(ctx, b.v_scales, ns))
    ue = oracle.generate_embeddings(67, U, H * d).astype(np.float32)
    r1 = ek.collaborative_decode(ek.Session(model, kvc, U + T), ue, T)
    r2 = ek.collaborative_decode(ek.Session(model, kv2, U + T), ue, T)
    assert np.array_equal(r1[1], r2[1]) and np.array_equal(r1[0], r2[0])
    # corruption in transit is caught before anything is written
    bad = pack.clone()
    bad[-3] ^= 0xFF
    with pytest.raises(ek.EkvError, match="checksum mismatch in layer 2"):
        ek.kvpack_import(kv2, bad)
    other = ek.AssembledContext(model, S + 16, formats, group=kvc.segment(1).group)
    with pytest.raises(ek.EkvError, match="dim mismatch"):
        ek.kvpack_import(other, pack)


def test_forward_pack_eq20_over_the_wire_format(ek, ctx, oracle):
    """ekv_session_forward_pack: the pack's layers uploaded + hashed layer by layer while
    the user rows run layer-major == the resident-context forward, bit for bit; decode
    continues from it; a corrupted layer is reported."""
    L, H, d, S, U, T = 3, 4, 64, 256, 9, 3
    formats = [16, 8, 8]
    bits, _ = host_bf16_model(oracle, L, H, d, S + U + T + 1, seed=71)
    model = upload_model(ek, ctx, bits, L, H, d, S + U + T + 1)
    kvc, _, _ = make_context(ek, ctx, oracle, model, S, formats, seed=73)
    ue = torch.from_numpy(oracle.generate_embeddings(79, U, H * d).astype(np.float32)).cuda()
    ref = ek.Session(model, kvc, U + T)
    want = ref.forward_streamed(ue, {}).cpu().numpy()   # the same layer-major forward, resident
    want_steps = ref.decode(T).cpu().numpy()
    pack = ek.kvpack_export(kvc, [1, 2], [4, 6], list(range(0, 2 * d, 2)), 2 * d)
    kv2 = ek.AssembledContext(model, S, formats, group=kvc.segment(1).group)
    s0 = kvc.segment(0)
    kv2.upload_bf16(0, dev_bytes(ctx, s0.k, H * S * d * 2).view(np.uint16),
                    dev_bytes(ctx, s0.v, H * S * d * 2).view(np.uint16))
    sess = ek.Session(model, kv2, U + T)
    got = sess.forward_pack(ue, pack).cpu().numpy()
    assert np.array_equal(got, want)
    assert np.array_equal(sess.decode(T).cpu().numpy(), want_steps)
    bad = pack.clone()
    bad[-5] ^= 0x40
    s3 = ek.Session(model, kv2, U + T)
    with pytest.raises(ek.EkvError, match="checksum mismatch in layer 2"):
        s3.forward_pack(ue, bad)
