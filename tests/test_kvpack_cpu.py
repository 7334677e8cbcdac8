"""Packed-KV wire format (EKVPACK1, include/ekv_capi.h) -- host side, no GPU:
the FNV-1a 64 checksum is the reference's fnv1a64 (rng.cpp:7-15, pinned through
the oracle), and packs written here independently from the documented layout
(version 1: FNV over each layer payload; version 2: FNV over 4 KiB chunk FNVs)
are accepted by ekv_kvpack_parse, while corruption anywhere is rejected."""
import struct

import numpy as np
import pytest

from paper_2505_14085_b200 import edgekv as ek


def test_fnv1a64_matches_reference_restatement(oracle):
    assert ek.fnv1a64(b"") == 0xCBF29CE484222325
    assert ek.fnv1a64(b"a") == 0xAF63DC4C8601EC8C
    rng = np.random.default_rng(5)
    for n in (1, 7, 1000, 65537):
        buf = rng.integers(0, 256, n, dtype=np.uint8)
        want = oracle.lib.ekvo_fnv1a64(buf.ctypes.data, buf.nbytes, 14695981039346656037)
        assert ek.fnv1a64(buf) == want


def fnv(b: bytes) -> int:
    h = 14695981039346656037
    for x in b:
        h = ((h ^ x) * 1099511628211) & 0xFFFFFFFFFFFFFFFF
    return h


def write_pack(n, H, S, d_e, d_c, bits, group, seed=0):
    rng = np.random.default_rng(seed)
    rows = H * S
    layer = [rng.integers(0, 256, 2 * rows * d_e * bits // 8, dtype=np.uint8).tobytes() +
             rng.standard_normal(2 * rows * (d_e // group)).astype(np.float32).tobytes() for _ in range(n)]
    edge = list(range(10, 10 + n)); cloud = [2 * e for e in edge]; kept = list(range(0, 2 * d_e, 2))
    body = struct.pack(f"<{n}i{n}i{d_e}i", *edge, *cloud, *kept) + struct.pack(f"<{n}Q", *[fnv(p) for p in layer])
    hb = (64 + len(body) + 255) // 256 * 256
    head = b"EKVPACK1" + struct.pack("<12I", 1, n, H, S, d_e, d_c, bits, group, hb, 0, 0, 0)
    hdr = bytearray(head + struct.pack("<Q", 0) + body + bytes(hb - 64 - len(body)))
    struct.pack_into("<Q", hdr, 56, fnv(bytes(hdr)))
    return bytes(hdr) + b"".join(layer), edge, cloud, kept


def chunked_fnv(arrays: list) -> int:
    """Version-2 layer checksum: FNV-1a 64 over the little-endian u64 FNV-1a 64s of
    4 KiB chunks of each array, in payload order."""
    hs = []
    for a in arrays:
        for off in range(0, len(a), 4096):
            hs.append(fnv(a[off:off + 4096]))
    return fnv(struct.pack(f"<{len(hs)}Q", *hs))


def write_pack_v2(n, H, S, d_e, d_c, bits, group, seed=0):
    rng = np.random.default_rng(seed)
    rows = H * S
    cb, sb = rows * d_e * bits // 8, rows * (d_e // group) * 4
    layers = []
    for _ in range(n):
        arrs = [rng.integers(0, 256, cb, dtype=np.uint8).tobytes() for _ in range(2)] + \
               [rng.standard_normal(sb // 4).astype(np.float32).tobytes() for _ in range(2)]
        layers.append(arrs)
    edge = list(range(3, 3 + n)); cloud = [e + 1 for e in edge]; kept = list(range(d_e))
    body = struct.pack(f"<{n}i{n}i{d_e}i", *edge, *cloud, *kept) + \
        struct.pack(f"<{n}Q", *[chunked_fnv(a) for a in layers])
    hb = (64 + len(body) + 255) // 256 * 256
    head = b"EKVPACK1" + struct.pack("<12I", 2, n, H, S, d_e, d_c, bits, group, hb, 0, 0, 0)
    hdr = bytearray(head + struct.pack("<Q", 0) + body + bytes(hb - 64 - len(body)))
    struct.pack_into("<Q", hdr, 56, fnv(bytes(hdr)))
    return bytes(hdr) + b"".join(b"".join(a) for a in layers), edge


def test_parse_version2_chunked_checksums():
    # arrays longer than one 4 KiB chunk, with a short last chunk
    buf, edge = write_pack_v2(2, 3, 100, 64, 128, 8, 64, seed=3)
    info = ek.kvpack_parse(np.frombuffer(buf, np.uint8))
    assert info["layers"] == edge and info["bytes"] == len(buf)
    a = np.frombuffer(buf, np.uint8).copy()
    a[-7] ^= 0x10  # the last layer's V scales
    with pytest.raises(ek.EkvError, match="checksum mismatch in layer 4"):
        ek.kvpack_parse(a)


@pytest.mark.parametrize("bits,group", [(8, 64), (4, 32)])
def test_parse_independently_written_pack(bits, group):
    n, H, S, d_e, d_c = 3, 4, 40, 64, 128
    buf, edge, cloud, kept = write_pack(n, H, S, d_e, d_c, bits, group)
    assert len(buf) == ek.kvpack_size(n, H, S, d_e, bits, group)
    info = ek.kvpack_parse(np.frombuffer(buf, np.uint8))
    assert (info["n_layers"], info["H"], info["S"], info["d_e"], info["d_c"], info["bits"], info["group"]) == \
        (n, H, S, d_e, d_c, bits, group)
    assert info["layers"] == edge and info["cloud_layers"] == cloud and info["kept"] == kept
    assert info["bytes"] == len(buf)


def test_parse_rejects_corruption():
    buf, _, _, _ = write_pack(2, 2, 16, 64, 128, 8, 64, seed=1)
    a = np.frombuffer(buf, np.uint8).copy()
    b = a.copy(); b[-1] ^= 1
    with pytest.raises(ek.EkvError, match="checksum mismatch in layer 11"):
        ek.kvpack_parse(b)
    b = a.copy(); b[0] = ord("X")
    with pytest.raises(ek.EkvError, match="bad magic"):
        ek.kvpack_parse(b)
    b = a.copy(); b[64] ^= 1  # the layer map
    with pytest.raises(ek.EkvError, match="header checksum mismatch"):
        ek.kvpack_parse(b)
    with pytest.raises(ek.EkvError, match="truncated"):
        ek.kvpack_parse(a[:-5])
    with pytest.raises(ek.EkvError, match="bits must be 8 or 4"):
        ek.kvpack_size(1, 2, 16, 64, 16, 64)
