"""Multi-rank host logic on CPU (gloo, world size 2): session sharding, the
cloud->edge packed-KV broadcast and the max-over-ranks job time."""
import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2505_14085_b200 import dist as ekd
    g = torch.Generator().manual_seed(7)
    codes = torch.randint(0, 255, (11, 32, 64, 64), dtype=torch.uint8, generator=g)
    scales = torch.rand((11, 32, 64, 1), generator=g)
    kept = torch.arange(0, 128, 2, dtype=torch.int32)
    if rank != 0:  # edge ranks start with garbage
        codes.zero_(); scales.fill_(-1.0); kept.fill_(-1)
    info = ekd.broadcast_packed_kv([codes, scales, kept])
    # the per-layer link (Sim::fetch_deep_layer): layer by layer from the cloud rank
    layers = [[torch.full((5,), float(rank * 100 + l)), torch.full((3,), -float(l))] for l in range(4)]
    if rank == 0:
        for l in range(4):
            layers[l][0].fill_(float(l)); layers[l][1].fill_(float(10 + l))
    st = ekd.stream_layers(layers, src=0)
    assert st["bytes"] == 4 * (5 + 3) * 4 and len(st["events"]) == 4
    assert all(float(layers[l][0][0]) == l and float(layers[l][1][2]) == 10 + l for l in range(4))
    digest = (int(codes.long().sum()), float(scales.sum()), kept.tolist()[:4])
    t = ekd.max_over_ranks(1.0 + rank)
    q.put((rank, digest, info["bytes"], t, ekd.session_shard(10, world, rank)))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.timeout(120)
def test_two_rank_broadcast_shard_and_max():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=100) for _ in range(world))
    for p in procs:
        p.join(timeout=30)
        assert p.exitcode == 0
    (r0, d0, b0, t0, s0), (r1, d1, b1, t1, s1) = res
    assert d0 == d1 and d0[2] == [0, 2, 4, 6]          # every edge rank holds the cloud's KV
    assert b0 == b1 == 11 * 32 * 64 * 64 + 11 * 32 * 64 * 4 + 64 * 4
    assert t0 == t1 == 2.0                              # job time = slowest rank
    assert sorted(s0 + s1) == list(range(10)) and not set(s0) & set(s1)


def test_session_shard_rejects_bad_rank():
    from paper_2505_14085_b200 import dist as ekd
    with pytest.raises(ValueError):
        ekd.session_shard(4, 2, 2)
    assert ekd.session_shard(5, 1, 0) == [0, 1, 2, 3, 4]
