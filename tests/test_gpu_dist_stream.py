"""The emulated cloud -> edge link at N > 1 over NCCL (paper_2505_14085_b200/dist.py):
the cloud rank's deep layers broadcast layer by layer into the edge rank's context,
each landed layer releasing that layer of the edge's layer-major user prefill
(ekv_session_forward_streamed, Eq. 20 on real streams).  The streamed forward must
equal the forward over the fully resident context bit for bit.  Needs two GPUs
(gpurun --gpus 2); one process per GPU."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.multiprocessing as mp

pytestmark = pytest.mark.gpu


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    import torch.distributed as dist
    from oracle import Oracle
    from paper_2505_14085_b200 import edgekv as ek
    from paper_2505_14085_b200 import dist as ekd
    from test_gpu_decode import host_bf16_model, make_context, upload_model
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    torch.cuda.set_device(rank)
    dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device(f"cuda:{rank}"))
    oracle = Oracle()
    ctx = ek.Context(rank)
    L, H, d, S, U = 4, 4, 64, 1024, 8
    formats = [16, 16, 8, 8]
    bits, _ = host_bf16_model(oracle, L, H, d, S + U + 4, seed=91)
    model = upload_model(ek, ctx, bits, L, H, d, S + U + 4)
    kvc, _, _ = make_context(ek, ctx, oracle, model, S, formats, seed=93)  # identical local layers
    if rank != 0:  # the edge's deep layers arrive over the link
        for l in (2, 3):
            for t in ekd.context_layer_views(kvc, [l])[0]:
                t.zero_()
        torch.cuda.synchronize()
    ue = torch.from_numpy(oracle.generate_embeddings(97, U, H * d).astype(np.float32)).cuda()
    sess = ek.Session(model, kvc, U)
    views = ekd.context_layer_views(kvc, [2, 3])
    torch.cuda.synchronize()
    info = ekd.stream_layers(views, src=0)
    got = sess.forward_streamed(ue, {2: info["events"][0], 3: info["events"][1]}).cpu().numpy()
    ekd.finish_stream(info)
    ref = ek.Session(model, kvc, U).forward(ue).cpu().numpy()   # everything resident now
    q.put((rank, bool(np.array_equal(got, ref)), info["bytes"], info["seconds"] > 0))
    dist.barrier()
    dist.destroy_process_group()


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (gpurun --gpus 2)")
@pytest.mark.timeout(300)
def test_per_layer_nccl_link_overlapped_with_prefill():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = sorted(q.get(timeout=240) for _ in range(world))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, nbytes, timed in res:
        assert same, rank
        assert nbytes == 2 * (2 * 4 * 1024 * 64 + 2 * 4 * 1024 * 4) and timed


def _link_worker(rank, world, q_id, q_out):
    import sys
    sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__))))
    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    from oracle import Oracle
    from paper_2505_14085_b200 import edgekv as ek
    from paper_2505_14085_b200 import dist as ekd
    from test_gpu_decode import host_bf16_model, make_context, upload_model
    torch.cuda.set_device(rank)
    oracle = Oracle()
    ctx = ek.Context(rank)
    L, H, d, S, U = 4, 4, 64, 1024, 8
    formats = [16, 16, 8, 8]
    bits, _ = host_bf16_model(oracle, L, H, d, S + U + 4, seed=91)
    model = upload_model(ek, ctx, bits, L, H, d, S + U + 4)
    kvc, _, _ = make_context(ek, ctx, oracle, model, S, formats, seed=93)
    if rank == 0:
        uid = ek.Link.unique_id()
        q_id.put(uid)
    else:
        uid = q_id.get(timeout=60)
        for l in (2, 3):   # the edge's deep layers arrive over the link
            for t in ekd.context_layer_views(kvc, [l])[0]:
                t.zero_()
        torch.cuda.synchronize()
    link = ek.Link(ctx, uid, world, rank)
    ue = torch.from_numpy(oracle.generate_embeddings(97, U, H * d).astype(np.float32)).cuda()
    if rank == 0:
        sec = link.send_layers(kvc, [2, 3], peer=1)
        q_out.put((rank, True, sec))
    else:
        sess = ek.Session(model, kvc, U)
        got, sec = link.recv_forward(sess, [2, 3], peer=0, emb=ue)
        ref = ek.Session(model, kvc, U).forward_streamed(ue, {}).cpu().numpy()
        q_out.put((rank, bool(np.array_equal(got.cpu().numpy(), ref)), sec))
    del link


@pytest.mark.skipif(torch.cuda.device_count() < 2, reason="needs two GPUs (gpurun --gpus 2)")
@pytest.mark.timeout(300)
def test_capi_nccl_link_per_layer():
    """The same link from the C ABI (ekv_link_*: ncclSend / ncclRecv per layer, NCCL
    resolved at run time), the receive overlapped with the edge's layer-major prefill."""
    ctx = mp.get_context("spawn")
    q_id, q_out = ctx.Queue(), ctx.Queue()
    procs = [ctx.Process(target=_link_worker, args=(r, 2, q_id, q_out)) for r in range(2)]
    for p in procs:
        p.start()
    res = sorted(q_out.get(timeout=240) for _ in range(2))
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    for rank, same, sec in res:
        assert same, rank
        assert sec > 0
