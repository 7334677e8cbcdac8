"""Multi-GPU plumbing of the path (torch.distributed; NCCL on the GPUs, gloo in
the CPU tests).

Sessions shard with no collective on the decode path: each rank replicates the
edge model and serves its own sessions (the reference round-robins requests
over edge nodes, scenario.cpp:302).  The only data movement is the emulated
cloud -> edge link: the cloud role (rank 0) aligns and compresses the deep
layers once per prompt and broadcasts the packed KV (codes, scales, kept
channel mask) to every edge rank -- the B200 counterpart of
Sim::submit_transfer (sim.cpp:417-449).  The transfer is per layer
(Sim::fetch_deep_layer, sim.cpp:802-814): layer l lands with its own CUDA
event, so the edge's layer-major prefill (ekv_session_forward_streamed) starts
layer l as soon as layer l arrived -- the Eq. 20 overlap of transfer and
compute (cost_model.cpp:73-100) on real streams.
"""
from __future__ import annotations

import time

import torch
import torch.distributed as dist


def session_shard(n_sessions: int, world: int, rank: int) -> list[int]:
    """Round-robin assignment of session ids to ranks (scenario.cpp:302)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} for world size {world}")
    return list(range(rank, n_sessions, world))


def broadcast_packed_kv(tensors: list[torch.Tensor], src: int = 0, group=None) -> dict:
    """Broadcast the packed deep-layer KV from the cloud rank to every edge rank.
    Tensors are updated in place on every rank.  Returns {bytes, seconds}."""
    nbytes = int(sum(t.numel() * t.element_size() for t in tensors))
    if dist.is_initialized() and dist.get_world_size(group) > 1:
        cuda = bool(tensors) and tensors[0].is_cuda
        # communicator set-up is not link time: one small warm-up collective first
        warm = torch.zeros(1, device=tensors[0].device if tensors else None)
        dist.broadcast(warm, src=src, group=group)
        dist.barrier(group)
        if cuda:
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
        t0 = time.perf_counter()
        for t in tensors:
            dist.broadcast(t, src=src, group=group)
        if cuda:
            e1.record()
            torch.cuda.synchronize()
            sec = max_over_ranks(e0.elapsed_time(e1) * 1e-3, device=tensors[0].device, group=group)
        else:
            sec = time.perf_counter() - t0
        return {"bytes": nbytes, "seconds": sec}
    return {"bytes": nbytes, "seconds": 0.0}


def max_over_ranks(value: float, device=None, group=None) -> float:
    """The job-level time of a timed region: the maximum over ranks."""
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return float(value)
    t = torch.tensor([float(value)], dtype=torch.float64, device=device)
    dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return float(t.item())


class _DevPtr:
    """__cuda_array_interface__ over raw device memory owned by the C ABI."""

    def __init__(self, ptr: int, nbytes: int):
        self.__cuda_array_interface__ = {"shape": (nbytes,), "typestr": "|u1", "data": (ptr, False),
                                         "version": 3, "strides": None}


def device_bytes(ptr: int, nbytes: int, device) -> torch.Tensor:
    """A uint8 tensor view of `nbytes` of device memory at `ptr` (no copy)."""
    return torch.as_tensor(_DevPtr(int(ptr), int(nbytes)), device=device)


def stream_layers(layer_bufs: list, src: int = 0, group=None, link_stream=None) -> dict:
    """Broadcast every layer's buffers from `src`, one layer after the other, on
    `link_stream` (CUDA) and record one event per layer when it has landed.  Returns
    {bytes, seconds (max over ranks), events}.  Works with CPU tensors under gloo
    (no events then)."""
    nbytes = int(sum(t.numel() * t.element_size() for bufs in layer_bufs for t in bufs))
    if not (dist.is_initialized() and dist.get_world_size(group) > 1):
        return {"bytes": nbytes, "seconds": 0.0, "events": [None] * len(layer_bufs)}
    cuda = bool(layer_bufs) and layer_bufs[0][0].is_cuda
    dev = layer_bufs[0][0].device
    warm = torch.zeros(1, device=dev)
    dist.broadcast(warm, src=src, group=group)  # communicator set-up is not link time
    dist.barrier(group)
    if not cuda:
        t0 = time.perf_counter()
        for bufs in layer_bufs:
            for t in bufs:
                dist.broadcast(t, src=src, group=group)
        return {"bytes": nbytes, "seconds": max_over_ranks(time.perf_counter() - t0, group=group),
                "events": [None] * len(layer_bufs)}
    torch.cuda.synchronize()
    link = link_stream or torch.cuda.Stream(device=dev)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    events = []
    with torch.cuda.stream(link):
        e0.record(link)
        for bufs in layer_bufs:
            for t in bufs:
                dist.broadcast(t, src=src, group=group)
            ev = torch.cuda.Event()
            ev.record(link)
            events.append(ev)
        e1.record(link)
    return {"bytes": nbytes, "events": events, "timing": (e0, e1), "stream": link}


def finish_stream(info: dict, group=None) -> dict:
    """Wait for a stream_layers transfer and fill in its link time (max over ranks)."""
    if "timing" in info:
        e0, e1 = info.pop("timing")
        info.pop("stream").synchronize()
        info["seconds"] = max_over_ranks(e0.elapsed_time(e1) * 1e-3, device="cuda", group=group)
    return info


def context_layer_views(context, layers) -> list:
    """The storage of each listed layer of an AssembledContext as uint8 device views
    (codes K, codes V, scales K, scales V for quantised layers; K, V for bf16)."""
    m = context.model
    dev = torch.device("cuda", m.ctx.device)
    out = []
    for l in layers:
        seg = context.segment(l)
        rows = m.H * seg.S
        if seg.format == 16:
            cb, sb = rows * m.d * 2, 0
        else:
            cb, sb = rows * m.d * seg.format // 8, rows * (m.d // seg.group) * 4
        bufs = [device_bytes(seg.k, cb, dev), device_bytes(seg.v, cb, dev)]
        if sb:
            bufs += [device_bytes(seg.k_scales, sb, dev), device_bytes(seg.v_scales, sb, dev)]
        out.append(bufs)
    return out


def stream_deep_layers(context, layers, src: int = 0, group=None) -> dict:
    """The emulated cloud -> edge link at N > 1: every listed layer of the cloud rank's
    assembled context broadcast into every edge rank's, layer by layer (NCCL over
    NVLink); waits for completion and reports {bytes, ms, gbs, layers, how}."""
    info = finish_stream(stream_layers(context_layer_views(context, layers), src, group), group)
    sec = info.get("seconds", 0.0)
    return {"ms": 1e3 * sec, "bytes": info["bytes"], "gbs": info["bytes"] / max(sec, 1e-12) / 1e9,
            "layers": len(layers),
            "how": "per-layer NCCL broadcast (codes + scales of each deep layer) from rank 0 (cloud "
                   "role) into every rank's context storage, one CUDA event per landed layer "
                   "(Sim::fetch_deep_layer, sim.cpp:802-814); once per prompt, outside the decode "
                   "timing"}


def capi_link(ctx, group=None):
    """An ekv_link (the C ABI's NCCL link) over the ranks of `group`: rank 0 makes the
    NCCL unique id, every rank receives it through torch.distributed (plumbing only)."""
    from . import edgekv as ek
    uid = [ek.Link.unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(uid, src=0, group=group)
    return ek.Link(ctx, uid[0], dist.get_world_size(group), dist.get_rank(group))


def link_deep_layers(link, context, session, layers) -> dict:
    """The cloud rank (0) sends `layers` of its context to every other rank through the C
    ABI's link (ncclSend / ncclRecv per layer); returns the per-destination link time."""
    rank, world = dist.get_rank(), dist.get_world_size()
    secs = []
    for dst in range(1, world):
        for rep in range(2):  # the first transfer of a pair also sets up NCCL's P2P connection
            if rank == 0:
                t = link.send_layers(context, layers, dst)
            elif rank == dst:
                t = link.recv_forward(session, layers, 0)[1]
            else:
                t = None
            if rep == 1 and t is not None:
                secs.append(t)
            dist.barrier()
    sec = max_over_ranks(max(secs) if secs else 0.0, device="cuda")
    nbytes = int(sum(t.numel() for bufs in context_layer_views(context, layers) for t in bufs))
    return {"ms_per_destination": 1e3 * sec, "bytes": nbytes, "gbs": nbytes / max(sec, 1e-12) / 1e9,
            "destinations": world - 1, "layers": len(layers),
            "how": "C-ABI link (ekv_link_send_layers / ekv_link_recv_forward): ncclSend/ncclRecv of "
                   "each deep layer's codes + scales, one NCCL group per layer, from rank 0 (cloud "
                   "role) to each edge rank in turn (second transfer of each pair: the first sets up "
                   "the P2P connection); once per prompt, outside the decode timing"}
