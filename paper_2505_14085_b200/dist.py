"""Multi-GPU plumbing of the path (torch.distributed; NCCL on the GPUs, gloo in
the CPU tests).

Sessions shard with no collective on the decode path: each rank replicates the
edge model and serves its own sessions (the reference round-robins requests
over edge nodes, scenario.cpp:302).  The only data movement is the emulated
cloud -> edge link: the cloud role (rank 0) aligns and compresses the deep
layers once per prompt and broadcasts the packed KV (codes, scales, kept
channel mask) to every edge rank -- the B200 counterpart of
Sim::submit_transfer (sim.cpp:417-449).
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
