"""Where each context layer of a prompt comes from: the edge's own prefill, a peer
edge GPU, the cloud, or the historical cache (the reference's context preparation,
sim.cpp:721-820, 881-895, with the Eq. 19 source rule cache_source,
cost_model.cpp:64-71).

* shallow layers [0, boundary): cache_source picks local (the edge's own context
  prefill) or peer (a peer edge GPU already holding the prompt's context: copied
  device to device over NVLink, AssembledContext.copy_layers_from, or over NCCL
  across processes, dist.stream_layers);
* deep layers [boundary, M): the cloud's aligned + compressed KV arrives as an
  EKVPACK1 stream over the link; a prompt whose pack is in the historical cache
  (pinned host memory, pre-seeded or kept from an earlier fetch) is served from it
  without the link (sim.cpp:885-895: "historical_cache_hit"); with the link down and
  no cached pack the request fails with "cloud unreachable" (sim.cpp:816-820).
"""
from __future__ import annotations

from typing import Callable

import torch

from . import edgekv as ek


class CloudUnreachable(ek.EkvError):
    def __init__(self, prompt_id: int):
        super().__init__(-1, f"cloud unreachable (prompt {prompt_id}: link down, no historical cache)")


class HistoricalCache:
    """Packed deep-layer KV per prompt id, kept in pinned host memory."""

    def __init__(self):
        self._packs: dict[int, torch.Tensor] = {}

    def put(self, prompt_id: int, pack: torch.Tensor) -> None:
        ek.kvpack_parse(pack)  # only valid packs are kept
        buf = pack if pack.is_pinned() else pack.pin_memory()
        self._packs[prompt_id] = buf

    def get(self, prompt_id: int) -> torch.Tensor | None:
        return self._packs.get(prompt_id)

    def __contains__(self, prompt_id: int) -> bool:
        return prompt_id in self._packs

    def __len__(self) -> int:
        return len(self._packs)


def shallow_sources(boundary: int, M: int, cost_local: float, cost_peer: float | None) -> list[str]:
    """Eq. 19 per shallow layer (layers are 1-based in cache_source): 'local' or 'peer'
    (no peer holding the prompt = infinite peer cost)."""
    cp = float("inf") if cost_peer is None else cost_peer
    return [ek.cache_source(l + 1, cost_local, cp, boundary, M) for l in range(boundary)]


def prepare_context(context: "ek.AssembledContext", prompt_id: int, boundary: int, *,
                    local: Callable[[list], None], peer: "ek.AssembledContext | None" = None,
                    cost_local: float = 1.0, cost_peer: float | None = None,
                    cloud: Callable[[], torch.Tensor] | None = None, link_up: bool = True,
                    history: HistoricalCache | None = None) -> dict:
    """Fill `context` for one prompt and return {layer: source}.

    local(layers): computes the listed shallow layers on this edge (its own context
    prefill); peer: a context holding the same prompt on a peer GPU; cloud(): returns
    the prompt's EKVPACK1 stream (align + compress on the cloud, then the link)."""
    M = context.model.L
    src = {}
    shallow = shallow_sources(boundary, M, cost_local, cost_peer if peer is not None else None)
    mine = [l for l, s in enumerate(shallow) if s == "local"]
    theirs = [l for l, s in enumerate(shallow) if s == "peer"]
    if mine:
        local(mine)
    if theirs:
        context.copy_layers_from(peer, theirs)
    src.update({l: "local" for l in mine})
    src.update({l: "peer" for l in theirs})
    if boundary < M:
        pack = history.get(prompt_id) if history is not None else None
        how = "historical"
        if pack is None:
            if not link_up or cloud is None:
                raise CloudUnreachable(prompt_id)
            pack = cloud()
            how = "cloud"
            if history is not None:
                history.put(prompt_id, pack)
        ek.kvpack_import(context, pack)
        info = ek.kvpack_parse(pack)
        missing = sorted(set(range(boundary, M)) - set(info["layers"]))
        if missing:
            raise ek.EkvError(-1, f"assemble_context: missing layer {missing[0]}")
        src.update({l: how for l in range(boundary, M)})
    return src
