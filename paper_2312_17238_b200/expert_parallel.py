"""Expert-parallel ownership for one node of N GPUs.

Rank r owns experts ``{e : floor(e * N / E) == r}`` of every layer: their
pinned-arena shard, their HBM cache slots and staging buffers, and their
store (the reference TieredExpertStore restricted to the owned keys,
store.py:85-92 accepts such subsets).  The dense path (embedding, attention,
gate / top-k / guesses, lm_head) is replicated deterministically on every
rank, so routing is identical everywhere without a broadcast.  Each rank
writes the SwiGLU outputs of the routed experts it owns into a
(top_k x d_model) fp32 slot buffer, zero elsewhere; one sum-exchange of that
buffer per layer is exact (exactly one rank contributes each slot, x + 0 is
exact), after which every rank applies the reference-ordered combine
``h + w0*y0 + w1*y1`` (model.py:251-254).
"""

from __future__ import annotations

import numpy as np


def owner_of(expert: int, n_experts: int, world: int) -> int:
    return (expert * world) // n_experts


def owned_experts(n_experts: int, rank: int, world: int) -> list[int]:
    return [e for e in range(n_experts) if owner_of(e, n_experts, world) == rank]


def owned_keys(n_layers: int, n_experts: int, rank: int, world: int) -> set:
    return {(l, e) for l in range(n_layers) for e in owned_experts(n_experts, rank, world)}


def owned_mask(n_layers: int, n_experts: int, rank: int, world: int) -> np.ndarray:
    m = np.zeros((n_layers, n_experts), np.uint8)
    m[:, owned_experts(n_experts, rank, world)] = 1
    return m


def local_cache_k(k: int, n_experts: int, world: int) -> int:
    """Per-rank LRU capacity under a node-wide budget of k experts per layer:
    the budget is split evenly and capped by the experts a rank owns."""
    return min(-(-k // world), len(owned_experts(n_experts, 0, world)))


def slot_exchange(slots_local: np.ndarray, all_reduce) -> np.ndarray:
    """Sum-exchange of the (top_k, d) slot buffer; ``all_reduce`` is the
    collective (NCCL on the GPU engine, gloo in the CPU tests)."""
    out = np.ascontiguousarray(slots_local, np.float32).copy()
    all_reduce(out)
    return out


def combine(h: np.ndarray, weights, slots: np.ndarray) -> np.ndarray:
    """Reference-ordered residual mixture over the exchanged slots."""
    out = h
    for w, y in zip(weights, slots):
        out = out + np.float32(w) * y
    return out


def connect(engine, group=None) -> None:
    """Exchange the engines' IPC handles over torch.distributed and connect
    every rank's engine to its peers (all ranks call this collectively)."""
    import torch.distributed as dist
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, engine.ep_handle(), group=group)
    engine.ep_connect(handles)
