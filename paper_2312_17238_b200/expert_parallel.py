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


def rank_budget(k: int, b: int, m: int, n_experts: int, rank: int, world: int):
    """(k_r, b_r, m_r) of rank r under the single-GPU budget: the
    node-wide cache of k experts per layer and b staging buffers is split over
    the ranks -- rank r gets floor(k/N) + (r < k % N) slots, capped by the
    experts it owns, and floor(b/N) + (r < b % N) staging buffers -- so the node
    never caches more than one GPU would and offloading stays forced at every N
    (at N = 8, k = 4: four ranks cache one expert per layer, four cache none).
    A rank left with b_r = 0 staging buffers cannot prefetch (m_r = 0)."""
    own = len(owned_experts(n_experts, rank, world))
    kr = min(own, k // world + (1 if rank < k % world else 0))
    br = b // world + (1 if rank < b % world else 0)
    return kr, br, min(m, br)


def slot_exchange(slots_local: np.ndarray, all_reduce) -> np.ndarray:
    """Sum-exchange of the (top_k, d) slot buffer; ``all_reduce`` is the
    collective (gloo in the CPU tests).  The GPU engine does the same exchange
    inside its decode graph with k_exchange over peer memory (CUDA IPC)."""
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
