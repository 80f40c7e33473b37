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
    inside its decode graph: k_exchange over peer memory (CUDA IPC), or one
    ncclAllGather whose rank-major output the combine sums in rank order."""
    out = np.ascontiguousarray(slots_local, np.float32).copy()
    all_reduce(out)
    return out


def combine(h: np.ndarray, weights, slots: np.ndarray) -> np.ndarray:
    """Reference-ordered residual mixture over the exchanged slots."""
    out = h
    for w, y in zip(weights, slots):
        out = out + np.float32(w) * y
    return out


TRANSPORTS = ("ipc", "nccl")


def transport_of(transport=None) -> str:
    """The slot-exchange transport: ``ipc`` (default: k_exchange, peer-memory
    stores and flags inside the decode graph) or ``nccl`` (one ncclAllGather
    per layer and position); ``MOE_EP_TRANSPORT`` overrides the default."""
    import os
    t = (transport or os.environ.get("MOE_EP_TRANSPORT") or "ipc").lower()
    if t not in TRANSPORTS:
        raise ValueError(f"unknown expert-parallel transport {t!r} (one of {TRANSPORTS})")
    return t


def nccl_unique_id() -> bytes:
    """A fresh 128-byte NCCL unique id (rank 0 makes it, every rank joins)."""
    import ctypes as C

    from ._lib import check, lib
    buf = C.create_string_buffer(128)
    check(lib().moe_nccl_unique_id(buf))
    return buf.raw


def share_nccl_id(group=None) -> bytes:
    """Rank 0's NCCL unique id on every rank of ``group`` (torch.distributed
    broadcast: the process group only carries the 128 bytes)."""
    import torch.distributed as dist
    box = [nccl_unique_id() if dist.get_rank(group) == 0 else None]
    dist.broadcast_object_list(box, src=dist.get_global_rank(group, 0) if group else 0,
                               group=group)
    return box[0]


def gather_combine(h: np.ndarray, weights, gathered: np.ndarray) -> np.ndarray:
    """The NCCL transport's combine: ``gathered`` is the all-gather output
    [N][top_k][d] (rank-major); slot j's contributions are summed in rank
    order, then the reference-ordered mixture (k_combine, rank_major)."""
    g = np.asarray(gathered, np.float32)
    slots = g[0].copy()
    for r in range(1, g.shape[0]):
        slots = slots + g[r]
    return combine(h, weights, slots)


def connect(engine, group=None, transport=None) -> str:
    """Connect every rank's engine to its peers over torch.distributed (all
    ranks call this collectively); returns the transport used.

    ``ipc``: all-gather the engines' CUDA IPC handles and open them.
    ``nccl``: rank 0's NCCL unique id is broadcast and every rank joins the
    communicator (the torch process group only carries the id)."""
    import torch.distributed as dist
    t = transport_of(transport)
    if t == "nccl":
        engine.ep_connect_nccl(share_nccl_id(group))
        return t
    handles = [None] * dist.get_world_size(group)
    dist.all_gather_object(handles, engine.ep_handle(), group=group)
    engine.ep_connect(handles)
    return t
