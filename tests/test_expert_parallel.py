"""Expert-parallel host logic on CPU: world_size 2 over gloo (127.0.0.1).

Each rank owns half of every layer's experts, computes the SwiGLU output of
the routed experts it owns into a (top_k, d) slot buffer (zero elsewhere),
sum-exchanges it, and applies the reference-ordered combine.  The result
must equal the single-process moe_forward (model.py:238-254) bit for bit,
because exactly one rank contributes each slot and x + 0 is exact.
"""

import os
import socket

import numpy as np
import pytest

from paper_2312_17238_b200.expert_parallel import (rank_budget, owned_experts, owned_keys,
                                                   owned_mask, owner_of)


def test_partition_covers_every_expert_once():
    for E in (8, 16):
        for N in (1, 2, 4, 8):
            seen = []
            for r in range(N):
                seen += owned_experts(E, r, N)
                assert owned_mask(3, E, r, N).sum() == 3 * len(owned_experts(E, r, N))
            assert sorted(seen) == list(range(E))
            assert all(owner_of(e, E, N) in range(N) for e in range(E))
    assert owned_keys(2, 8, 1, 2) == {(l, e) for l in range(2) for e in (4, 5, 6, 7)}
    # the node-wide budget is split, never exceeded: sum over ranks == k (and b)
    for world in (1, 2, 4, 8):
        for k, b, m in ((4, 4, 0), (2, 4, 2), (0, 4, 2), (8, 4, 1)):
            rb = [rank_budget(k, b, m, 8, r, world) for r in range(world)]
            assert sum(x[0] for x in rb) == min(k, 8) and sum(x[1] for x in rb) == b
            assert all(x[2] <= x[1] and x[2] <= m for x in rb)
    assert rank_budget(4, 4, 0, 8, 0, 8) == (1, 1, 0) and rank_budget(4, 4, 0, 8, 7, 8) == (0, 0, 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import model as OM
    from paper_2312_17238_b200.expert_parallel import combine, owned_experts, slot_exchange
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        cfg = OM.ModelConfig(vocab_size=32, d_model=64, n_layers=2, n_heads=2, d_ffn=96,
                             n_experts=8)
        m = OM.Model(cfg, OM.init_params(cfg))
        rng = np.random.default_rng(0)          # same h on every rank (replicated dense path)
        mine = set(owned_experts(cfg.n_experts, rank, world))
        results = []
        for layer in range(cfg.n_layers):
            for _ in range(5):
                h = rng.normal(size=cfg.d_model).astype(np.float32)
                out = OM.gate(m, layer, h)
                slots = np.zeros((len(out.experts), cfg.d_model), np.float32)
                for j, e in enumerate(out.experts):
                    if e in mine:
                        slots[j] = OM.swiglu(*m.expert(layer, e), h)

                def ar(buf):
                    t = torch.from_numpy(buf)
                    dist.all_reduce(t, op=dist.ReduceOp.SUM)

                y = combine(h, out.weights, slot_exchange(slots, ar))
                ref = OM.moe_forward(h, out, [m.expert(layer, e) for e in out.experts])
                results.append(bool(np.array_equal(y, ref)))
        q.put((rank, all(results), len(results)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_slot_exchange_is_exact_world2():
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, _, _ in out) == [0, 1]
    assert all(ok for _, ok, _ in out), out
    assert all(n == 10 for _, _, n in out)


def _nccl_worker(rank, world, port, q):
    import torch
    import torch.distributed as dist

    from oracle import model as OM
    from paper_2312_17238_b200.expert_parallel import (gather_combine, owned_experts,
                                                       share_nccl_id)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        # the NCCL transport's id exchange: every rank ends up with rank 0's id
        uid = share_nccl_id()
        ids = [None] * world
        dist.all_gather_object(ids, uid)
        same_id = len(uid) == 128 and all(i == ids[0] for i in ids)
        # its exchange: an all-gather of the slot buffers ([N][top_k][d],
        # rank-major, like ncclAllGather) summed in rank order by the combine
        cfg = OM.ModelConfig(vocab_size=32, d_model=64, n_layers=2, n_heads=2, d_ffn=96,
                             n_experts=8)
        m = OM.Model(cfg, OM.init_params(cfg))
        rng = np.random.default_rng(1)
        mine = set(owned_experts(cfg.n_experts, rank, world))
        ok = []
        for layer in range(cfg.n_layers):
            for _ in range(5):
                h = rng.normal(size=cfg.d_model).astype(np.float32)
                out = OM.gate(m, layer, h)
                slots = np.zeros((len(out.experts), cfg.d_model), np.float32)
                for j, e in enumerate(out.experts):
                    if e in mine:
                        slots[j] = OM.swiglu(*m.expert(layer, e), h)
                parts = [torch.zeros(slots.shape, dtype=torch.float32) for _ in range(world)]
                dist.all_gather(parts, torch.from_numpy(slots))
                y = gather_combine(h, out.weights, np.stack([p.numpy() for p in parts]))
                ref = OM.moe_forward(h, out, [m.expert(layer, e) for e in out.experts])
                ok.append(bool(np.array_equal(y, ref)))
        q.put((rank, same_id, all(ok), len(ok)))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_nccl_transport_id_and_gather_combine_world2():
    """Host side of the NCCL transport (moe_ep_connect_nccl) on CPU: the
    unique-id broadcast and the rank-major all-gather combine are exact."""
    import torch.multiprocessing as mp
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_nccl_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    out = [q.get(timeout=240) for _ in procs]
    for p in procs:
        p.join(timeout=60)
    assert sorted(r for r, *_ in out) == [0, 1]
    assert all(same for _, same, _, _ in out), out
    assert all(ok for _, _, ok, _ in out), out
    assert all(n == 10 for *_, n in out)


def test_transport_choice(monkeypatch):
    from paper_2312_17238_b200.expert_parallel import transport_of
    monkeypatch.delenv("MOE_EP_TRANSPORT", raising=False)
    assert transport_of() == "ipc" and transport_of("NCCL") == "nccl"
    monkeypatch.setenv("MOE_EP_TRANSPORT", "nccl")
    assert transport_of() == "nccl" and transport_of("ipc") == "ipc"
    with pytest.raises(ValueError):
        transport_of("mpi")
