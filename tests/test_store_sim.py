"""The engine's device store code (csrc/store_dev.cuh), executed on the host,
against the oracle store and the reference's golden event logs (CPU).

Same functions the k_tail / k_prefill_bk kernels run, so this pins the
product bookkeeping — event grammar, LRU order, staging replacement, seq
numbering — without a GPU, and checks the physical buffer invariants the
reference never has to care about (k < top_k, k = 0 transients, staging
slot recycling within one layer).
"""

import json
import os

import numpy as np
import pytest

from oracle.store import KINDS, CacheConfig as OCache, ExpertStore
from paper_2312_17238_b200.api import CacheConfig
from paper_2312_17238_b200.store_sim import DeviceStoreSim

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def rows(events):
    return [[e.seq, KINDS.index(e.kind), e.key.layer, e.key.expert, e.token_pos, e.bytes_moved]
            for e in events]


def orows(events):
    return [[sq, KINDS.index(k), l, e, p, b] for sq, k, l, e, p, b in events]


@pytest.mark.parametrize("i", range(6))
def test_device_store_matches_reference_golden(i):
    with open(os.path.join(GOLDEN, "store_golden.json")) as fh:
        c = json.load(fh)[i]
    s = DeviceStoreSim(c["L"], c["E"], CacheConfig(c["k"], c["b"], 64), top_k=1, m=2)
    for op in c["ops"]:
        if op[0] == "spec":
            _, pos, cur, keys = op
            tgt = keys[0][0]
            s.resolve_token(cur, pos, [], [k[1] for k in keys], tgt)
        else:
            _, pos, l, e = op
            buf = s.resolve_token(l, pos, [e])
            assert s.buffers()["content"][buf[0]] == l * c["E"] + e
        s.audit()
    assert rows(s.events) == c["events"]
    assert {str(l): [k.expert for k in v] for l, v in s.device_state().items()} == \
        c["device_state"]
    assert [list(k) for k in s.staged_keys()] == c["staged"]


GEOMS = [(k, b, m) for k in (0, 1, 2, 4, 8) for b in (0, 1, 2, 4) for m in (0, 1, 2) if m <= b]


@pytest.mark.parametrize("k,b,m", GEOMS)
def test_decode_sequences_match_oracle_and_buffers_hold_keys(k, b, m):
    L, E, T = 4, 8, 40
    rng = np.random.default_rng(1000 * k + 10 * b + m)
    sim = DeviceStoreSim(L, E, CacheConfig(k, b, 4096), top_k=2, m=m)
    ref = ExpertStore(L, E, OCache(k, b, 4096))
    for pos in range(T):
        for l in range(L):
            ex = [int(x) for x in rng.choice(E, 2, replace=False)]
            g = [int(x) for x in rng.choice(E, m, replace=False)] if m else []
            gl = l + 1 if (m and l + 1 < L) else -1
            bufs = sim.resolve_token(l, pos, ex, g if gl >= 0 else [], gl)
            for e in ex:
                ref.acquire(l, e, pos)
            if gl >= 0:
                ref.speculative_load([(gl, x) for x in g], pos, current_layer=l)
            content = sim.buffers()["content"]
            for e, bf in zip(ex, bufs):      # the routed buffer holds the routed expert
                assert content[bf] == l * E + e
            assert len(set(bufs.tolist())) == 2
    assert rows(sim.events) == orows(ref.events)
    assert {l: tuple(x.expert for x in v) for l, v in sim.device_state().items()} == \
        ref.device_state()
    assert tuple(tuple(x) for x in sim.staged_keys()) == ref.staged_keys()
    sim.audit()
    n_loads = sum(1 for e in ref.events if e[1] in ("miss_load", "speculative_load"))
    assert sim.copies == n_loads  # one H2D copy per MISS_LOAD / SPECULATIVE_LOAD, none per evict


@pytest.mark.parametrize("k", [0, 1, 2, 8])
def test_prefill_dedupe_matches_oracle(k):
    L, E, n = 3, 8, 17
    rng = np.random.default_rng(k)
    sim = DeviceStoreSim(L, E, CacheConfig(k, 4, 64), top_k=2)
    ref = ExpertStore(L, E, OCache(k, 4, 64))
    for l in range(L):
        ex = np.stack([rng.choice(E, 2, replace=False) for _ in range(n)]).astype(np.int32)
        bufs = sim.resolve_prefill(l, ex)
        seen = set()
        for p in range(n):
            for e in ex[p]:
                if int(e) not in seen:
                    ref.acquire(l, int(e), p)
                    seen.add(int(e))
        content = sim.buffers()["content"]
        for p in range(n):
            for j in range(2):
                assert content[bufs[p, j]] == l * E + ex[p, j]
    assert rows(sim.events) == orows(ref.events)


def test_unknown_expert_raises():
    from paper_2312_17238_b200 import UnknownExpertError
    sim = DeviceStoreSim(2, 8, CacheConfig(2, 4, 64))
    with pytest.raises(UnknownExpertError):
        sim.resolve_token(0, 0, [9])


def test_ep_rank_store_equals_oracle_on_owned_subset():
    """Expert parallel: each rank's store is the reference store over its owned
    keys; together the ranks resolve every routed expert once."""
    from paper_2312_17238_b200.expert_parallel import owned_keys
    L, E, N = 3, 8, 4
    rng = np.random.default_rng(7)
    ops = []
    for pos in range(30):
        for l in range(L):
            ops.append((l, pos, [int(x) for x in rng.choice(E, 2, replace=False)],
                        [int(x) for x in rng.choice(E, 2, replace=False)]))
    resolved = {}
    for r in range(N):
        own = owned_keys(L, E, r, N)
        sim = DeviceStoreSim(L, E, CacheConfig(1, 2, 64), top_k=2, m=2, owned=own)
        ref = ExpertStore(L, E, OCache(1, 2, 64), owned=own)
        for l, pos, ex, g in ops:
            gl = l + 1 if l + 1 < L else -1
            bufs = sim.resolve_token(l, pos, ex, g if gl >= 0 else [], gl)
            for e, bf in zip(ex, bufs):
                if (l, e) in own:
                    ref.acquire(l, e, pos)
                    assert bf >= 0
                    resolved[(l, pos, e)] = resolved.get((l, pos, e), 0) + 1
                else:
                    assert bf == -1
            if gl >= 0:
                keys = [(gl, x) for x in g if (gl, x) in own]
                if keys:
                    ref.speculative_load(keys, pos, current_layer=l)
        assert rows(sim.events) == orows(ref.events)
        sim.audit()
    assert len(resolved) == len(ops) * 2 and set(resolved.values()) == {1}


@pytest.mark.parametrize("k,b,m", [(0, 4, 2), (1, 2, 1), (2, 4, 2), (4, 4, 2), (2, 2, 2)])
@pytest.mark.parametrize("progress", [0, 1, 3])
def test_copy_engine_policy_never_deadlocks(k, b, m, progress):
    """The engine's copy scheduling (copy_sched.h: demand first, speculation
    newest-first, promotion on staging hits, stale-job dropping, chunked jobs)
    driven by the device store's real request stream: every routed buffer is
    eventually published with the right contents, whatever the copy progress
    between bookkeeping calls."""
    import ctypes as C

    from paper_2312_17238_b200 import _lib
    L, E, T = 4, 8, 30
    rng = np.random.default_rng(17 * k + 5 * b + m + progress)
    sim = DeviceStoreSim(L, E, CacheConfig(k, b, 4096), top_k=2, m=m)
    assert _lib.lib().moe_store_sim_copy_policy(sim._h, 4096, 1024, progress) == 0
    ref = ExpertStore(L, E, OCache(k, b, 4096))
    for pos in range(T):
        for l in range(L):
            ex = [int(x) for x in rng.choice(E, 2, replace=False)]
            g = [int(x) for x in rng.choice(E, m, replace=False)]
            gl = l + 1 if l + 1 < L else -1
            bufs = sim.resolve_token(l, pos, ex, g if gl >= 0 else [], gl)
            for e in ex:
                ref.acquire(l, e, pos)
            if gl >= 0:
                ref.speculative_load([(gl, x) for x in g], pos, current_layer=l)
            content = sim.buffers()["content"]
            for e, bf in zip(ex, bufs):
                assert content[bf] == l * E + e
    assert rows(sim.events) == orows(ref.events)
    chunks = _lib.lib().moe_store_sim_chunks(sim._h)
    assert chunks <= 4 * sim.copies  # stale speculative jobs may be dropped, never duplicated


def test_trace_replay_through_device_store_equals_reference_replay():
    """§8(f)2: the reference ``replay`` of a recorded trace (engine.py:263-313)
    and the same trace driven through the engine's device store code
    (store_sim.replay_device) give identical event logs over a k x m grid,
    speculation re-evaluated from the recorded hidden states."""
    from moe_offload.engine import OffloadEngine as RefEngine, SpeculationConfig, replay
    from moe_offload.model import build_model, toy_config
    from paper_2312_17238_b200.store_sim import replay_device
    cfg = toy_config(vocab_size=32, d_model=32, n_layers=4, n_heads=4, d_ffn=48, n_experts=8,
                     max_seq_len=128)
    model = build_model(cfg)
    eng = RefEngine(model, CacheConfig(k=2, b=4), SpeculationConfig(True, 2))
    prompt = [int(t) for t in np.random.default_rng(7).integers(0, 32, 6)]
    eng.prefill(prompt)
    eng.decode(20, sampler="categorical", sampler_seed=1)
    tr = eng.trace()
    for k in (0, 1, 2, 4, 8):
        for m in (0, 1, 2, 4):
            spec = SpeculationConfig(enabled=m > 0, m=max(m, 1))
            cache = CacheConfig(k=k, b=4, expert_bytes=eng.store.config.expert_bytes)
            ref = replay(tr, cache, spec).events
            dev = replay_device(tr, cache, spec).events
            assert dev == ref, (k, m)
    live = replay(tr, CacheConfig(k=2, b=4, expert_bytes=eng.store.config.expert_bytes),
                  SpeculationConfig(True, 2)).events
    assert live == eng.events


@pytest.mark.parametrize("k,b,m", [(1, 2, 1), (2, 4, 2), (0, 4, 2)])
def test_copy_engine_parks_passed_speculation(k, b, m):
    """copy_sched.h parking: with no copy progress between bookkeeping calls,
    speculative jobs whose target layer the decode has passed are parked
    (not copied further) -- every routed buffer is still published with the
    right contents (a staging hit promotes a parked job), the event log still
    equals the reference store's, and no more chunks are copied than without
    parking."""
    from paper_2312_17238_b200 import _lib
    L, E, T = 4, 8, 30
    chunks = {}
    for park in (1, 0):
        rng = np.random.default_rng(7 * k + b + m)
        sim = DeviceStoreSim(L, E, CacheConfig(k, b, 4096), top_k=2, m=m)
        lib = _lib.lib()
        assert lib.moe_store_sim_copy_policy(sim._h, 4096, 1024, 0) == 0
        assert lib.moe_store_sim_set_park(sim._h, park) == 0
        ref = ExpertStore(L, E, OCache(k, b, 4096))
        for pos in range(T):
            for l in range(L):
                ex = [int(x) for x in rng.choice(E, 2, replace=False)]
                g = [int(x) for x in rng.choice(E, m, replace=False)]
                gl = l + 1 if l + 1 < L else -1
                bufs = sim.resolve_token(l, pos, ex, g if gl >= 0 else [], gl)
                for e in ex:
                    ref.acquire(l, e, pos)
                if gl >= 0:
                    ref.speculative_load([(gl, x) for x in g], pos, current_layer=l)
                content = sim.buffers()["content"]
                for e, bf in zip(ex, bufs):
                    assert content[bf] == l * E + e
        assert rows(sim.events) == orows(ref.events)
        chunks[park] = (lib.moe_store_sim_chunks(sim._h), lib.moe_store_sim_parked(sim._h))
    assert chunks[1][1] > 0 and chunks[0][1] == 0
    assert chunks[1][0] <= chunks[0][0]
