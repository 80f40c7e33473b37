"""Pins the oracle's expert store to the reference TieredExpertStore (CPU).

Golden event logs (tests/golden/store_golden.json) come from the unmodified
reference on random acquire / speculative_load sequences; the hand-computed
cases restate reference pkg/tests/test_store.py.
"""

import json
import os

import pytest
from hypothesis import given, settings
from hypothesis import strategies as st

from oracle.store import (EVICT_TO_HOST, HIT, KINDS, MISS_LOAD, PROMOTE_FROM_STAGING,
                          SPECULATIVE_LOAD, STAGING_HIT, CacheConfig, ExpertStore,
                          UnknownExpertError, recall)

GOLDEN = os.path.join(os.path.dirname(__file__), "golden")


def load_cases():
    with open(os.path.join(GOLDEN, "store_golden.json")) as fh:
        return json.load(fh)


def run_ops(store, ops):
    for op in ops:
        if op[0] == "spec":
            _, pos, cur, keys = op
            store.speculative_load([tuple(k) for k in keys], pos, current_layer=cur)
        else:
            _, pos, l, e = op
            store.acquire(l, e, pos)


@pytest.mark.parametrize("i", range(6))
def test_oracle_store_matches_reference_golden(i):
    c = load_cases()[i]
    s = ExpertStore(c["L"], c["E"], CacheConfig(c["k"], c["b"], 64))
    run_ops(s, c["ops"])
    got = [[sq, KINDS.index(k), l, e, p, b] for sq, k, l, e, p, b in s.events]
    assert got == c["events"]
    assert {str(l): list(v) for l, v in s.device_state().items()} == c["device_state"]
    assert [list(k) for k in s.staged_keys()] == c["staged"]
    s.audit()


def mk(k=2, b=4, L=2, E=8):
    return ExpertStore(L, E, CacheConfig(k, b, 64))


def test_hand_simulated_lru_sequence():
    """reference test_store.py:67-78."""
    s = mk(k=2)
    for pos, e in enumerate([3, 7, 3, 1, 7]):
        s.acquire(0, e, pos)
    assert [(ev[1], ev[3]) for ev in s.events] == [
        (MISS_LOAD, 3), (MISS_LOAD, 7), (HIT, 3), (MISS_LOAD, 1), (EVICT_TO_HOST, 7),
        (MISS_LOAD, 7), (EVICT_TO_HOST, 3)]


def test_staged_promotion_evicts_lru():
    """reference test_store.py:80-91."""
    s = mk(k=2)
    s.acquire(0, 0, 0)
    s.acquire(0, 1, 0)
    s.speculative_load([(0, 5)], 0)
    n = len(s.events)
    assert s.acquire(0, 5, 1) == STAGING_HIT
    assert [(ev[1], ev[3]) for ev in s.events[n:]] == [
        (STAGING_HIT, 5), (PROMOTE_FROM_STAGING, 5), (EVICT_TO_HOST, 0)]
    assert s.device_state()[0] == (5, 1)
    assert (0, 5) not in s.staged_keys()


def test_k0_b0_streaming():
    s = mk(k=0, b=0)
    for pos in range(3):
        assert s.acquire(0, 2, pos) == MISS_LOAD
    assert recall(s.events) == 0.0
    s.audit()


def test_bytes_moved_accounting():
    s = mk(k=1)
    for e in [0, 1, 0]:
        s.acquire(0, e, 0)
    for ev in s.events:
        assert ev[5] == (64 if ev[1] in (MISS_LOAD, EVICT_TO_HOST, SPECULATIVE_LOAD) else 0)
    seqs = [ev[0] for ev in s.events]
    assert seqs == sorted(seqs) and len(set(seqs)) == len(seqs)


def test_speculative_replacement_and_protection():
    """reference test_store.py:153-166: oldest unprotected slot is replaced;
    slots holding the current layer are protected."""
    s = mk(k=1, b=2, L=3)
    s.speculative_load([(1, 0)], 0, current_layer=0)
    s.speculative_load([(2, 1)], 0, current_layer=1)
    s.speculative_load([(2, 2)], 1, current_layer=0)   # replaces (1,0), the oldest
    assert set(s.staged_keys()) == {(2, 1), (2, 2)}
    n = len(s.events)
    s.speculative_load([(1, 3)], 2, current_layer=2)   # both slots hold layer 2: skip
    assert len(s.events) == n


def test_unknown_key_and_preconditions():
    s = mk()
    with pytest.raises(UnknownExpertError):
        s.acquire(0, 99, 0)
    with pytest.raises(ValueError):
        s.speculative_load([(1, 0), (1, 1), (1, 2), (1, 3), (1, 4)], 0)
    with pytest.raises(ValueError):
        s.speculative_load([(0, 1), (1, 1)], 0)
    with pytest.raises(ValueError):
        ExpertStore(2, 8, CacheConfig(9, 4, 64))


class ReferenceLRU:
    """Independent recency list (reference test_store.py:36-52)."""

    def __init__(self, k):
        self.k, self.order = k, []

    def access(self, item):
        if item in self.order:
            self.order.remove(item)
            self.order.insert(0, item)
            return True, None
        self.order.insert(0, item)
        if len(self.order) > self.k:
            return False, self.order.pop()
        return False, None


@settings(max_examples=50, deadline=None)
@given(k=st.sampled_from([0, 1, 2, 4, 8]),
       seq=st.lists(st.integers(0, 7), min_size=1, max_size=60))
def test_lru_matches_reference_lru(k, seq):
    """reference test_store.py:198-219."""
    s = mk(k=k, b=0, L=1)
    ref = ReferenceLRU(k)
    for pos, e in enumerate(seq):
        n = len(s.events)
        kind = s.acquire(0, e, pos)
        hit, ev = ref.access(e) if k else (False, None)
        assert (kind == HIT) == hit
        evicted = [x[3] for x in s.events[n:] if x[1] == EVICT_TO_HOST]
        assert evicted == ([] if ev is None else [ev])
        s.audit()
