"""Oracle restatement of the two-tier expert store (TEST INFRASTRUCTURE ONLY).

Follows ``/root/reference/pkg/src/moe_offload/store.py``:
  * event kinds ............................. store.py:22-32
  * CacheConfig ............................. store.py:46-56
  * acquire (hit / staging hit + promote /
    miss + LRU eviction) .................... store.py:148-186
  * speculative_load (free slot, else the
    oldest slot not of the current layer) ... store.py:188-220
  * recall .................................. store.py:223-240
  * audit ................................... store.py:114-125

Payloads are opaque; the store only keeps keys.  Events are plain tuples
``(seq, kind, layer, expert, token_pos, bytes_moved)`` so they compare directly
with both the reference ``StoreEvent`` and the B200 engine's event records.
"""

from __future__ import annotations

from dataclasses import dataclass

HIT = "hit"
STAGING_HIT = "staging_hit"
MISS_LOAD = "miss_load"
EVICT_TO_HOST = "evict_to_host"
SPECULATIVE_LOAD = "speculative_load"
PROMOTE_FROM_STAGING = "promote_from_staging"
ACQUIRE_KINDS = (HIT, STAGING_HIT, MISS_LOAD)
KINDS = (HIT, STAGING_HIT, MISS_LOAD, EVICT_TO_HOST, SPECULATIVE_LOAD, PROMOTE_FROM_STAGING)


class UnknownExpertError(KeyError):
    pass


@dataclass(frozen=True)
class CacheConfig:
    k: int
    b: int = 4
    expert_bytes: int = 1

    def __post_init__(self):
        if self.k < 0 or self.b < 0 or self.expert_bytes <= 0:
            raise ValueError("k and b must be >= 0 and expert_bytes positive")


class ExpertStore:
    """Per-layer MRU-first LRU lists (<= k) plus ``b`` shared staging slots."""

    def __init__(self, n_layers: int, n_experts: int, cfg: CacheConfig, owned=None):
        if cfg.k > n_experts:
            raise ValueError(f"k={cfg.k} exceeds experts per layer ({n_experts})")
        self.L, self.E, self.cfg = n_layers, n_experts, cfg
        self.owned = None if owned is None else set(owned)
        self.lru = [[] for _ in range(n_layers)]
        self.stage = [None] * cfg.b          # (layer, expert, stamp) or None
        self.stamp = 0
        self.seq = 0
        self.events: list[tuple] = []

    # -- helpers
    def _emit(self, kind, layer, expert, pos, moved):
        self.events.append((self.seq, kind, layer, expert, pos,
                            self.cfg.expert_bytes if moved else 0))
        self.seq += 1

    def _check(self, layer, expert):
        if not (0 <= layer < self.L and 0 <= expert < self.E) or (
                self.owned is not None and (layer, expert) not in self.owned):
            raise UnknownExpertError(f"no such expert: layer={layer} expert={expert}")

    def _staged_at(self, layer, expert):
        for i, s in enumerate(self.stage):
            if s is not None and s[0] == layer and s[1] == expert:
                return i
        return None

    def _make_resident(self, layer, expert, pos):
        lst = self.lru[layer]
        lst.insert(0, expert)
        if len(lst) > self.cfg.k:
            self._emit(EVICT_TO_HOST, layer, lst.pop(), pos, True)

    # -- operations
    def acquire(self, layer: int, expert: int, pos: int) -> str:
        self._check(layer, expert)
        lst = self.lru[layer]
        if expert in lst:
            lst.remove(expert)
            lst.insert(0, expert)
            self._emit(HIT, layer, expert, pos, False)
            return HIT
        i = self._staged_at(layer, expert)
        if i is not None:
            self._emit(STAGING_HIT, layer, expert, pos, False)
            self.stage[i] = None
            if self.cfg.k > 0:
                self._emit(PROMOTE_FROM_STAGING, layer, expert, pos, False)
                self._make_resident(layer, expert, pos)
            return STAGING_HIT
        self._emit(MISS_LOAD, layer, expert, pos, True)
        if self.cfg.k > 0:
            self._make_resident(layer, expert, pos)
        return MISS_LOAD

    def speculative_load(self, keys, pos: int, current_layer=None) -> int:
        keys = list(keys)
        for (l, e) in keys:
            self._check(l, e)
        if len(keys) > self.cfg.b:
            raise ValueError(f"{len(keys)} speculative keys exceed b={self.cfg.b} buffers")
        if len({l for l, _ in keys}) > 1:
            raise ValueError("speculative keys must target a single layer")
        n = 0
        for (l, e) in keys:
            if e in self.lru[l] or self._staged_at(l, e) is not None:
                continue
            slot = next((i for i, s in enumerate(self.stage) if s is None), None)
            if slot is None:
                cands = [(s[2], i) for i, s in enumerate(self.stage)
                         if current_layer is None or s[0] != current_layer]
                if not cands:
                    continue
                slot = min(cands)[1]
            self.stage[slot] = (l, e, self.stamp)
            self.stamp += 1
            self._emit(SPECULATIVE_LOAD, l, e, pos, True)
            n += 1
        return n

    def device_state(self):
        return {l: tuple(v) for l, v in enumerate(self.lru)}

    def staged_keys(self):
        return tuple((s[0], s[1]) for s in self.stage if s is not None)

    def audit(self):
        seen = set()
        for l, lst in enumerate(self.lru):
            if len(lst) > self.cfg.k:
                raise AssertionError(f"layer {l} holds {len(lst)} > k experts")
            for e in lst:
                if (l, e) in seen:
                    raise AssertionError("duplicate resident")
                seen.add((l, e))
        if sum(s is not None for s in self.stage) > self.cfg.b:
            raise AssertionError("staging overflow")


def recall(events, definition: str = "device_or_staging") -> float:
    """(hits [+ staging hits]) / acquires (store.py:223-240)."""
    if definition not in ("device_only", "device_or_staging"):
        raise ValueError(f"unknown recall definition {definition!r}")
    tot = hit = 0
    for ev in events:
        kind = ev[1]
        if kind not in ACQUIRE_KINDS:
            continue
        tot += 1
        if kind == HIT or (kind == STAGING_HIT and definition == "device_or_staging"):
            hit += 1
    if tot == 0:
        raise ValueError("no acquire events in log")
    return hit / tot
