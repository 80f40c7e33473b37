"""Reference-compatible value types of the hot path's public API.

Same names, fields and validation as the reference package so that callers
and the reference's own analysis tools work unchanged:
  * ExpertKey / CacheConfig / StoreEvent / recall / events JSONL  (store.py:22-73, 223-265)
  * SpeculationConfig                                            (engine.py:43-57)
  * TraceRecord / Trace / config_digest                          (trace.py:33-98)
  * GenerationResult                                             (engine.py:90-94)
  * greedy / categorical samplers                                (model.py:374-401)
"""

from __future__ import annotations

import hashlib
import json
from dataclasses import dataclass, field
from typing import Iterable, NamedTuple

import numpy as np

from .errors import TraceFormatError

HIT = "hit"
STAGING_HIT = "staging_hit"
MISS_LOAD = "miss_load"
EVICT_TO_HOST = "evict_to_host"
SPECULATIVE_LOAD = "speculative_load"
PROMOTE_FROM_STAGING = "promote_from_staging"
EVENT_KINDS = (HIT, STAGING_HIT, MISS_LOAD, EVICT_TO_HOST, SPECULATIVE_LOAD, PROMOTE_FROM_STAGING)
ACQUIRE_KINDS = (HIT, STAGING_HIT, MISS_LOAD)
LOAD_KINDS = (MISS_LOAD, SPECULATIVE_LOAD)


class ExpertKey(NamedTuple):
    layer: int
    expert: int


@dataclass(frozen=True)
class CacheConfig:
    """k experts per layer on device, b shared staging buffers."""

    k: int
    b: int = 4
    expert_bytes: int = 1

    def __post_init__(self):
        if self.k < 0 or self.b < 0 or self.expert_bytes <= 0:
            raise ValueError("k and b must be >= 0 and expert_bytes positive")


@dataclass(frozen=True)
class StoreEvent:
    seq: int
    kind: str
    key: ExpertKey
    token_pos: int
    bytes_moved: int

    @property
    def layer(self) -> int:
        return self.key.layer

    @property
    def expert(self) -> int:
        return self.key.expert


def recall(events: Iterable[StoreEvent], definition: str = "device_or_staging") -> float:
    if definition not in ("device_only", "device_or_staging"):
        raise ValueError(f"unknown recall definition {definition!r}")
    total = hits = 0
    for ev in events:
        if ev.kind not in ACQUIRE_KINDS:
            continue
        total += 1
        if ev.kind == HIT or (ev.kind == STAGING_HIT and definition == "device_or_staging"):
            hits += 1
    if total == 0:
        raise ValueError("no acquire events in log")
    return hits / total


def events_to_jsonl(events: Iterable[StoreEvent]) -> str:
    rows = [json.dumps({"seq": e.seq, "kind": e.kind, "layer": e.key.layer,
                        "expert": e.key.expert, "token_pos": e.token_pos,
                        "bytes_moved": e.bytes_moved}, sort_keys=True, separators=(",", ":"))
            for e in events]
    return "\n".join(rows) + ("\n" if rows else "")


def events_from_jsonl(text: str) -> list[StoreEvent]:
    out = []
    for line in text.splitlines():
        if not line.strip():
            continue
        r = json.loads(line)
        if r["kind"] not in EVENT_KINDS:
            raise ValueError(f"unknown event kind {r['kind']!r}")
        out.append(StoreEvent(r["seq"], r["kind"], ExpertKey(r["layer"], r["expert"]),
                              r["token_pos"], r["bytes_moved"]))
    return out


@dataclass(frozen=True)
class SpeculationConfig:
    enabled: bool = False
    m: int = 2
    lookahead: int = 1

    def __post_init__(self):
        if self.m < 0:
            raise ValueError("m must be >= 0")
        if self.lookahead < 1:
            raise ValueError("lookahead must be >= 1")


def config_digest(config_dict: dict) -> str:
    blob = json.dumps(config_dict, sort_keys=True, separators=(",", ":"))
    return hashlib.sha256(blob.encode()).hexdigest()[:16]


@dataclass
class TraceRecord:
    token_pos: int
    layer: int
    experts: tuple
    weights: np.ndarray
    hidden: np.ndarray | None = None

    def __eq__(self, other):
        return (self.token_pos == other.token_pos and self.layer == other.layer
                and tuple(self.experts) == tuple(other.experts)
                and np.array_equal(self.weights, other.weights)
                and (self.hidden is None) == (other.hidden is None)
                and (self.hidden is None or np.array_equal(self.hidden, other.hidden)))


@dataclass
class Trace:
    config_digest: str
    n_layers: int
    n_experts: int
    top_k: int
    records_hidden: bool
    prompt_len: int = 0
    d_model: int | None = None
    gates: np.ndarray | None = None
    records: list = field(default_factory=list)

    def validate(self) -> None:
        keys = [(r.token_pos, r.layer) for r in self.records]
        if keys != sorted(keys):
            raise TraceFormatError("records must be sorted by (token_pos, layer)")
        if len(set(keys)) != len(keys):
            raise TraceFormatError("duplicate (token_pos, layer) record")
        for r in self.records:
            if len(r.experts) != self.top_k or len(set(r.experts)) != self.top_k:
                raise TraceFormatError("record must select top_k distinct experts")
            if any(not 0 <= e < self.n_experts for e in r.experts):
                raise TraceFormatError("expert index out of range")
            if r.layer >= self.n_layers:
                raise TraceFormatError("layer index out of range")
            if self.records_hidden and r.hidden is None:
                raise TraceFormatError("records_hidden is set but a record has no hidden state")
        if self.records_hidden:
            if self.gates is None or self.d_model is None:
                raise TraceFormatError("hidden-recording traces must embed gate matrices")
            if self.gates.shape != (self.n_layers, self.d_model, self.n_experts):
                raise TraceFormatError("gate matrix shape mismatch")

    def sort_records(self) -> None:
        self.records.sort(key=lambda r: (r.token_pos, r.layer))

    @property
    def n_tokens(self) -> int:
        return len({r.token_pos for r in self.records})

    def gate_logits(self, layer: int, hidden: np.ndarray) -> np.ndarray:
        if self.gates is None:
            raise TraceFormatError("trace has no gate matrices")
        return hidden @ self.gates[layer]


@dataclass
class GenerationResult:
    tokens: list
    final_logits: np.ndarray
    trace: Trace


def sample_greedy(logits: np.ndarray) -> int:
    return int(np.argmax(logits))


@dataclass
class CategoricalSampler:
    """numpy-stream categorical sampler (same RNG stream as the reference)."""

    seed: int
    _rng: np.random.Generator = field(init=False, repr=False)

    def __post_init__(self):
        self._rng = np.random.default_rng(self.seed)

    def __call__(self, logits: np.ndarray) -> int:
        z = logits.astype(np.float64)
        z -= z.max()
        p = np.exp(z)
        p /= p.sum()
        return int(self._rng.choice(p.size, p=p))


def make_sampler(name: str, seed: int = 0):
    if name == "greedy":
        return sample_greedy
    if name == "categorical":
        return CategoricalSampler(seed)
    raise ValueError(f"unknown sampler {name!r}")
