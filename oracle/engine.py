"""Oracle restatement of the session / offload / replay flow (TEST INFRASTRUCTURE ONLY).

Follows ``/root/reference/pkg/src/moe_offload/engine.py``:
  * SpeculationConfig ................ engine.py:43-57
  * guess_experts .................... engine.py:60-68
  * materialize / payload bytes ...... engine.py:71-82
  * _Session prefill/run_token/decode  engine.py:97-182
  * DenseRunner ...................... engine.py:185-197
  * OffloadEngine resolve hooks ...... engine.py:200-247
  * replay / guess_recall ............ engine.py:263-338

Payloads are ``(w_gate_proj, w_up_proj, w_down_proj)`` triples whose members are
either float32 arrays or quantized blocks (dequantized on every acquire, like
the reference's ``materialize``).  ``build_mixed_quant`` produces the
mixed-precision model of BASELINE configs 2/3 from a float parameter dict.
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import model as M
from . import quant as Q
from .store import ACQUIRE_KINDS, CacheConfig, ExpertStore, recall


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


def guess_experts(model, h, target_layer: int, m: int):
    """Top-m of the target layer's gate on the current h (engine.py:60-68)."""
    if target_layer >= model.config.n_layers:
        return []
    return [(target_layer, int(e)) for e in M.top_k(h @ model.gate_matrix(target_layer), m)]


def materialize(payload):
    return tuple(Q.dequantize(w) if hasattr(w, "packed_codes") else w for w in payload)


def payload_bytes(payload) -> int:
    """H2D bytes of one expert (engine.py:79-82 + quant.py:332-343)."""
    return int(sum(Q.payload_nbytes(w) if hasattr(w, "packed_codes") else w.nbytes
                   for w in payload))


def dense_payloads(model):
    return {(l, e): model.expert(l, e) for l in range(model.config.n_layers)
            for e in range(model.config.n_experts)}


@dataclass
class TraceRec:
    token_pos: int
    layer: int
    experts: tuple
    weights: np.ndarray
    hidden: np.ndarray | None


class Session:
    """Shared flow (engine.py:97-182); subclasses resolve experts."""

    def __init__(self, model, record_hidden: bool = True):
        self.model = model
        self.record_hidden = record_hidden
        self.reset_session()

    def reset_session(self):
        self.kv = M.KVCache(self.model.config)
        self.pos = 0
        self.last_logits = None
        self.records: list[TraceRec] = []
        self.prompt_len = 0

    def _on_gate(self, layer, out, h):
        self.records.append(TraceRec(out.token_pos, layer, out.experts, out.weights.copy(),
                                     h.astype(np.float32).copy() if self.record_hidden else None))

    def sorted_records(self):
        return sorted(self.records, key=lambda r: (r.token_pos, r.layer))

    def prefill(self, tokens):
        self.reset_session()
        logits = M.prefill_pass(self.model, list(tokens), self.kv, self._resolve_layer,
                                on_gate=self._on_gate)
        self.pos = self.prompt_len = len(tokens)
        self.last_logits = logits[-1]
        return logits

    def run_token(self, token: int):
        if self.last_logits is None:
            raise RuntimeError("prefill must run before decoding")
        logits = M.forward_token(self.model, token, self.pos, self.kv, self._resolve_token,
                                 on_gate=self._on_gate)
        self.pos += 1
        self.last_logits = logits
        return logits

    def decode(self, n: int, sampler="greedy", sampler_seed: int = 0):
        if n < 1:
            raise ValueError("n_tokens must be >= 1")
        if isinstance(sampler, str):
            sampler = M.make_sampler(sampler, sampler_seed)
        logits = self.last_logits
        if logits is None:
            raise RuntimeError("prefill must run before decoding")
        toks = []
        for _ in range(n):
            t = sampler(logits)
            toks.append(t)
            logits = self.run_token(t)
        return toks, logits


class DenseRunner(Session):
    """No-store reference path (engine.py:185-197)."""

    def _resolve_token(self, layer, out, h):
        return [self.model.expert(layer, e) for e in out.experts]

    def _resolve_layer(self, layer, outs):
        return {(layer, e): self.model.expert(layer, e) for o in outs for e in o.experts}


class OffloadEngine(Session):
    """Tiered store + optional speculation (engine.py:200-247)."""

    def __init__(self, model, cache: CacheConfig | None = None,
                 speculation: SpeculationConfig = SpeculationConfig(), payloads=None,
                 record_hidden: bool = True, owned=None):
        self.payloads = dense_payloads(model) if payloads is None else dict(payloads)
        nbytes = payload_bytes(next(iter(self.payloads.values())))
        if cache is None:
            cache = CacheConfig(k=2, b=4, expert_bytes=nbytes)
        elif cache.expert_bytes == 1:
            cache = CacheConfig(k=cache.k, b=cache.b, expert_bytes=nbytes)
        if speculation.enabled and speculation.m > cache.b:
            raise ValueError(f"m={speculation.m} exceeds b={cache.b} staging buffers")
        self.speculation = speculation
        self.store = ExpertStore(model.config.n_layers, model.config.n_experts, cache, owned)
        super().__init__(model, record_hidden)

    def _resolve_token(self, layer, out, h):
        pos = out.token_pos
        for e in out.experts:
            self.store.acquire(layer, e, pos)
        sp = self.speculation
        if sp.enabled and sp.m > 0:
            g = guess_experts(self.model, h, layer + sp.lookahead, sp.m)
            if g:
                self.store.speculative_load(g, pos, current_layer=layer)
        return [materialize(self.payloads[(layer, e)]) for e in out.experts]

    def _resolve_layer(self, layer, outs):
        table = {}
        for o in outs:
            for e in o.experts:
                if (layer, e) not in table:
                    self.store.acquire(layer, e, o.token_pos)
                    table[(layer, e)] = materialize(self.payloads[(layer, e)])
        return table

    @property
    def events(self):
        return self.store.events

    def recall(self, definition="device_or_staging"):
        return recall(self.store.events, definition)


def replay(records, n_layers, n_experts, prompt_len, cache: CacheConfig,
           speculation: SpeculationConfig = SpeculationConfig(), gates=None):
    """Model-free store replay from (token_pos, layer, experts, hidden) records
    (engine.py:263-313)."""
    st = ExpertStore(n_layers, n_experts, cache)
    by_tok = {}
    for r in records:
        by_tok.setdefault(r.token_pos, []).append(r)
    toks = sorted(by_tok)
    for l in range(n_layers):
        seen = set()
        for t in (t for t in toks if t < prompt_len):
            rec = next(r for r in by_tok[t] if r.layer == l)
            for e in rec.experts:
                if e not in seen:
                    st.acquire(l, e, t)
                    seen.add(e)
    for t in (t for t in toks if t >= prompt_len):
        for rec in sorted(by_tok[t], key=lambda r: r.layer):
            for e in rec.experts:
                st.acquire(rec.layer, e, t)
            if speculation.enabled and speculation.m > 0:
                tgt = rec.layer + speculation.lookahead
                if tgt < n_layers:
                    g = M.top_k(rec.hidden @ gates[tgt], speculation.m)
                    st.speculative_load([(tgt, int(e)) for e in g], t, current_layer=rec.layer)
    return st.events


# --------------------------------------------------------- mixed-quant build

def build_mixed_quant(params: dict, cfg, attn_bits: int = 4, expert_bits: int = 2):
    """Mixed-precision model of BASELINE configs 2/3: attention projections are
    group-quantized (the float model holds their dequantized values), experts
    are quantized payloads, and embeddings / lm_head / gates are fp16
    passthrough (quant.py:428 REQUIRED_FP16_ROLES; norms stay 1/0).

    Returns (fake-quant params, expert payloads, attention blocks).
    """
    fq = dict(params)
    for nm in ("wte", "wpe", "lm_head"):
        fq[nm] = params[nm].astype(np.float16).astype(np.float32)
    attn_blocks = {}
    payloads = {}
    for l in range(cfg.n_layers):
        pre = f"layers.{l}"
        fq[f"{pre}.gate"] = params[f"{pre}.gate"].astype(np.float16).astype(np.float32)
        for nm in ("wq", "wk", "wv", "wo"):
            key = f"{pre}.attn.{nm}"
            if attn_bits == 32:
                continue
            blk = Q.encode(params[key], Q.PRESETS[attn_bits])
            attn_blocks[key] = blk
            fq[key] = Q.dequantize(blk)
        for e in range(cfg.n_experts):
            eb = f"{pre}.experts.{e}"
            trip = tuple(Q.encode(params[f"{eb}.{nm}"], Q.PRESETS[expert_bits])
                         for nm in ("w_gate_proj", "w_up_proj", "w_down_proj"))
            payloads[(l, e)] = trip
            deq = materialize(trip)
            for nm, w in zip(("w_gate_proj", "w_up_proj", "w_down_proj"), deq):
                fq[f"{eb}.{nm}"] = w
    return fq, payloads, attn_blocks
