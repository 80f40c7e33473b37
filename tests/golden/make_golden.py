"""Generate golden fixtures from the UNMODIFIED reference package.

Run in the build container (where /root/reference exists):
    python tests/golden/make_golden.py
The fixtures are committed; the GPU box never reads /root/reference.

Outputs (all small):
  quant_golden.npz   serialized blocks + dequantized values for seeded inputs
  store_golden.json  event logs of the reference TieredExpertStore on random
                     acquire / speculative_load sequences
  engine_golden.npz  greedy tokens, final logits, event logs and trace records
                     of the reference OffloadEngine on tiny (C1-family) configs,
                     fp32 and mixed-quant payloads, several cache geometries
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, REF)

from moe_offload import engine as RE  # noqa: E402
from moe_offload import model as RM  # noqa: E402
from moe_offload import quant as RQ  # noqa: E402
from moe_offload import store as RS  # noqa: E402

C1 = dict(vocab_size=512, d_model=256, n_layers=2, n_heads=2, d_ffn=896, n_experts=8,
          top_k_gate=2, seed=0, max_seq_len=256)

QUANT_CASES = [  # (scheme bits, shape, seed, scale)
    (2, (128, 128), 42, 1.0), (3, (64, 256), 1, 0.3), (4, (64, 1024), 2, 0.05),
    (2, (7, 33), 3, 2.0), (3, (5, 200), 4, 1.0), (4, (16, 100), 5, 10.0),
    (2, (256, 896), 6, 1 / 16), (3, (256, 896), 7, 1 / 16), (4, (256, 256), 8, 1 / 16),
    (2, (896, 256), 9, 1 / 30), (3, (896, 256), 10, 1 / 30),
]


def ev_rows(events):
    return [[e.seq, RS.EVENT_KINDS.index(e.kind), e.key.layer, e.key.expert, e.token_pos,
             e.bytes_moved] for e in events]


def make_quant():
    out = {}
    for i, (bits, shape, seed, scale) in enumerate(QUANT_CASES):
        w = (np.random.default_rng(seed).normal(size=shape) * scale).astype(np.float32)
        blk = RQ.quantize(w, RQ.PRESET_SCHEMES[bits])
        out[f"ser{i}"] = np.frombuffer(RQ.serialize_block(blk), np.uint8)
        out[f"deq_sha{i}"] = np.frombuffer(
            hashlib.sha256(RQ.dequantize(blk).astype("<f4").tobytes()).digest(), np.uint8)
        out[f"nbytes{i}"] = np.int64(RQ.payload_nbytes(blk))
    out["bits"] = np.array([c[0] for c in QUANT_CASES])
    np.savez_compressed(os.path.join(HERE, "quant_golden.npz"), **out)


def make_store():
    cases = []
    for seed, (L, E, k, b) in enumerate([(3, 8, 2, 4), (3, 8, 0, 4), (3, 8, 1, 2),
                                         (4, 8, 4, 3), (2, 8, 8, 4), (3, 8, 0, 0)]):
        rng = np.random.default_rng(100 + seed)
        payloads = {RS.ExpertKey(l, e): () for l in range(L) for e in range(E)}
        st = RS.TieredExpertStore(payloads, L, E, RS.CacheConfig(k=k, b=b, expert_bytes=64))
        ops = []
        for pos in range(300):
            l = int(rng.integers(L))
            if b and rng.random() < 0.4:
                tgt = (l + 1) % L
                m = int(rng.integers(1, min(b, 2) + 1))
                keys = [RS.ExpertKey(tgt, int(g)) for g in rng.choice(E, m, replace=False)]
                st.speculative_load(keys, pos, current_layer=l)
                ops.append(["spec", pos, l, [[kk.layer, kk.expert] for kk in keys]])
            e = int(rng.integers(E))
            st.acquire(RS.ExpertKey(l, e), pos)
            ops.append(["acq", pos, l, e])
        cases.append({"L": L, "E": E, "k": k, "b": b, "ops": ops, "events": ev_rows(st.events),
                      "device_state": {str(kk): [x.expert for x in v]
                                       for kk, v in st.device_state().items()},
                      "staged": [[x.layer, x.expert] for x in st.staged_keys()]})
    with open(os.path.join(HERE, "store_golden.json"), "w") as fh:
        json.dump(cases, fh)


class _QuantPayload:
    """The materialize/nbytes adapter the reference engine expects (SURVEY §0:
    no payload class exists in the reference)."""

    def __init__(self, blocks):
        self.blocks = blocks
        self.nbytes = sum(RQ.payload_nbytes(b) for b in blocks)

    def materialize(self, key):
        return RM.ExpertWeights(key, *[RQ.dequantize(b) for b in self.blocks])


def mixed_model(cfg, attn_bits, expert_bits):
    model = RM.build_model(cfg)
    p = dict(model.params)
    for nm in ("wte", "wpe", "lm_head"):
        p[nm] = p[nm].astype(np.float16).astype(np.float32)
    payloads = {}
    for l in range(cfg.n_layers):
        pre = f"layers.{l}"
        p[f"{pre}.gate"] = p[f"{pre}.gate"].astype(np.float16).astype(np.float32)
        for nm in ("wq", "wk", "wv", "wo"):
            p[f"{pre}.attn.{nm}"] = RQ.dequantize(RQ.quantize(p[f"{pre}.attn.{nm}"],
                                                              RQ.PRESET_SCHEMES[attn_bits]))
        for e in range(cfg.n_experts):
            eb = f"{pre}.experts.{e}"
            blocks = [RQ.quantize(p[f"{eb}.{nm}"], RQ.PRESET_SCHEMES[expert_bits])
                      for nm in ("w_gate_proj", "w_up_proj", "w_down_proj")]
            payloads[RS.ExpertKey(l, e)] = _QuantPayload(blocks)
            for nm, b in zip(("w_gate_proj", "w_up_proj", "w_down_proj"), blocks):
                p[f"{eb}.{nm}"] = RQ.dequantize(b)
    return RM.Model(cfg, p), payloads


ENGINE_CASES = [  # name, quant (attn,expert) or None, k, b, spec m (0=off), ntok
    ("fp32_k2_nospec", None, 2, 4, 0, 32),
    ("fp32_k2_m2", None, 2, 4, 2, 32),
    ("mq42_k2_m2", (4, 2), 2, 4, 2, 32),
    ("mq43_k4_nospec", (4, 3), 4, 4, 0, 32),
    ("mq42_k0_m2", (4, 2), 0, 4, 2, 24),
    ("mq42_k1_m1", (4, 2), 1, 2, 1, 24),
]


def make_engine():
    cfg = RM.ModelConfig(**C1)
    prompt = [int(t) for t in np.random.default_rng(0).integers(0, cfg.vocab_size, 8)]
    out = {"prompt": np.array(prompt, np.int32)}
    models = {}
    for name, q, k, b, m, ntok in ENGINE_CASES:
        if q not in models:
            models[q] = (RM.build_model(cfg), None) if q is None else mixed_model(cfg, *q)
        model, payloads = models[q]
        eng = RE.OffloadEngine(model, RS.CacheConfig(k=k, b=b),
                               RE.SpeculationConfig(enabled=m > 0, m=max(m, 1)),
                               payloads=payloads, record_hidden=True)
        pre_logits = eng.prefill(prompt)
        res = eng.decode(ntok, sampler="greedy")
        recs = res.trace.records
        out[f"{name}/tokens"] = np.array(res.tokens, np.int32)
        out[f"{name}/final_logits"] = res.final_logits.astype(np.float32)
        out[f"{name}/prefill_logits"] = pre_logits.astype(np.float32)
        out[f"{name}/events"] = np.array(ev_rows(eng.events), np.int64)
        out[f"{name}/rec_meta"] = np.array([[r.token_pos, r.layer, *r.experts] for r in recs],
                                           np.int32)
        out[f"{name}/rec_w"] = np.array([r.weights for r in recs], np.float32)
        out[f"{name}/rec_h"] = np.array([r.hidden for r in recs], np.float32)
        out[f"{name}/recall"] = np.float64(eng.recall())
        print(name, res.tokens[:6], len(eng.events), f"recall={eng.recall():.3f}")
    np.savez_compressed(os.path.join(HERE, "engine_golden.npz"), **out)
    with open(os.path.join(HERE, "engine_cases.json"), "w") as fh:
        json.dump({"config": C1, "cases": ENGINE_CASES}, fh)


if __name__ == "__main__":
    make_quant()
    make_store()
    make_engine()
