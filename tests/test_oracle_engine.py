"""Pins the oracle's decode flow to the reference OffloadEngine (CPU).

tests/golden/engine_golden.npz holds greedy tokens, logits, store event logs
and trace records of the unmodified reference engine on the C1 family
(BASELINE configs[0]: d=256, 2 layers, 8 experts top-2) in six cache /
speculation / quantization geometries.  The oracle must reproduce tokens,
routing and events exactly and the float outputs bit for bit (same numpy ops
in the same order).
"""

import numpy as np
import pytest

from oracle import engine as OE
from oracle import model as OM
from oracle.store import KINDS, CacheConfig
from tests.conftest import make_prompt


def ev_rows(events):
    return [[sq, KINDS.index(k), l, e, p, b] for sq, k, l, e, p, b in events]


@pytest.mark.parametrize("case", range(6))
def test_oracle_engine_matches_reference(case, engine_golden, c1_models):
    data, meta = engine_golden
    name, q, k, b, m, ntok = meta["cases"][case]
    cfg, get = c1_models
    model, pay, _ = get(tuple(q) if q else None)
    eng = OE.OffloadEngine(model, CacheConfig(k, b), OE.SpeculationConfig(m > 0, max(m, 1)),
                           payloads=pay, record_hidden=True)
    pre = eng.prefill([int(t) for t in data["prompt"]])
    np.testing.assert_array_equal(pre, data[f"{name}/prefill_logits"])
    toks, logits = eng.decode(ntok)
    assert toks == [int(t) for t in data[f"{name}/tokens"]]
    np.testing.assert_array_equal(logits, data[f"{name}/final_logits"])
    assert ev_rows(eng.events) == data[f"{name}/events"].tolist()
    recs = eng.sorted_records()
    meta_arr = np.array([[r.token_pos, r.layer, *r.experts] for r in recs], np.int32)
    np.testing.assert_array_equal(meta_arr, data[f"{name}/rec_meta"])
    np.testing.assert_array_equal(np.array([r.weights for r in recs]), data[f"{name}/rec_w"])
    np.testing.assert_array_equal(np.array([r.hidden for r in recs]), data[f"{name}/rec_h"])
    assert eng.recall() == float(data[f"{name}/recall"])


def test_offload_equals_dense_runner_bitwise(c1_models):
    """Mixed-quant payloads dequantized on acquire == fake-quant dense model."""
    cfg, get = c1_models
    model, pay, _ = get((4, 2))
    prompt = make_prompt(5, 6, cfg.vocab_size)
    a = OE.OffloadEngine(model, CacheConfig(2, 4), OE.SpeculationConfig(True, 2), payloads=pay)
    a.prefill(prompt)
    ta, la = a.decode(10, "categorical", 7)
    d = OE.DenseRunner(model)
    d.prefill(prompt)
    td, ld = d.decode(10, "categorical", 7)
    assert ta == td and np.array_equal(la, ld)


def test_replay_reproduces_live_log(c1_models):
    """reference test_engine.py:208-217."""
    cfg, get = c1_models
    model, pay, _ = get((4, 2))
    gates = np.stack([model.params[f"layers.{l}.gate"] for l in range(cfg.n_layers)])
    for spec in (False, True):
        e = OE.OffloadEngine(model, CacheConfig(2, 4), OE.SpeculationConfig(spec, 2),
                             payloads=pay)
        e.prefill(make_prompt(1, 5, cfg.vocab_size))
        e.decode(8)
        ev = OE.replay(e.sorted_records(), cfg.n_layers, cfg.n_experts, e.prompt_len,
                       e.store.cfg, OE.SpeculationConfig(spec, 2), gates=gates)
        assert ev == e.events


def test_gate_known_answers():
    """reference test_model.py:72-85."""
    cfg = OM.ModelConfig(vocab_size=8, d_model=4, n_layers=1, n_heads=1, d_ffn=4, n_experts=4)
    p = OM.init_params(cfg)
    p["layers.0.gate"] = np.zeros((4, 4), np.float32)
    m = OM.Model(cfg, p)
    out = OM.gate(m, 0, np.ones(4, np.float32))
    assert out.experts == (0, 1) and np.allclose(out.weights, [0.5, 0.5])
    p["layers.0.gate"] = np.eye(4, dtype=np.float32)
    out = OM.gate(m, 0, np.array([1, 3, 2, -1], np.float32))
    assert out.experts == (1, 2)
    assert np.allclose(out.weights, [0.7310586, 0.2689414], atol=1e-6)
    with pytest.raises(OM.NonFiniteError):
        OM.gate(m, 0, np.array([np.inf, 0, 0, 0], np.float32))


def test_greedy_lowest_index_and_zero_experts_identity():
    assert OM.sample_greedy(np.array([1.0, 3.0, 3.0, 2.0])) == 1
    h = np.random.default_rng(0).normal(size=16).astype(np.float32)
    z = np.zeros((16, 8), np.float32), np.zeros((16, 8), np.float32), np.zeros((8, 16), np.float32)
    out = OM.GateOutcome(0, 0, (0, 1), np.array([0.6, 0.4], np.float32), None)
    assert np.array_equal(OM.moe_forward(h, out, [z, z]), h)


def test_session_errors(c1_models):
    cfg, get = c1_models
    model, _, _ = get(None)
    e = OE.OffloadEngine(model, CacheConfig(2, 4))
    with pytest.raises(RuntimeError):
        e.decode(1)
    with pytest.raises(ValueError):
        e.prefill([])
    with pytest.raises(ValueError):
        e.prefill([cfg.vocab_size])
    with pytest.raises(ValueError):
        OE.OffloadEngine(model, CacheConfig(2, 1), OE.SpeculationConfig(True, 2))


def test_synth_tensor_statistics_and_determinism():
    """The counter-hash weight source used at Mixtral shape: deterministic,
    zero-mean, the requested std, integer-exact (so the device matches)."""
    a = OM.synth_tensor(0, 1017, (4096, 64), 1 / 64)
    b = OM.synth_tensor(0, 1017, (4096, 64), 1 / 64)
    assert np.array_equal(a, b)
    assert abs(float(a.mean())) < 1e-3 / 64 * 10
    assert float(a.std()) == pytest.approx(1 / 64, rel=0.02)
    part = OM.synth_tensor(0, 1017, (4096, 64), 1 / 64, offset=1000, count=77)
    assert np.array_equal(part, a.reshape(-1)[1000:1077])
    assert not np.array_equal(a, OM.synth_tensor(1, 1017, (4096, 64), 1 / 64))
