"""GPU parity: the B200 engine vs the reference's golden outputs and the oracle.

Bit-exact: greedy tokens, routing (trace experts), store event logs.
Tolerance: logits and gate weights (fp32 summation order differs from numpy/
OpenBLAS): |d logits| <= 2e-3 * max|logits| + 1e-4, |d weights| <= 1e-4.
"""

import numpy as np
import pytest

from tests.conftest import make_prompt

pytestmark = pytest.mark.gpu

LOGIT_RTOL = 2e-3


def _engine(model, payloads, attn, k, b, m, record_hidden=True):
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig
    pay = None
    if payloads is not None:
        from paper_2312_17238_b200 import ExpertKey
        pay = {ExpertKey(*key): v for key, v in payloads.items()}
    return OffloadEngine(model, CacheConfig(k=k, b=b),
                         SpeculationConfig(enabled=m > 0, m=max(m, 1)), payloads=pay,
                         record_hidden=record_hidden, attn_blocks=attn)


def _ev_rows(events):
    from paper_2312_17238_b200 import EVENT_KINDS
    return [[e.seq, EVENT_KINDS.index(e.kind), e.key.layer, e.key.expert, e.token_pos,
             e.bytes_moved] for e in events]


def _close(a, b, rtol=LOGIT_RTOL):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    tol = rtol * np.abs(b).max() + 1e-4
    return float(np.abs(a - b).max()), tol


@pytest.mark.parametrize("case", range(6))
def test_engine_matches_reference_golden(case, engine_golden, c1_models):
    data, meta = engine_golden
    name, q, k, b, m, ntok = meta["cases"][case]
    q = tuple(q) if q else None
    cfg, get = c1_models
    model, payloads, attn = get(q)
    eng = _engine(model, payloads, attn, k, b, m)
    prompt = [int(t) for t in data["prompt"]]
    pre = eng.prefill(prompt)
    err, tol = _close(pre, data[f"{name}/prefill_logits"])
    assert err <= tol, f"prefill logits {err} > {tol}"
    res = eng.decode(ntok, sampler="greedy")
    assert res.tokens == [int(t) for t in data[f"{name}/tokens"]]
    err, tol = _close(res.final_logits, data[f"{name}/final_logits"])
    assert err <= tol, f"final logits {err} > {tol}"
    got = np.array(_ev_rows(eng.events), np.int64)
    np.testing.assert_array_equal(got, data[f"{name}/events"])
    recs = res.trace.records
    meta_arr = np.array([[r.token_pos, r.layer, *r.experts] for r in recs], np.int32)
    np.testing.assert_array_equal(meta_arr, data[f"{name}/rec_meta"])
    w = np.array([r.weights for r in recs], np.float32)
    assert np.abs(w - data[f"{name}/rec_w"]).max() < 1e-4
    hid = np.array([r.hidden for r in recs], np.float32)
    ref_h = data[f"{name}/rec_h"]
    assert np.abs(hid - ref_h).max() <= 1e-3 * np.abs(ref_h).max()
    assert eng.recall() == pytest.approx(float(data[f"{name}/recall"]))
    eng.close()


def test_device_quantizer_bit_exact():
    import ctypes as C

    from oracle import quant as OQ
    from paper_2312_17238_b200 import _lib
    L = _lib.lib()
    rng = np.random.default_rng(0)
    for bits, shape in [(2, (128, 128)), (3, (64, 256)), (4, (64, 1024)), (2, (256, 896)),
                        (3, (896, 256)), (4, (256, 256)), (2, (4096, 512)), (3, (32, 14336))]:
        w = (rng.normal(size=shape) / 16).astype(np.float32)
        sch = OQ.PRESETS[bits]
        ref = OQ.quantize(w, sch)
        n = w.size
        ng = n // sch.group_size
        codes = np.empty(n * bits // 8, np.uint8)
        zeros = np.empty(ng, np.uint8)
        nr = -(-ng // sch.scale_group_size)
        nsg = -(-ng // (sch.scale_group_size // sch.group_size))
        zs, zo, sc = np.empty(nr, np.uint16), np.empty(nr, np.uint16), np.empty(nsg, np.uint16)
        vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
        _lib.check(L.moe_quantize_device(w.ctypes.data_as(_lib.FP), shape[0], shape[1], bits,
                                         sch.group_size, sch.scale_group_size, vp(codes),
                                         vp(zeros), vp(zs), vp(zo), vp(sc)))
        assert codes.tobytes() == ref.packed_codes, (bits, shape)
        np.testing.assert_array_equal(zeros, ref.zeros)
        np.testing.assert_array_equal(zs, ref.zero_scales.view(np.uint16))
        np.testing.assert_array_equal(zo, ref.zero_offsets.view(np.uint16))
        np.testing.assert_array_equal(sc, ref.scales.view(np.uint16))


def test_device_synth_matches_oracle():
    from oracle import model as OM
    from paper_2312_17238_b200 import _lib
    L = _lib.lib()
    for tid, n, std in [(1, 10000, 0.02), (1017, 4096 * 64, 1 / 64), (1212, 99991, 1 / 119.7)]:
        ref = OM.synth_tensor(7, tid, (n,), std)
        out = np.empty(n, np.float32)
        _lib.check(L.moe_synth_tensor_device(7, tid, n, float(OM.synth_scale(std)),
                                             out.ctypes.data_as(_lib.FP)))
        np.testing.assert_array_equal(out, ref)


@pytest.mark.parametrize("bits,shape", [(2, (256, 896)), (3, (256, 896)), (4, (256, 256)),
                                        (2, (896, 256)), (3, (896, 256)), (2, (4096, 14336)),
                                        (3, (4096, 14336)), (2, (14336, 4096)),
                                        (3, (14336, 4096)), (4, (4096, 4096)), (16, (256, 512)),
                                        (32, (64, 96)), (16, (4096, 32000))])
def test_gemv_matches_dequantized_matmul(bits, shape):
    import ctypes as C

    from oracle import quant as OQ
    from paper_2312_17238_b200 import _lib
    from paper_2312_17238_b200.engine import _Marshal
    rng = np.random.default_rng(bits * 1000 + shape[0])
    w = (rng.normal(size=shape) / np.sqrt(shape[0])).astype(np.float32)
    x = rng.normal(size=shape[0]).astype(np.float32)
    if bits <= 4:
        blk = OQ.quantize(w, OQ.PRESETS[bits])
        wd = OQ.dequantize(blk)
        m = _Marshal().block(blk)
        mk = m
    else:
        wd = w.astype(np.float16).astype(np.float32) if bits == 16 else w
        mk = _Marshal()
        m = mk.dense(wd, allow_half=bits == 16)
    y = np.empty(shape[1], np.float32)
    _lib.check(_lib.lib().moe_gemv_device(C.byref(m), x.ctypes.data_as(_lib.FP),
                                          y.ctypes.data_as(_lib.FP)))
    ref = x.astype(np.float64) @ wd.astype(np.float64)
    scale = np.abs(x).astype(np.float64) @ np.abs(wd).astype(np.float64)
    rel = np.abs(y - ref) / (scale + 1e-30)
    assert rel.max() < 5e-6, rel.max()


def test_speculation_transparent_and_deterministic(c1_models):
    cfg, get = c1_models
    model, pay, attn = get((4, 2))
    prompt = make_prompt(2, 5, cfg.vocab_size)
    outs = []
    for m in (0, 2, 2):
        eng = _engine(model, pay, attn, 2, 4, m)
        eng.prefill(prompt)
        r = eng.decode(12, sampler="categorical", sampler_seed=7)
        outs.append((r.tokens, r.final_logits, [x.kind for x in eng.events]))
        eng.close()
    assert outs[0][0] == outs[1][0] == outs[2][0]
    assert np.array_equal(outs[0][1], outs[1][1])
    assert np.array_equal(outs[1][1], outs[2][1])
    assert outs[1][2] == outs[2][2]
    assert "speculative_load" in outs[1][2] and "speculative_load" not in outs[0][2]


def test_prefill_equals_teacher_forced_decode(c1_models):
    cfg, get = c1_models
    model, pay, attn = get((4, 3))
    toks = make_prompt(1, 6, cfg.vocab_size)
    a = _engine(model, pay, attn, 3, 4, 0)
    a.prefill(toks)
    b = _engine(model, pay, attn, 3, 4, 0)
    b.prefill(toks[:1])
    for t in toks[1:]:
        b.run_token(t)
    ra, rb = a.trace().records, b.trace().records
    assert len(ra) == len(rb)
    for x, y in zip(ra, rb):
        assert x.experts == y.experts
        assert np.array_equal(x.weights, y.weights)
        assert np.array_equal(x.hidden, y.hidden)


def test_replay_of_device_trace_reproduces_device_events(c1_models):
    from oracle import engine as OE
    from oracle.store import KINDS, CacheConfig
    cfg, get = c1_models
    model, pay, attn = get((4, 2))
    for spec in (False, True):
        eng = _engine(model, pay, attn, 2, 4, 2 if spec else 0)
        eng.prefill(make_prompt(4, 6, cfg.vocab_size))
        res = eng.decode(15, sampler="categorical", sampler_seed=3)
        gates = np.stack([model.params[f"layers.{l}.gate"] for l in range(cfg.n_layers)])
        ev = OE.replay(res.trace.records, cfg.n_layers, cfg.n_experts, res.trace.prompt_len,
                       CacheConfig(2, 4, eng.cache.expert_bytes),
                       OE.SpeculationConfig(enabled=spec, m=2), gates=gates)
        got = [(e.seq, e.kind, e.key.layer, e.key.expert, e.token_pos, e.bytes_moved)
               for e in eng.events]
        assert got == ev
        assert all(k in KINDS for _, k, *_ in ev)


def test_degenerate_model_guesses_exact(c1_models):
    from oracle import model as OM
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig
    cfg = OM.ModelConfig(vocab_size=32, d_model=32, n_layers=4, n_heads=4, d_ffn=48, n_experts=8)
    p = OM.init_params(cfg)
    for l in range(cfg.n_layers):
        for e in range(cfg.n_experts):
            p[f"layers.{l}.experts.{e}.w_down_proj"][:] = 0.0
        if l >= 1:
            p[f"layers.{l}.attn.wo"][:] = 0.0
    eng = OffloadEngine(OM.Model(cfg, p), CacheConfig(k=0, b=4), SpeculationConfig(True, 2))
    eng.prefill([3])
    eng.decode(12, sampler="greedy")
    misses = [e for e in eng.events if e.token_pos >= 1 and e.kind == "miss_load"
              and e.key.layer >= 1]
    assert misses == []


def test_errors_map_to_reference_exceptions(c1_models):
    cfg, get = c1_models
    model, pay, attn = get(None)
    eng = _engine(model, pay, attn, 2, 4, 0)
    with pytest.raises(RuntimeError):
        eng.decode(1)
    with pytest.raises(ValueError):
        eng.prefill([])
    with pytest.raises(ValueError):
        eng.prefill([cfg.vocab_size])
    with pytest.raises(ValueError):
        _engine(model, pay, attn, 2, 1, 2)


def test_mixtral_width_decode_bitwise_reproducible():
    """The split-K reductions are order independent (int64 fixed-point sums,
    kernels.cuh MOE_FX_*), so two decodes of the same prompt give bit-identical
    logits and tokens whatever the CTA timing and cache state."""
    import bench
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig
    from paper_2312_17238_b200 import synthetic_model
    cfg = dict(bench.MIXTRAL)
    cfg["n_layers"] = 2
    cobj = bench.cfg_obj(cfg)
    eng = OffloadEngine(synthetic_model(cobj, 0), CacheConfig(k=1, b=4),
                        SpeculationConfig(enabled=True, m=2), record_hidden=False,
                        synth=(0, 4, 3), expert_bytes=bench.expert_bytes(bench.MIXTRAL, 3))
    prompt = [int(t) for t in np.random.default_rng(1).integers(0, cobj.vocab_size, 4)]
    runs = []
    for _ in range(2):
        eng.reset_session()
        eng.prefill(prompt)
        r = eng.decode(4)
        runs.append((r.tokens, r.final_logits.copy()))
    eng.close()
    assert runs[0][0] == runs[1][0]
    assert np.array_equal(runs[0][1], runs[1][1])


@pytest.mark.parametrize("bits,n", [(3, 9), (2, 70)])
def test_mixtral_width_batched_prefill_equals_per_position(bits, n, monkeypatch):
    """Batched prefill (the positions as input columns of the tensor-core
    GEMVs, one pass over each distinct expert per layer; engine.cu
    prefill_batched) gives bit-identical logits, trace and store event log to
    running the decode kernels once per position (MOE_PREFILL_BATCH=0), for a
    ragged last column group (9 = 2 x 4 + 1) and a prompt longer than one
    64-position chunk (70)."""
    import bench
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig
    from paper_2312_17238_b200 import synthetic_model
    cfg = dict(bench.MIXTRAL)
    cfg["n_layers"] = 2
    cobj = bench.cfg_obj(cfg)
    prompt = [int(t) for t in np.random.default_rng(5).integers(0, cobj.vocab_size, n)]
    outs = []
    for batch in ("1", "0"):
        monkeypatch.setenv("MOE_PREFILL_BATCH", batch)
        eng = OffloadEngine(synthetic_model(cobj, 0), CacheConfig(k=2, b=4),
                            SpeculationConfig(enabled=False), record_hidden=True,
                            synth=(0, 4, bits), expert_bytes=bench.expert_bytes(bench.MIXTRAL, bits))
        logits = eng.prefill(prompt)
        r = eng.decode(2)
        tr = eng.trace()
        outs.append((np.asarray(logits).copy(), r.tokens, _ev_rows(eng.events),
                     [(x.token_pos, x.layer, tuple(x.experts)) for x in tr.records],
                     np.stack([x.hidden for x in tr.records]),
                     np.stack([x.weights for x in tr.records])))
        eng.close()
    a, b = outs
    assert np.array_equal(a[0], b[0])
    assert a[1] == b[1]
    assert a[2] == b[2]
    assert a[3] == b[3]
    assert np.array_equal(a[4], b[4])
    assert np.array_equal(a[5], b[5])


def test_engine_from_serialized_blocks_equals_engine_from_blocks(c1_models):
    """§8(f)3: expert payloads and attention blocks handed over as the
    reference's serialized bytes (quant.serialize_block, e.g. read from disk)
    are parsed in C++ (csrc/blockio.cu) straight into the pinned arena and the
    device weights; the engine then matches the one built from block objects
    bit for bit (logits, tokens, store events)."""
    from oracle import quant as OQ
    from paper_2312_17238_b200 import CacheConfig, ExpertKey, OffloadEngine, SpeculationConfig
    cfg, get = c1_models
    model, pay, attn = get((4, 3))
    pay = {ExpertKey(*k): v for k, v in pay.items()}
    ser_pay = {k: tuple(OQ.serialize(b) for b in v) for k, v in pay.items()}
    ser_attn = {k: OQ.serialize(v) for k, v in attn.items()}
    prompt = make_prompt(3, 7, cfg.vocab_size)
    outs = []
    for p, a in ((pay, attn), (ser_pay, ser_attn)):
        eng = OffloadEngine(model, CacheConfig(k=2, b=4), SpeculationConfig(True, 2),
                            payloads=p, attn_blocks=a)
        logits = np.asarray(eng.prefill(prompt)).copy()
        r = eng.decode(6)
        outs.append((logits, r.tokens, r.final_logits.copy(), _ev_rows(eng.events),
                     eng.cache.expert_bytes))
        eng.close()
    a, b = outs
    assert np.array_equal(a[0], b[0]) and a[1] == b[1] and np.array_equal(a[2], b[2])
    assert a[3] == b[3] and a[4] == b[4]


def test_mixtral_width_fused_attention_equals_attention_kernel(monkeypatch):
    """The decode attention fused into the Wo GEMV prologue (X_ATTN: every Wo
    CTA computes its head dims with attend_head) gives bit-identical logits,
    tokens, trace and events to the separate per-head attention kernel
    (MOE_ATTN_FUSED=0), including the KV rows later tokens read back."""
    import bench
    from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig
    from paper_2312_17238_b200 import synthetic_model
    cfg = dict(bench.MIXTRAL)
    cfg["n_layers"] = 2
    cobj = bench.cfg_obj(cfg)
    prompt = [int(t) for t in np.random.default_rng(11).integers(0, cobj.vocab_size, 3)]
    outs = []
    for fused in ("1", "0"):
        monkeypatch.setenv("MOE_ATTN_FUSED", fused)
        eng = OffloadEngine(synthetic_model(cobj, 0), CacheConfig(k=2, b=4),
                            SpeculationConfig(enabled=True, m=2), record_hidden=True,
                            synth=(0, 4, 3), expert_bytes=bench.expert_bytes(bench.MIXTRAL, 3))
        logits = np.asarray(eng.prefill(prompt)).copy()
        r = eng.decode(40)
        tr = eng.trace()
        outs.append((logits, r.tokens, r.final_logits.copy(), _ev_rows(eng.events),
                     np.stack([x.hidden for x in tr.records])))
        eng.close()
    a, b = outs
    assert np.array_equal(a[0], b[0]) and a[1] == b[1] and np.array_equal(a[2], b[2])
    assert a[3] == b[3] and np.array_equal(a[4], b[4])


def test_decode_past_max_seq_len_matches_reference(c1_models):
    """KVCache.append (model.py:265-268): decoding past max_seq_len decodes the
    tokens that fit, then raises ValueError('position T exceeds max_seq_len=T');
    the event log, trace and position match the reference engine's state after
    the same exception."""
    import dataclasses

    from moe_offload.engine import OffloadEngine as RefEngine
    from moe_offload.engine import SpeculationConfig as RSpec
    from moe_offload.model import Model as RModel, ModelConfig as RConfig
    from paper_2312_17238_b200 import CacheConfig
    cfg, get = c1_models
    model, pay, attn = get(None)
    T = cfg.max_seq_len
    prompt = make_prompt(9, T - 3, cfg.vocab_size)
    rmodel = RModel(RConfig(**dataclasses.asdict(cfg)), model.params)  # the same weights
    ref = RefEngine(rmodel, CacheConfig(k=2, b=4), RSpec(enabled=False))
    ref.prefill(prompt)
    with pytest.raises(ValueError) as re_:
        ref.decode(6)
    eng = _engine(model, pay, attn, 2, 4, 0)
    eng.prefill(prompt)
    with pytest.raises(ValueError) as ge:
        eng.decode(6)
    assert str(ge.value) == str(re_.value)
    assert len(eng.trace().records) == len(ref.trace().records)
    assert [r.experts for r in eng.trace().records] == [r.experts for r in ref.trace().records]
    assert _ev_rows(eng.events) == _ev_rows(ref.events)
    with pytest.raises(ValueError):
        eng.prefill(make_prompt(9, T + 1, cfg.vocab_size))
