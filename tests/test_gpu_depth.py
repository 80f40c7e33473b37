"""Full-depth parity at the benchmark configurations (GPU).

BASELINE configs C2 (Mixtral-8x7B shape, 32 layers, 4-bit attention / 3-bit
experts, LRU k=4, b=4, no prefetch) and C3 (2-bit experts, k=2, speculative
prefetch m=2, lookahead 1) on the reference's own init_params weights
(model.py:145-175, oracle/mixtral.py), prompts default_rng(s).integers(0,
32000, 16) for s = 0..4 run one after another on one engine,
N_NEW greedy tokens each, against the batched full-depth oracle
(oracle/depth.py).

Bit-exact: greedy tokens, routing (every trace record's experts), the whole
store event log.  Tolerance: prefill / final logits |d| <= 2e-3 * max|ref| +
1e-4, gate weights 5e-4, hidden states 1e-3 relative (at 32 layers the fp32
summation-order difference compounds: measured 2e-4 / 4e-4 worst case on C3,
against 4e-5 / 1e-4 on C2).  Every routing, guess and
lm_head decision's oracle margin is logged (gpurun_out/depth_parity.json).
"""

import json
import os
import time

import numpy as np
import pytest

from tests.conftest import ROOT, make_prompt

pytestmark = pytest.mark.gpu

N_PROMPTS = int(os.environ.get("DEPTH_PROMPTS", 5))
N_NEW = int(os.environ.get("DEPTH_NEW", 4))
LOGIT_RTOL = 2e-3
# the three matrices of one 3-bit/2-bit expert and one 4-bit attention projection:
# device quantizer vs the oracle quantizer on full-size matrices
CHECK = ("layers.0.experts.0.w_gate_proj", "layers.0.experts.0.w_down_proj",
         "layers.31.experts.7.w_up_proj", "layers.31.attn.wq")
_summary = {}


def _dump():
    out = os.path.join(ROOT, "gpurun_out")
    if os.path.isdir(out):
        with open(os.path.join(out, "depth_parity.json"), "w") as fh:
            json.dump(_summary, fh, indent=1)


@pytest.fixture(scope="module")
def mixtral():
    from oracle import mixtral as OMX
    t0 = time.time()
    w = OMX.build(expert_bits=(3, 2), keep_f32=CHECK)
    _summary["weights_s"] = round(time.time() - t0, 1)
    return w


def test_device_quantizer_full_matrices(mixtral):
    import ctypes as C

    from oracle import quant as OQ
    from paper_2312_17238_b200 import _lib
    L = _lib.lib()
    for name in CHECK:
        w = mixtral["f32"][name]
        if ".attn." in name:
            pairs = [(4, mixtral["attn"][name])]
        else:
            p = name.split(".")
            key, i = (int(p[1]), int(p[3])), ("w_gate_proj", "w_up_proj", "w_down_proj").index(p[4])
            pairs = [(b, mixtral["experts"][b][key][i]) for b in (3, 2)]
        for bits, ref in pairs:
            sch = OQ.PRESETS[bits]
            n, g, sg = w.size, sch.group_size, sch.scale_group_size
            ng = n // g
            codes, zeros = np.empty(n * bits // 8, np.uint8), np.empty(ng, np.uint8)
            nr, nsg = -(-ng // sg), -(-ng // (sg // g))
            zs, zo, sc = np.empty(nr, np.uint16), np.empty(nr, np.uint16), np.empty(nsg, np.uint16)
            vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
            _lib.check(L.moe_quantize_device(w.ctypes.data_as(_lib.FP), w.shape[0], w.shape[1],
                                             bits, g, sg, vp(codes), vp(zeros), vp(zs), vp(zo),
                                             vp(sc)))
            assert codes.tobytes() == bytes(ref.packed_codes), (name, bits)
            np.testing.assert_array_equal(zeros, ref.zeros)
            np.testing.assert_array_equal(zs, ref.zero_scales.view(np.uint16))
            np.testing.assert_array_equal(zo, ref.zero_offsets.view(np.uint16))
            np.testing.assert_array_equal(sc, ref.scales.view(np.uint16))


def _close(a, b, rtol=LOGIT_RTOL):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    return float(np.abs(a - b).max()), rtol * float(np.abs(b).max()) + 1e-4


@pytest.mark.parametrize("conf", ["C2", "C3"])
def test_full_depth_parity(mixtral, conf):
    from types import SimpleNamespace

    from oracle import depth as OD
    from oracle import fastq as FQ
    from oracle.store import CacheConfig as OCache
    from paper_2312_17238_b200 import CacheConfig, ExpertKey, OffloadEngine, SpeculationConfig

    bits, k, m = (3, 4, 0) if conf == "C2" else (2, 2, 2)
    cfg = mixtral["cfg"]
    experts = mixtral["experts"][bits]
    prompts = [make_prompt(s, 16, cfg.vocab_size) for s in range(N_PROMPTS)]
    model = SimpleNamespace(config=cfg, params=mixtral["dense"])

    t0 = time.time()
    eng = OffloadEngine(model, CacheConfig(k=k, b=4), SpeculationConfig(m > 0, max(m, 1)),
                        payloads={ExpertKey(*key): v for key, v in experts.items()},
                        attn_blocks=mixtral["attn"], record_hidden=True)
    t_load = time.time() - t0
    gpu = []
    t0 = time.time()
    for p in prompts:
        pre = eng.prefill(p)
        res = eng.decode(N_NEW)
        gpu.append((pre[-1].copy(), res.tokens, res.final_logits.copy(), res.trace.records))
    t_gpu = time.time() - t0
    events = [(e.seq, e.kind, e.key.layer, e.key.expert, e.token_pos, e.bytes_moved)
              for e in eng.events]
    expert_bytes = eng.cache.expert_bytes
    eng.close()

    t0 = time.time()
    dm = OD.DepthModel(cfg, mixtral["dense"])
    for name, blk in mixtral["attn"].items():
        dm.attn[(int(name.split(".")[1]), name.split(".")[-1])] = FQ.prepared(blk)
    for key, trip in experts.items():
        dm.experts[key] = tuple(FQ.prepared(b) for b in trip)
    sess = OD.DepthOracle(dm, spec_m=m).run(prompts, N_NEW)
    gates = np.stack([mixtral["dense"][f"layers.{l}.gate"] for l in range(cfg.n_layers)])
    ref_ev = OD.replay_sessions(sess, cfg.n_layers, cfg.n_experts,
                                OCache(k=k, b=4, expert_bytes=expert_bytes), m, 1, gates)
    t_oracle = time.time() - t0

    rep = {"load_s": round(t_load, 1), "gpu_s": round(t_gpu, 1), "oracle_s": round(t_oracle, 1),
           "prompts": []}
    _summary[conf] = rep
    failures = []
    for i, ((pre, toks, fin, recs), s) in enumerate(zip(gpu, sess)):
        e_pre, tol_pre = _close(pre, s.prefill_last)
        e_fin, tol_fin = _close(fin, s.logits)
        got = [(r.token_pos, r.layer, tuple(r.experts)) for r in recs]
        want = [(r.token_pos, r.layer, r.experts) for r in sorted(s.recs, key=lambda r: (r.token_pos, r.layer))]
        by = {(r.token_pos, r.layer): r for r in s.recs}
        route_bad = [(g, w, by[w[:2]].gate_margin) for g, w in zip(got, want) if g != w]
        w_err = max(float(np.abs(r.weights - by[(r.token_pos, r.layer)].weights).max()) for r in recs)
        h_err = max(float(np.abs(r.hidden - by[(r.token_pos, r.layer)].hidden).max() /
                          max(1e-30, np.abs(by[(r.token_pos, r.layer)].hidden).max())) for r in recs)
        rep["prompts"].append({
            "prompt": i, "tokens": toks, "oracle_tokens": s.out_tokens,
            "prefill_err": e_pre, "prefill_tol": tol_pre, "final_err": e_fin, "final_tol": tol_fin,
            "gate_w_err": w_err, "hidden_rel_err": h_err,
            "min_gate_margin": min(r.gate_margin for r in s.recs),
            "min_guess_margin": min(r.guess_margin for r in s.recs),
            "lm_margins": s.lm_margins, "routing_mismatches": len(route_bad)})
        if toks != s.out_tokens:
            failures.append(f"prompt {i}: tokens {toks} != oracle {s.out_tokens} "
                            f"(lm margins {s.lm_margins})")
        if route_bad:
            failures.append(f"prompt {i}: routing differs at {route_bad[:3]}")
        if e_pre > tol_pre or e_fin > tol_fin:
            failures.append(f"prompt {i}: logits err {e_pre:.3g}/{e_fin:.3g} > tol")
        if w_err > 5e-4 or h_err > 1e-3:
            failures.append(f"prompt {i}: gate weight err {w_err:.3g}, hidden rel err {h_err:.3g}")
    rep["events"] = len(events)
    rep["events_equal"] = events == ref_ev
    acq = [e for e in events if e[1] in ("hit", "staging_hit", "miss_load")]
    rep["hit_rate"] = sum(e[1] in ("hit", "staging_hit") for e in acq) / max(1, len(acq))
    if events != ref_ev:
        j = next((i for i, (a, b) in enumerate(zip(events, ref_ev)) if a != b),
                 min(len(events), len(ref_ev)))
        failures.append(f"event log differs at {j}: {events[j:j + 2]} vs {ref_ev[j:j + 2]} "
                        f"(lengths {len(events)} / {len(ref_ev)})")
    _dump()
    assert not failures, "\n".join(failures)
