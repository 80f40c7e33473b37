"""The batched full-depth oracle (oracle/depth.py) reproduces the sequential
oracle engine (the reference flow, pinned to reference goldens) on a small
mixed-quant model: greedy tokens, routing, store event log (one store across
prompts), logits within fp32 summation-order tolerance (CPU)."""

import numpy as np
import pytest

from oracle import depth as OD
from oracle import engine as OE
from oracle import fastq as FQ
from oracle import model as OM
from oracle.store import CacheConfig


def depth_model(cfg, fq, pay, attn):
    dense = {k: v for k, v in fq.items() if ".experts." not in k and ".attn." not in k}
    dm = OD.DepthModel(cfg, dense)
    for key, blk in attn.items():
        l = int(key.split(".")[1])
        dm.attn[(l, key.split(".")[-1])] = FQ.prepared(blk)
    for (l, e), trip in pay.items():
        dm.experts[(l, e)] = tuple(FQ.prepared(b) for b in trip)
    return dm


@pytest.mark.parametrize("ebits,k,m", [(3, 4, 0), (2, 2, 2)])
def test_depth_oracle_equals_sequential_oracle(ebits, k, m):
    cfg = OM.ModelConfig(vocab_size=512, d_model=256, n_layers=3, n_heads=2, d_ffn=896,
                         n_experts=8, max_seq_len=64, seed=1)
    params = OM.init_params(cfg)
    fq, pay, attn = OE.build_mixed_quant(params, cfg, 4, ebits)
    prompts = [[int(t) for t in np.random.default_rng(s).integers(0, 512, 6)] for s in range(3)]
    n = 4
    ora = OD.DepthOracle(depth_model(cfg, fq, pay, attn), spec_m=m)
    sess = ora.run(prompts, n)
    cc = CacheConfig(k=k, b=4, expert_bytes=OE.payload_bytes(pay[(0, 0)]))
    spec = OE.SpeculationConfig(m > 0, max(m, 1))
    ref = OE.OffloadEngine(OM.Model(cfg, fq), cc, spec, payloads=pay, record_hidden=True)
    for s, p in zip(sess, prompts):
        pre = ref.prefill(p)
        np.testing.assert_allclose(s.prefill_last, pre[-1], rtol=0, atol=2e-5 * np.abs(pre).max())
        toks, fin = ref.decode(n)
        assert s.out_tokens == toks
        np.testing.assert_allclose(s.logits, fin, rtol=0, atol=2e-5 * np.abs(fin).max())
        got = sorted((r.token_pos, r.layer, r.experts) for r in s.recs)
        assert [(r.token_pos, r.layer, tuple(r.experts)) for r in ref.sorted_records()] == got
    gates = np.stack([fq[f"layers.{l}.gate"] for l in range(cfg.n_layers)])
    ev = OD.replay_sessions(sess, cfg.n_layers, cfg.n_experts, cc, m, 1, gates)
    assert ev == ref.events
    assert min(r.gate_margin for s in sess for r in s.recs) > 0
