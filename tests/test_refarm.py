"""The CPU reference arm (oracle/refarm.py) is the unmodified reference engine
plus the quantized payload adapter: on a small mixed-quant model it must give
the oracle engine's tokens, event log and logits (CPU)."""

import numpy as np
import pytest

from oracle import engine as OE
from oracle import model as OM
from oracle import refarm
from oracle.store import CacheConfig


@pytest.mark.parametrize("ebits,k,m", [(3, 4, 0), (2, 2, 2)])
def test_reference_arm_matches_oracle(ebits, k, m):
    cfg = OM.ModelConfig(vocab_size=128, d_model=256, n_layers=2, n_heads=2, d_ffn=896,
                         n_experts=8, max_seq_len=64)
    params = OM.init_params(cfg)
    fq, pay, attn = OE.build_mixed_quant(params, cfg, 4, ebits)
    dense = {n: v for n, v in fq.items() if ".experts." not in n and ".attn." not in n}
    eng = refarm.build_engine(cfg.to_dict(), dense, attn, pay, k, m, threads=2)
    assert type(eng).__module__ == "moe_offload.engine"
    prompt = [int(t) for t in np.random.default_rng(3).integers(0, 128, 5)]
    eng.prefill(prompt)
    times, toks = refarm.time_tokens(eng, 6)
    ref = OE.OffloadEngine(OM.Model(cfg, fq), CacheConfig(k=k, b=4),
                           OE.SpeculationConfig(m > 0, max(m, 1)), payloads=pay,
                           record_hidden=False)
    ref.prefill(prompt)
    rt, rl = ref.decode(6)
    assert toks == rt
    got = [(e.seq, e.kind, e.key.layer, e.key.expert, e.token_pos, e.bytes_moved)
           for e in eng.events]
    assert got == ref.events
    np.testing.assert_array_equal(eng._last_logits, rl)  # same numpy math, same bits
    assert len(times) == 6 and min(times) > 0
