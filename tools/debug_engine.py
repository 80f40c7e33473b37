"""Step-by-step smoke of the engine on the C1 tiny model (debug aid, GPU)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from oracle import engine as OE  # noqa: E402
from oracle import model as OM  # noqa: E402


def log(*a):
    print(f"[{time.strftime('%H:%M:%S')}]", *a, flush=True)


def main():
    from paper_2312_17238_b200 import CacheConfig, ExpertKey, OffloadEngine, SpeculationConfig
    cfg = OM.ModelConfig(vocab_size=512, d_model=256, n_layers=2, n_heads=2, d_ffn=896,
                         n_experts=8, seed=0)
    params = OM.init_params(cfg)
    quant = os.environ.get("Q", "none")
    if quant == "none":
        model, pay, attn = OM.Model(cfg, params), None, None
    else:
        a, x = (int(c) for c in quant)
        fq, pay, attn = OE.build_mixed_quant(params, cfg, a, x)
        model = OM.Model(cfg, fq)
        pay = {ExpertKey(*k): v for k, v in pay.items()}
    log("model built", quant)
    eng = OffloadEngine(model, CacheConfig(k=2, b=4), SpeculationConfig(True, 2), payloads=pay,
                        attn_blocks=attn)
    log("engine created", eng.stats())
    prompt = [int(t) for t in np.random.default_rng(0).integers(0, 512, 8)]
    lg = eng.prefill(prompt)
    log("prefill ok", lg.shape, lg[-1][:4], len(eng.events))
    res = eng.decode(8)
    log("decode ok", res.tokens)
    ref = OE.OffloadEngine(model, OE.CacheConfig(k=2, b=4), OE.SpeculationConfig(True, 2),
                           payloads=None if pay is None else {tuple(k): v for k, v in pay.items()})
    rl = ref.prefill(prompt)
    rt, rf = ref.decode(8)
    log("oracle", rt, "max|dlogit| prefill", float(np.abs(rl - lg).max()),
        "final", float(np.abs(rf - res.final_logits).max()))
    ev = [(e.seq, e.kind, e.key.layer, e.key.expert, e.token_pos, e.bytes_moved) for e in eng.events]
    log("events equal", ev == ref.events, len(ev), len(ref.events))
    log("stats", eng.stats())
    eng.close()


if __name__ == "__main__":
    main()
