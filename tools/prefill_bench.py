"""Batched vs per-position prefill at Mixtral width with every expert resident
(compute-bound: k = 8 = E, so no miss traffic after the warm-up prefill).

    python tools/prefill_bench.py [n_layers] [prompt_len ...]

Prints one JSON line per prompt length: prefill ms of the batched path
(engine.cu prefill_batched) and of the per-position path (MOE_PREFILL_BATCH=0),
one greedy decode token's ms on the same engine, and the ratios, per layer and
scaled to 32 layers.
"""
import json
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import bench  # noqa: E402
from paper_2312_17238_b200 import CacheConfig, OffloadEngine, SpeculationConfig  # noqa: E402
from paper_2312_17238_b200 import synthetic_model  # noqa: E402


def main():
    nl = int(sys.argv[1]) if len(sys.argv) > 1 else 4
    lens = [int(a) for a in sys.argv[2:]] or [1, 4, 16, 64]
    bits = int(os.environ.get("PREFILL_BENCH_BITS", "3"))
    cfg = dict(bench.MIXTRAL)
    cfg["n_layers"] = nl
    cobj = bench.cfg_obj(cfg)
    eng = OffloadEngine(synthetic_model(cobj, 0), CacheConfig(k=8, b=4),
                        SpeculationConfig(enabled=False), record_hidden=False,
                        synth=(0, 4, bits), expert_bytes=bench.expert_bytes(bench.MIXTRAL, bits))
    rng = np.random.default_rng(0)
    warm = [int(t) for t in rng.integers(0, cobj.vocab_size, 64)]
    eng.prefill(warm)  # loads every expert of every layer (k = E)
    eng.prefill(warm)
    eng.decode(4)
    dec = []
    for _ in range(3):
        eng.prefill(warm[:8])
        eng.decode(8)
        dec.append(eng.stats()["last_call_ms"] / 8)
    dec_ms = float(np.median(dec))
    if os.environ.get("MOE_NCU_RANGE") == "1":  # ncu --profile-from-start off: one prefill
        from paper_2312_17238_b200 import _lib
        prompt = [int(t) for t in rng.integers(0, cobj.vocab_size, lens[0])]
        eng.prefill(prompt)
        _lib.check(_lib.lib().moe_profiler_range(1))
        eng.prefill(prompt)
        _lib.check(_lib.lib().moe_profiler_range(0))
        eng.close()
        return
    for n in lens:
        prompt = [int(t) for t in rng.integers(0, cobj.vocab_size, n)]
        res = {}
        for mode in ("1", "0"):
            os.environ["MOE_PREFILL_BATCH"] = mode
            ts = []
            for _ in range(3):
                eng.prefill(prompt)
                ts.append(eng.stats()["last_call_ms"])
            res[mode] = float(np.median(ts))
        os.environ.pop("MOE_PREFILL_BATCH", None)
        out = {"prompt_len": n, "n_layers": nl, "expert_bits": bits,
               "batched_ms": round(res["1"], 3), "per_position_ms": round(res["0"], 3),
               "decode_token_ms": round(dec_ms, 3),
               "speedup": round(res["0"] / res["1"], 2),
               "batched_prefill_in_decode_tokens": round(res["1"] / dec_ms, 2),
               "batched_ms_per_layer": round(res["1"] / nl, 3),
               "batched_ms_32_layers": round(res["1"] / nl * 32, 2)}
        print(json.dumps(out), flush=True)
    eng.close()


if __name__ == "__main__":
    main()
