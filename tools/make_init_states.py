"""Record the numpy PCG64 state at the start of every tensor that the
reference ``init_params`` (model.py:145-175) draws, for a given ModelConfig.

``init_params`` draws every tensor from ONE ``default_rng(seed)`` stream in a
fixed order; the ziggurat normal sampler consumes a data-dependent number of
64-bit draws, so tensor t's first draw can only be located by generating the
whole stream once.  With the state at each tensor start recorded, any tensor
can then be regenerated independently (and in parallel) bit-for-bit:

    rng = np.random.default_rng(); rng.bit_generator.state = rec["state"]
    w = (rng.standard_normal(shape) * std).astype(np.float32)

Usage: python tools/make_init_states.py OUT.json [vocab d L H f E max_seq seed]
(defaults: the Mixtral-8x7B shape of SURVEY.md §8(d)).  Takes ~10-20 min on
one core for the full shape.
"""
import json
import sys
import time

import numpy as np


def draw_order(v, d, L, f, E, T):
    proj = 1.0 / np.sqrt(d)
    yield "wte", (v, d), 0.02
    yield "wpe", (T, d), 0.02
    yield "lm_head", (d, v), 0.02
    for ell in range(L):
        base = f"layers.{ell}"
        for nm in ("wq", "wk", "wv", "wo"):
            yield f"{base}.attn.{nm}", (d, d), proj
        yield f"{base}.gate", (d, E), proj
        for e in range(E):
            eb = f"{base}.experts.{e}"
            yield f"{eb}.w_gate_proj", (d, f), proj
            yield f"{eb}.w_up_proj", (d, f), proj
            yield f"{eb}.w_down_proj", (f, d), 1.0 / np.sqrt(f)


def main():
    out = sys.argv[1]
    v, d, L, H, f, E, T, seed = (int(x) for x in sys.argv[2:10]) if len(sys.argv) > 2 else \
        (32000, 4096, 32, 32, 14336, 8, 256, 0)
    rng = np.random.default_rng(seed)
    buf = np.empty(1 << 22, np.float64)
    recs = []
    t0 = time.time()
    for name, shape, std in draw_order(v, d, L, f, E, T):
        st = rng.bit_generator.state
        recs.append({"name": name, "shape": list(shape), "std": float(std),
                     "state": str(st["state"]["state"]), "inc": str(st["state"]["inc"])})
        n = int(np.prod(shape))
        while n:
            c = min(n, buf.size)
            rng.standard_normal(out=buf[:c])
            n -= c
        print(f"{name} {time.time() - t0:.0f}s", flush=True)
    st = rng.bit_generator.state
    doc = {"config": {"vocab_size": v, "d_model": d, "n_layers": L, "n_heads": H, "d_ffn": f,
                      "n_experts": E, "max_seq_len": T, "seed": seed},
           "end_state": str(st["state"]["state"]), "tensors": recs}
    with open(out, "w") as fh:
        json.dump(doc, fh, indent=0)


if __name__ == "__main__":
    main()
