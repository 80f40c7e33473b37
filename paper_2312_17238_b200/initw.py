"""The reference's random-init weights at any size, regenerated in parallel.

Reference ``init_params`` (model.py:145-175) draws every tensor, in a fixed
order, from ONE ``np.random.default_rng(seed)`` stream:
``(rng.standard_normal(shape) * std).astype(np.float32)``.  The ziggurat normal
sampler consumes a data-dependent number of 64-bit draws, so the position of a
tensor in the stream is only known after generating everything before it;
``tools/make_init_states.py`` does that once and records the PCG64 state at
the start of every tensor (``data/*.json``).  With those states any tensor is
regenerated independently and bit-for-bit, on many threads at once
(``Generator.standard_normal`` releases the GIL), so the Mixtral-shape model
(47.5e9 weights) takes about a minute instead of the reference's serial pass.

This is input synthesis (the reference's weights), not part of the decode path.
"""

from __future__ import annotations

import json
import os
from concurrent.futures import ThreadPoolExecutor

import numpy as np

DATA = os.path.join(os.path.dirname(os.path.abspath(__file__)), "data")
MIXTRAL_STATES = os.path.join(DATA, "mixtral_init_states.json")


def load_states(path: str = MIXTRAL_STATES) -> dict:
    with open(path) as fh:
        doc = json.load(fh)
    doc["by_name"] = {t["name"]: t for t in doc["tensors"]}
    return doc


def gen_tensor(rec: dict) -> np.ndarray:
    """One tensor of init_params from its recorded stream state (model.py:153-154)."""
    rng = np.random.default_rng()
    st = rng.bit_generator.state
    st["state"] = {"state": int(rec["state"]), "inc": int(rec["inc"])}
    st["has_uint32"], st["uinteger"] = 0, 0
    rng.bit_generator.state = st
    # same stream and same rounding as (rng.standard_normal(shape) * std).astype(f32),
    # in cache-sized chunks
    out = np.empty(tuple(rec["shape"]), np.float32)
    flat = out.reshape(-1)
    buf = np.empty(min(flat.size, 1 << 18))
    std = float(rec["std"])
    for o in range(0, flat.size, buf.size):
        c = buf[:min(buf.size, flat.size - o)]
        rng.standard_normal(out=c)
        np.multiply(c, std, out=c)
        flat[o:o + c.size] = c
    return out


def iter_tensors(doc: dict, names, threads: int | None = None, window: int | None = None,
                 fn=None):
    """Yields (name, float32 array) -- or (name, fn(name, array)), fn applied on
    the worker thread -- in ``names`` order, generated ``threads`` at a time
    with at most ``window`` finished tensors held."""
    threads = threads or os.cpu_count() or 1
    window = window or 2 * threads
    names = list(names)
    with ThreadPoolExecutor(threads) as ex:
        futs = {}
        nxt = 0
        for i, nm in enumerate(names):
            while nxt < len(names) and nxt < i + window:
                futs[nxt] = ex.submit(_work, doc["by_name"][names[nxt]], fn)
                nxt += 1
            yield nm, futs.pop(i).result()


def _work(rec, fn):
    w = gen_tensor(rec)
    return w if fn is None else fn(rec["name"], w)


def dense_names(n_layers: int):
    """Non-expert tensors of init_params (the ones drawn from the stream)."""
    out = ["wte", "wpe", "lm_head"]
    for l in range(n_layers):
        out += [f"layers.{l}.attn.{nm}" for nm in ("wq", "wk", "wv", "wo")]
        out.append(f"layers.{l}.gate")
    return out


def expert_names(layer: int, expert: int):
    eb = f"layers.{layer}.experts.{expert}"
    return [f"{eb}.w_gate_proj", f"{eb}.w_up_proj", f"{eb}.w_down_proj"]
