"""Mixtral-shape mixed-quant model inputs for the oracle side (TEST INFRASTRUCTURE ONLY).

The weights are the reference's own ``init_params`` (model.py:145-175) at the
Mixtral-8x7B shape of SURVEY.md §8(d), regenerated in parallel from the
recorded stream states (paper_2312_17238_b200/initw.py), then mixed-quantized
like BASELINE configs 2/3 (oracle/engine.py build_mixed_quant): attention
projections group-quantized (4-bit), experts 2/3-bit, embeddings / lm_head /
gates float16-rounded, norms 1/0 -- with the C quantizer that is
byte-identical to reference quant.quantize (oracle/fastq.py).
"""

from __future__ import annotations

import os
import time

import numpy as np

from paper_2312_17238_b200 import initw

from . import fastq as FQ
from . import quant as Q
from .model import ModelConfig

MIXTRAL = dict(vocab_size=32000, d_model=4096, n_layers=32, n_heads=32, d_ffn=14336,
               n_experts=8, top_k_gate=2, seed=0, max_seq_len=256)


def mixtral_config(n_layers: int = 32) -> ModelConfig:
    return ModelConfig(**{**MIXTRAL, "n_layers": n_layers})


def build(expert_bits=(3,), attn_bits: int = 4, n_layers: int = 32, keep_f32=(),
          threads: int | None = None, experts=True, log=print):
    """Returns dict(cfg, dense, attn{name: block}, experts{bits: {(l,e): (b1,b3,b2)}},
    f32{name: array}).  Generation and quantization run on ``threads`` worker
    threads (numpy's normal sampler and the C quantizer release the GIL)."""
    t0 = time.time()
    doc = initw.load_states()
    cfg = mixtral_config(n_layers)
    L, E = cfg.n_layers, cfg.n_experts
    names = initw.dense_names(L)
    if experts:
        names += [n for l in range(L) for e in range(E) for n in initw.expert_names(l, e)]
    keep = set(keep_f32)

    def work(name, w):
        out = {"f32": w if name in keep else None}
        if ".experts." in name:
            out["q"] = {b: FQ.quantize(w, Q.PRESETS[b], nthreads=1) for b in expert_bits}
        elif ".attn." in name:
            out["q"] = FQ.quantize(w, Q.PRESETS[attn_bits], nthreads=1)
        else:  # fp16 passthrough roles (quant.py:428): float16-rounded float32
            out["d"] = w.astype(np.float16).astype(np.float32)
        return out

    res = {"cfg": cfg, "dense": {}, "attn": {}, "experts": {b: {} for b in expert_bits},
           "f32": {}}
    d = cfg.d_model
    res["dense"]["ln_f.gamma"] = np.ones(d, np.float32)
    res["dense"]["ln_f.beta"] = np.zeros(d, np.float32)
    for l in range(L):
        for nm in ("ln1", "ln2"):
            res["dense"][f"layers.{l}.{nm}.gamma"] = np.ones(d, np.float32)
            res["dense"][f"layers.{l}.{nm}.beta"] = np.zeros(d, np.float32)
    pend = {}
    for name, out in initw.iter_tensors(doc, names, threads=threads, fn=work):
        if out["f32"] is not None:
            res["f32"][name] = out["f32"]
        if "d" in out:
            res["dense"][name] = out["d"]
        elif ".attn." in name:
            res["attn"][name] = out["q"]
        else:
            parts = name.split(".")
            key = (int(parts[1]), int(parts[3]))
            pend.setdefault(key, {})[parts[4]] = out["q"]
            if len(pend[key]) == 3:
                p = pend.pop(key)
                for b in expert_bits:
                    res["experts"][b][key] = tuple(p[nm][b] for nm in ("w_gate_proj", "w_up_proj",
                                                                       "w_down_proj"))
    log(f"mixtral weights: {len(names)} tensors in {time.time() - t0:.1f}s "
        f"({threads or os.cpu_count()} threads)")
    return res
