"""Mixtral-shape mixed-quant inputs for the engine, built on the host + device.

The reference's random-init weights (init_params, model.py:145-175; see
initw.py) at the Mixtral-8x7B shape, generated on all host threads and
quantized on the GPU with the engine's quantizer (``moe_quantize_device``: the
reference's ``quant.quantize`` restated for sm_100a, byte-identical --
tests/test_gpu_engine.py, tests/test_gpu_depth.py) into the reference's own
``QuantizedBlock`` type: 4-bit attention projections, 2/3-bit experts, fp16
embeddings / lm_head / gates (quant.py:428 REQUIRED_FP16_ROLES), LayerNorm 1/0.
This is input preparation for the bench (what a user would load from a
checkpoint), not part of the decode path.
"""

from __future__ import annotations

import ctypes as C
import time
from types import SimpleNamespace

import numpy as np

from . import _lib, initw
from .api import moe_offload  # noqa: F401

PRESET = {2: (16, 128), 3: (64, 128), 4: (64, 256)}  # quant.py:68-73 (group, scale group)


def quantize_device(w: np.ndarray, bits: int):
    """reference quant.quantize(w, PRESET[bits]) on the GPU -> QuantizedBlock."""
    from moe_offload.quant import QuantizedBlock, QuantScheme
    g, sg = PRESET[bits]
    w = np.ascontiguousarray(w, np.float32)
    K, N = w.shape
    ng = K * N // g
    nr, nsg = -(-ng // sg), -(-ng // (sg // g))
    codes, zeros = np.empty(K * N * bits // 8, np.uint8), np.empty(ng, np.uint8)
    zs, zo, sc = np.empty(nr, np.uint16), np.empty(nr, np.uint16), np.empty(nsg, np.uint16)
    vp = lambda a: a.ctypes.data_as(C.c_void_p)  # noqa: E731
    _lib.check(_lib.lib().moe_quantize_device(w.ctypes.data_as(_lib.FP), K, N, bits, g, sg,
                                              vp(codes), vp(zeros), vp(zs), vp(zo), vp(sc)))
    return QuantizedBlock(QuantScheme(bits=bits, group_size=g, scale_group_size=sg), codes,
                          zeros, zs.view(np.float16), zo.view(np.float16), sc.view(np.float16),
                          (K, N), 0)


def mixtral_model(attn_bits: int, expert_bits: int, n_layers: int = 32, owned=None,
                  threads: int | None = None, log=None):
    """-> (model namespace with .config/.params, attn_blocks, expert payloads
    {(l, e): (W1, W3, W2)}).  ``owned(l, e)`` restricts the experts generated
    (expert parallel ranks)."""
    from moe_offload.model import ModelConfig
    t0 = time.time()
    doc = initw.load_states()
    c = dict(doc["config"])
    c["n_layers"] = n_layers
    cfg = ModelConfig(vocab_size=c["vocab_size"], d_model=c["d_model"], n_layers=n_layers,
                      n_heads=c["n_heads"], d_ffn=c["d_ffn"], n_experts=c["n_experts"],
                      top_k_gate=2, seed=c["seed"], max_seq_len=c["max_seq_len"])
    d, E = cfg.d_model, cfg.n_experts
    names = initw.dense_names(n_layers)
    keys = [(l, e) for l in range(n_layers) for e in range(E) if owned is None or owned(l, e)]
    for l, e in keys:
        names += initw.expert_names(l, e)
    params = {"ln_f.gamma": np.ones(d, np.float32), "ln_f.beta": np.zeros(d, np.float32)}
    for l in range(n_layers):
        for nm in ("ln1", "ln2"):
            params[f"layers.{l}.{nm}.gamma"] = np.ones(d, np.float32)
            params[f"layers.{l}.{nm}.beta"] = np.zeros(d, np.float32)
    attn, pend, experts = {}, {}, {}
    for name, w in initw.iter_tensors(doc, names, threads=threads):
        if ".attn." in name:
            attn[name] = quantize_device(w, attn_bits)
        elif ".experts." in name:
            p = name.split(".")
            key = (int(p[1]), int(p[3]))
            pend.setdefault(key, {})[p[4]] = quantize_device(w, expert_bits)
            if len(pend[key]) == 3:
                q = pend.pop(key)
                experts[key] = (q["w_gate_proj"], q["w_up_proj"], q["w_down_proj"])
        else:
            params[name] = w.astype(np.float16).astype(np.float32)
    if log:
        log(f"weights: {len(names)} tensors generated + quantized in {time.time() - t0:.1f}s")
    return SimpleNamespace(config=cfg, params=params), attn, experts
