"""CPU baseline timing of the oracle at full Mixtral width (TEST/BENCH INFRASTRUCTURE ONLY).

Used only by ``bench.py`` (``cpu_baseline`` and ``--impl reference``).  The
reference path is timed on a bounded sample: one greedy decode step through
``n_layers_sample`` Mixtral-width layers of the same mixed-quant model
(4-bit attention, 3- or 2-bit experts, fp16 embeddings / lm_head / gates),
following the reference flow (engine.py:222-231: every acquire materializes
= dequantizes the expert, quant.py:267-304).  Per-token time at 32 layers is
extrapolated linearly: t_tok = (32 / n) * t_layers + t_head.

Weights are the counter-hash synthetic model (oracle/model.py synth_params);
to keep the bench short the blocks are produced by the device quantizer,
which tests/test_gpu_engine.py proves byte-identical to quant.quantize.
"""

from __future__ import annotations

import os
import time
from concurrent.futures import ThreadPoolExecutor

import numpy as np

from . import engine as OE
from . import model as OM
from . import quant as OQ
from .store import CacheConfig


class ParallelOffloadEngine(OE.OffloadEngine):
    """The reference flow with the top-k experts' dequantization spread over a
    thread pool ("all host threads it can use"); arithmetic unchanged."""

    pool = None

    def _resolve_token(self, layer, out, h):
        pos = out.token_pos
        for e in out.experts:
            self.store.acquire(layer, e, pos)
        sp = self.speculation  # engine.py:226-229, as OE.OffloadEngine._resolve_token
        if sp.enabled and sp.m > 0:
            g = OE.guess_experts(self.model, h, layer + sp.lookahead, sp.m)
            if g:
                self.store.speculative_load(g, pos, current_layer=layer)
        if self.pool is None:
            return [OE.materialize(self.payloads[(layer, e)]) for e in out.experts]
        blocks = [w for e in out.experts for w in self.payloads[(layer, e)]]
        deq = list(self.pool.map(lambda b: OQ.dequantize(b) if hasattr(b, "packed_codes") else b,
                                 blocks))
        return [tuple(deq[3 * i:3 * i + 3]) for i in range(len(out.experts))]


def build_sample(device_quantize, device_synth, cfg_full, seed, attn_bits, expert_bits,
                 n_layers_sample=2):
    """Mixtral-width model with the first ``n_layers_sample`` layers.

    device_quantize(w, bits) -> oracle QuantizedBlock (reference layout)
    device_synth(name, shape, std) -> float32 array (counter hash)
    """
    cfg = OM.ModelConfig(**{**cfg_full.to_dict(), "n_layers": n_layers_sample})
    ids = OM.synth_tensor_ids(cfg_full)
    p = {}
    for nm in ("wte", "wpe", "lm_head"):
        shp = OM.synth_shape(nm, cfg)
        p[nm] = device_synth(ids[nm], shp, 0.02).astype(np.float16).astype(np.float32)
    d = cfg.d_model
    p["ln_f.gamma"], p["ln_f.beta"] = np.ones(d, np.float32), np.zeros(d, np.float32)
    payloads = {}
    for l in range(n_layers_sample):
        pre = f"layers.{l}"
        for nm in ("ln1", "ln2"):
            p[f"{pre}.{nm}.gamma"] = np.ones(d, np.float32)
            p[f"{pre}.{nm}.beta"] = np.zeros(d, np.float32)
        for nm in ("wq", "wk", "wv", "wo"):
            key = f"{pre}.attn.{nm}"
            w = device_synth(ids[key], (d, d), OM.synth_std(key, cfg))
            p[key] = OQ.dequantize(device_quantize(w, attn_bits))
        g = device_synth(ids[f"{pre}.gate"], (d, cfg.n_experts), 1 / np.sqrt(d))
        p[f"{pre}.gate"] = g.astype(np.float16).astype(np.float32)
        for e in range(cfg.n_experts):
            trip = []
            for nm in ("w_gate_proj", "w_up_proj", "w_down_proj"):
                key = f"{pre}.experts.{e}.{nm}"
                w = device_synth(ids[key], OM.synth_shape(key, cfg), OM.synth_std(key, cfg))
                trip.append(device_quantize(w, expert_bits))
            payloads[(l, e)] = tuple(trip)
    return OM.Model(cfg, p), payloads


def time_steps(model, payloads, steps: int, k: int = 4, threads: int | None = None,
               prompt_token: int = 1):
    """Times ``steps`` decode steps of the sampled model.  Returns a list of
    extrapolated per-token seconds (32 layers) and the thread count used."""
    threads = threads or os.cpu_count() or 1
    eng = ParallelOffloadEngine(model, CacheConfig(k=k, b=4), payloads=payloads,
                                record_hidden=False)
    eng.pool = ThreadPoolExecutor(max_workers=threads) if threads > 1 else None
    eng.prefill([prompt_token])
    n = model.config.n_layers
    x = np.random.default_rng(0).normal(size=model.config.d_model).astype(np.float32)
    t0 = time.perf_counter()
    OM.output_logits(model, x)
    t_head = time.perf_counter() - t0
    out = []
    tok = prompt_token
    for _ in range(steps):
        t0 = time.perf_counter()
        logits = eng.run_token(tok)
        dt = time.perf_counter() - t0
        tok = OM.sample_greedy(logits)
        out.append((32 / n) * (dt - t_head) + t_head)
    if eng.pool:
        eng.pool.shutdown()
    return out, threads
