"""The CPU reference arm: the UNMODIFIED reference ``moe_offload.OffloadEngine``
on the host cores (BENCH / TEST INFRASTRUCTURE ONLY -- bench.py's
``--impl reference`` and ``cpu_baseline`` legs).

Everything on the timed path is the reference's own code from the install in
``baseline/_ref`` -- ``_Session.decode`` / ``run_token`` / ``forward_token``,
``attention_step``, ``gate``, ``TieredExpertStore``, ``guess_experts``,
``moe_forward`` / ``swiglu`` (engine.py:97-247, model.py:186-367,
store.py:76-240) -- except the one piece the reference does not ship: the
quantized expert payload that ``materialize_expert`` duck-types
(engine.py:71-82).  ``QuantizedExpertPayload.materialize``
dequantizes its three blocks on every acquire, exactly as the reference's
payload contract implies, with the C restatement of ``quant.dequantize``
(bit-identical, tests/test_oracle_c.py) on all host threads; ``nbytes`` is the
reference's own ``quant.payload_nbytes``.  Attention projections are the
fake-quant float32 values (``quant.dequantize`` of the 4-bit blocks), as in the
reference's mixed-quant model.  No repo CUDA library is loaded.
"""

from __future__ import annotations

import os
import sys
import time

import numpy as np

from . import fastq as FQ

_REF = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "baseline", "_ref")


def ref_modules():
    try:
        import moe_offload  # noqa: F401
    except ImportError:
        sys.path.append(_REF)
    import moe_offload.engine as E
    import moe_offload.model as M
    import moe_offload.quant as Q
    import moe_offload.store as S
    return E, M, Q, S


def ref_block(b):
    """An oracle/product block as the reference's QuantizedBlock (same fields)."""
    _, _, Q, _ = ref_modules()
    if isinstance(b, Q.QuantizedBlock):
        return b
    s = b.scheme
    sch = Q.QuantScheme(bits=s.bits, group_size=s.group_size, scale_group_size=s.scale_group_size,
                        meta_bits=s.meta_bits)
    return Q.QuantizedBlock(sch, b.packed_codes, np.asarray(b.zeros, np.uint8),
                            np.asarray(b.zero_scales, np.float16),
                            np.asarray(b.zero_offsets, np.float16),
                            np.asarray(b.scales, np.float16), tuple(b.original_shape),
                            int(b.pad_count))


class QuantizedExpertPayload:
    """The payload duck type of engine.py:71-82: ``nbytes`` and ``materialize``."""

    def __init__(self, blocks, threads):
        _, _, Q, _ = ref_modules()
        self.blocks = tuple(blocks)
        self.threads = threads
        self.nbytes = int(sum(Q.payload_nbytes(b) for b in self.blocks))

    def materialize(self, key):
        _, M, _, _ = ref_modules()
        w1, w3, w2 = (FQ.dequantize(b, self.threads) for b in self.blocks)
        return M.ExpertWeights(key=key, w_gate_proj=w1, w_up_proj=w3, w_down_proj=w2)


def build_engine(cfg_dict, dense, attn_blocks, expert_blocks, k, m, b=4, threads=None,
                 record_hidden=False):
    """The reference OffloadEngine over the mixed-quant model.  dense: the
    non-quantized tensors (fp16-valued float32 embeddings / lm_head / gates,
    LayerNorm 1/0); attn_blocks: {name: 4-bit block}; expert_blocks:
    {(l, e): (W1, W3, W2) blocks}."""
    E, M, _, S = ref_modules()
    threads = threads or os.cpu_count() or 1
    params = dict(dense)
    for name, blk in attn_blocks.items():
        params[name] = FQ.dequantize(blk, threads)   # fake-quant float32 projections
    model = M.Model(config=M.ModelConfig(**cfg_dict), params=params)
    payloads = {S.ExpertKey(l, e): QuantizedExpertPayload([ref_block(x) for x in trip], threads)
                for (l, e), trip in expert_blocks.items()}
    return E.OffloadEngine(model, S.CacheConfig(k=k, b=b),
                           E.SpeculationConfig(enabled=m > 0, m=max(m, 1)), payloads=payloads,
                           record_hidden=record_hidden)


def time_tokens(eng, n):
    """Per-token wall time of n greedy steps through the public API
    (``decode(1, sampler="greedy")`` each)."""
    out, toks = [], []
    for _ in range(n):
        t0 = time.perf_counter()
        r = eng.decode(1, sampler="greedy")
        out.append(time.perf_counter() - t0)
        toks += r.tokens
    return out, toks


def blas_threads() -> int | None:
    try:
        from threadpoolctl import threadpool_info
        return max((p.get("num_threads") or 0) for p in threadpool_info()) or None
    except Exception:
        return None
