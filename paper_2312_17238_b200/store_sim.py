"""Host execution of the engine's device store (csrc/store_dev.cuh).

``DeviceStoreSim`` drives the *same* ``store::resolve_token`` /
``store::resolve_prefill`` code the bookkeeping kernels run, on the CPU, with
the reference store's surface (store.py:76-220: ``events``, ``device_state``,
``staged_keys``, ``audit``) plus the physical side the reference never sees
(which HBM buffer holds which expert).  Used by the CPU tests and by the
expert-parallel ownership logic; the decode path itself never calls it.
"""

from __future__ import annotations

import ctypes as C

import numpy as np

from . import _lib
from .api import EVENT_KINDS, CacheConfig, ExpertKey, StoreEvent
from .errors import UnknownExpertError


def _check(rc: int):
    if rc == 0:
        return
    msg = (_lib.lib().moe_store_sim_last_error() or b"").decode()
    if rc == _lib.MOE_ERR_UNKNOWN_EXPERT:
        raise UnknownExpertError(msg)
    if rc == _lib.MOE_ERR_VALUE:
        raise ValueError(msg)
    raise RuntimeError(msg)


class DeviceStoreSim:
    def __init__(self, n_layers: int, n_experts: int, cache: CacheConfig, top_k: int = 2,
                 m: int = 2, owned=None):
        self.L, self.E, self.cache, self.top_k = n_layers, n_experts, cache, top_k
        self._owned = None
        if owned is not None:
            mask = np.zeros((n_layers, n_experts), np.uint8)
            for l, e in owned:
                mask[l, e] = 1
            self._owned = mask
        h = C.c_void_p()
        _check(_lib.lib().moe_store_sim_create(
            n_layers, n_experts, cache.k, cache.b, cache.expert_bytes, top_k, m,
            self._owned.ctypes.data_as(C.c_void_p) if self._owned is not None else None,
            C.byref(h)))
        self._h = h

    def __del__(self):
        try:
            if self._h:
                _lib.lib().moe_store_sim_destroy(self._h)
                self._h = None
        except Exception:
            pass

    # -- the two bookkeeping entry points of the engine
    def resolve_token(self, layer: int, pos: int, experts, guesses=(), guess_layer: int = -1):
        """engine.py:222-231: acquire ``experts`` (descending weight), then
        speculative_load ``guesses`` into ``guess_layer``.  Returns buffers."""
        ex = np.ascontiguousarray(experts, np.int32)
        g = np.ascontiguousarray(list(guesses) or [0], np.int32)
        ex = ex if ex.size else np.zeros(0, np.int32)
        out = np.full(ex.size, -1, np.int32)
        _check(_lib.lib().moe_store_sim_token(
            self._h, layer, pos, ex.ctypes.data_as(_lib.IP), ex.size, g.ctypes.data_as(_lib.IP),
            len(guesses), guess_layer, out.ctypes.data_as(_lib.IP)))
        return out

    def resolve_prefill(self, layer: int, experts):
        """engine.py:233-240 for one layer; experts: (n, k).  Returns buffers."""
        ex = np.ascontiguousarray(experts, np.int32)
        n, k = ex.shape
        out = np.full((n, k), -1, np.int32)
        _check(_lib.lib().moe_store_sim_prefill(self._h, layer, ex.ctypes.data_as(_lib.IP), n, k,
                                                out.ctypes.data_as(_lib.IP)))
        return out

    # -- reference store surface
    @property
    def events(self) -> list[StoreEvent]:
        L = _lib.lib()
        n = L.moe_store_sim_num_events(self._h)
        buf = (_lib.Event * max(n, 1))()
        _check(L.moe_store_sim_events(self._h, buf, n))
        return [StoreEvent(int(e.seq), EVENT_KINDS[e.kind], ExpertKey(int(e.layer), int(e.expert)),
                           int(e.token_pos), int(e.bytes_moved)) for e in buf[:n]]

    def _state(self):
        L, E, k, b = self.L, self.E, self.cache.k, self.cache.b
        lru = np.full(max(L * k, 1), -1, np.int32)
        stg = np.full(max(b, 1), -1, np.int32)
        nbuf = C.c_int32()
        _check(_lib.lib().moe_store_sim_state(self._h, lru.ctypes.data_as(_lib.IP),
                                              stg.ctypes.data_as(_lib.IP), None, None, None,
                                              C.byref(nbuf)))
        content = np.full(nbuf.value, -1, np.int32)
        res = np.full(L * E, -1, np.int32)
        sbuf = np.full(max(b, 1), -1, np.int32)
        _check(_lib.lib().moe_store_sim_state(self._h, None, None, content.ctypes.data_as(_lib.IP),
                                              res.ctypes.data_as(_lib.IP),
                                              sbuf.ctypes.data_as(_lib.IP), None))
        return lru[:L * k].reshape(L, k), stg[:b], content, res.reshape(L, E), sbuf[:b]

    def device_state(self):
        lru = self._state()[0]
        return {l: tuple(ExpertKey(l, int(x)) for x in row if x >= 0) for l, row in enumerate(lru)}

    def staged_keys(self):
        stg = self._state()[1]
        return tuple(ExpertKey(int(s) // self.E, int(s) % self.E) for s in stg if s >= 0)

    def buffers(self):
        """Physical view: {'content': buffer -> layer*E+expert, 'resident':
        (L,E) buffer of each resident key or -1, 'staged': buffer per slot}."""
        _, _, content, res, sbuf = self._state()
        return {"content": content, "resident": res, "staged": sbuf}

    @property
    def copies(self) -> int:
        return int(_lib.lib().moe_store_sim_copies(self._h))

    def audit(self):
        """store.py:114-125 plus the physical invariants: every resident or
        staged key sits in its own buffer, and that buffer holds the key."""
        seen = set()
        for l, keys in self.device_state().items():
            if len(keys) > self.cache.k:
                raise AssertionError(f"layer {l} holds {len(keys)} > k experts")
            for key in keys:
                if key.layer != l or key in seen:
                    raise AssertionError(f"duplicate or misfiled resident {key}")
                seen.add(key)
        phys = self.buffers()
        live = {}
        for l in range(self.L):
            for e in range(self.E):
                b = int(phys["resident"][l, e])
                if b >= 0:
                    live.setdefault(b, []).append((l, e))
        for key, b in zip(self.staged_keys(), [x for x in phys["staged"] if x >= 0]):
            live.setdefault(int(b), []).append(tuple(key))
        for b, keys in live.items():
            if len(keys) != 1:
                raise AssertionError(f"buffer {b} shared by {keys}")
            l, e = keys[0]
            if phys["content"][b] != l * self.E + e:
                raise AssertionError(f"buffer {b} does not hold {keys[0]}")


def replay_device(trace, cache: CacheConfig, speculation=None):
    """The reference ``replay`` (engine.py:263-313) driven through the engine's
    device store code: prompt positions batched layer by layer (each distinct
    expert acquired once per layer), generated positions token by token with
    the speculative guesses re-evaluated from the recorded hidden states.
    Returns the simulator (``.events`` is the log to compare with
    ``replay(trace, cache, speculation).events``)."""
    from moe_offload.engine import SpeculationConfig
    from moe_offload.model import top_k_select
    spec = speculation or SpeculationConfig()
    m = spec.m if spec.enabled else 0
    trace.validate()
    sim = DeviceStoreSim(trace.n_layers, trace.n_experts, cache, top_k=trace.top_k, m=max(m, 1))
    by_tok = {}
    for r in trace.records:
        by_tok.setdefault(r.token_pos, []).append(r)
    prompt = [t for t in sorted(by_tok) if t < trace.prompt_len]
    gen = [t for t in sorted(by_tok) if t >= trace.prompt_len]
    if prompt:
        for ell in range(trace.n_layers):
            ex = np.array([next(r for r in by_tok[t] if r.layer == ell).experts for t in prompt],
                          np.int32)
            sim.resolve_prefill(ell, ex)
    for t in gen:
        for r in sorted(by_tok[t], key=lambda r: r.layer):
            target = r.layer + spec.lookahead
            guesses = ()
            if m > 0 and target < trace.n_layers:
                guesses = [int(e) for e in top_k_select(trace.gate_logits(target, r.hidden), m)]
            sim.resolve_token(r.layer, t, list(r.experts), guesses, target if guesses else -1)
    return sim
