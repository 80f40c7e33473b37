"""B200 drop-in for the reference ``OffloadEngine`` (engine.py:200-247).

Same constructor, same ``_Session`` surface (``prefill`` / ``run_token`` /
``decode`` / ``trace`` / ``events`` / ``recall`` / ``store``), same exceptions;
the decode path runs entirely in ``libmoeb200.so``: attention and expert
dequant-GEMVs, gating, the device-resident LRU/staging store, speculative
prefetch and the host->device copy engine.  Python only marshals weights in
and events / traces / logits out.
"""

from __future__ import annotations

import ctypes as C
from types import SimpleNamespace

import numpy as np

from . import _lib
from ._lib import check, lib
from .api import (EVENT_KINDS, CacheConfig, ExpertKey, GenerationResult, SpeculationConfig,
                  StoreEvent, Trace, TraceRecord, config_digest, make_sampler, recall)

_KIND_OF = {i: k for i, k in enumerate(EVENT_KINDS)}


# ------------------------------------------------------------ weight marshalling

def _is_block(w) -> bool:
    return hasattr(w, "packed_codes") and hasattr(w, "scheme")


def _is_serialized(w) -> bool:
    return isinstance(w, (bytes, bytearray, memoryview))


def block_payload_nbytes(block) -> int:
    """Serialized payload bytes (reference quant.py:332-343); for a serialized
    block (quant.serialize_block bytes) the bytes after its header."""
    if _is_serialized(block):
        ndim = bytes(block[11:12])[0] if len(block) >= 12 else 0
        return len(block) - (12 + 4 * ndim + 4)
    if block.scheme.bits == 16:
        return len(block.packed_codes)
    zb = -(-np.asarray(block.zeros).size * block.scheme.meta_bits // 8)
    return int(len(block.packed_codes) + zb + 2 * np.asarray(block.zero_scales).size
               + 2 * np.asarray(block.zero_offsets).size + 2 * np.asarray(block.scales).size)


def expert_triple(payload):
    """(w_gate_proj, w_up_proj, w_down_proj) of any supported payload."""
    if hasattr(payload, "w_gate_proj"):
        return payload.w_gate_proj, payload.w_up_proj, payload.w_down_proj
    if hasattr(payload, "blocks"):
        return tuple(payload.blocks)
    if isinstance(payload, (tuple, list)) and len(payload) == 3:
        return tuple(payload)
    raise TypeError(f"unsupported expert payload {type(payload).__name__}")


def payload_nbytes(payload) -> int:
    """engine.py:79-82: ExpertWeights -> summed array bytes, else .nbytes."""
    if hasattr(payload, "w_gate_proj") and not _is_block(payload.w_gate_proj):
        return int(payload.w_gate_proj.nbytes + payload.w_up_proj.nbytes
                   + payload.w_down_proj.nbytes)
    if hasattr(payload, "nbytes") and not isinstance(payload, np.ndarray):
        return int(payload.nbytes)
    tot = 0
    for w in expert_triple(payload):
        tot += (block_payload_nbytes(w) if _is_block(w) or _is_serialized(w)
                else int(np.asarray(w).nbytes))
    return tot


class _Marshal:
    """Builds moe_matrix structs, keeping the backing arrays alive."""

    def __init__(self):
        self.keep = []

    def _ptr(self, arr):
        arr = np.ascontiguousarray(arr)
        self.keep.append(arr)
        return arr.ctypes.data_as(C.c_void_p), arr

    def dense(self, a, allow_half: bool):
        a = np.asarray(a, dtype=np.float32)
        if a.ndim == 1:
            a = a[None, :]
        m = _lib.Matrix()
        m.rows, m.cols = a.shape
        h = a.astype(np.float16)
        if allow_half and np.array_equal(h.astype(np.float32), a):
            m.bits = 16
            m.codes, arr = self._ptr(h)
        else:
            m.bits = 32
            m.codes, arr = self._ptr(a)
        m.codes_len = arr.nbytes
        return m

    def block(self, b):
        sch = b.scheme
        shape = tuple(b.original_shape)
        m = _lib.Matrix()
        m.rows, m.cols = (shape if len(shape) == 2 else (1, int(np.prod(shape))))
        m.bits = sch.bits
        m.pad_count = int(b.pad_count)
        codes = np.frombuffer(b.packed_codes, dtype=np.uint8)
        m.codes, _ = self._ptr(codes)
        m.codes_len = codes.size
        if sch.bits == 16:
            return m
        m.group_size, m.scale_group_size, m.meta_bits = (sch.group_size, sch.scale_group_size,
                                                         sch.meta_bits)
        z = np.asarray(b.zeros, dtype=np.uint8)
        m.zeros, _ = self._ptr(z)
        m.n_groups = z.size
        zs = np.asarray(b.zero_scales, dtype=np.float16).view(np.uint16)
        zo = np.asarray(b.zero_offsets, dtype=np.float16).view(np.uint16)
        sc = np.asarray(b.scales, dtype=np.float16).view(np.uint16)
        m.zero_scales, _ = self._ptr(zs)
        m.zero_offsets, _ = self._ptr(zo)
        m.n_zruns = zs.size
        m.scales, _ = self._ptr(sc)
        m.n_scales = sc.size
        return m

    def any(self, w, allow_half=False):
        return self.block(w) if _is_block(w) else self.dense(w, allow_half)


def _model_desc(cfg) -> _lib.ModelDesc:
    d = _lib.ModelDesc()
    d.vocab_size, d.d_model, d.n_layers = cfg.vocab_size, cfg.d_model, cfg.n_layers
    d.n_heads, d.d_ffn, d.n_experts = cfg.n_heads, cfg.d_ffn, cfg.n_experts
    d.top_k, d.max_seq_len = cfg.top_k_gate, cfg.max_seq_len
    return d


class _StoreView:
    """Read-only view of the device store with the reference store's surface
    (store.py:105-125): events, config, device_state, staged_keys, audit."""

    def __init__(self, eng: "OffloadEngine"):
        self._eng = eng

    @property
    def config(self) -> CacheConfig:
        return self._eng.cache

    @property
    def events(self) -> list[StoreEvent]:
        return self._eng.events

    def _state(self):
        e = self._eng
        L, k, b, E = e.model.config.n_layers, e.cache.k, e.cache.b, e.model.config.n_experts
        lru = np.full(max(L * k, 1), -1, np.int32)
        stg = np.full(max(b, 1), -1, np.int32)
        check(lib().moe_device_state(e._h, lru.ctypes.data_as(_lib.IP),
                                     stg.ctypes.data_as(_lib.IP)))
        return lru[:L * k].reshape(L, k) if k else np.zeros((L, 0), np.int32), stg[:b], E

    def device_state(self):
        lru, _, _ = self._state()
        return {l: tuple(ExpertKey(l, int(x)) for x in row if x >= 0)
                for l, row in enumerate(lru)}

    def device_resident(self, layer: int):
        return self.device_state()[layer]

    def staged_keys(self):
        _, stg, E = self._state()
        return tuple(ExpertKey(int(s) // E, int(s) % E) for s in stg if s >= 0)

    def audit(self):
        seen = set()
        for l, keys in self.device_state().items():
            if len(keys) > self.config.k:
                raise AssertionError(f"layer {l} holds {len(keys)} > k experts")
            for key in keys:
                if key.layer != l or key in seen:
                    raise AssertionError(f"duplicate or misfiled resident {key}")
                seen.add(key)
        if len(self.staged_keys()) > self.config.b:
            raise AssertionError("staging overflow")


class OffloadEngine:
    """Generation with the device store (reference engine.py:200-247).

    Extra keyword arguments over the reference:
      attn_blocks : {"layers.{l}.attn.w{q,k,v,o}": QuantizedBlock} to run the
                    attention projections as quantized GEMVs (mixed-quant models);
                    default: the model's float32 projections.
      device      : CUDA device ordinal.
      synth       : (seed, attn_bits, expert_bits) -> skip host weights and build
                    the counter-hash synthetic model on device (bench path).
      ep_rank / ep_world : expert parallel (expert_parallel.py); after
                    construction call ``ep_connect`` with every rank's
                    ``ep_handle()`` (expert_parallel.connect does it over
                    torch.distributed).
    """

    def __init__(self, model, cache: CacheConfig | None = None,
                 speculation: SpeculationConfig = SpeculationConfig(), payloads=None,
                 record_hidden: bool = True, attn_blocks: dict | None = None, device: int = 0,
                 synth: tuple | None = None, expert_bytes: int | None = None,
                 ep_rank: int = 0, ep_world: int = 1):
        self.model = model
        self.record_hidden = record_hidden
        self._h = None
        cfg = model.config
        if synth is None:
            if payloads is None:
                payloads = {ExpertKey(l, e): tuple(model.params[f"layers.{l}.experts.{e}.{nm}"]
                                                   for nm in ("w_gate_proj", "w_up_proj",
                                                              "w_down_proj"))
                            for l in range(cfg.n_layers) for e in range(cfg.n_experts)}
            nbytes = payload_nbytes(next(iter(payloads.values())))
        else:
            nbytes = int(expert_bytes)
        if cache is None:
            cache = CacheConfig(k=2, b=4, expert_bytes=nbytes)
        elif cache.expert_bytes == 1:  # engine.py:213-214
            cache = CacheConfig(k=cache.k, b=cache.b, expert_bytes=nbytes)
        if speculation.enabled and speculation.m > cache.b:
            raise ValueError(f"m={speculation.m} exceeds b={cache.b} staging buffers")
        if cache.k > cfg.n_experts:
            raise ValueError(f"k={cache.k} exceeds experts per layer ({cfg.n_experts})")
        self.cache = cache
        self.speculation = speculation
        L = lib()
        cc = _lib.CacheCfg(cache.k, cache.b, cache.expert_bytes)
        sc = _lib.SpecCfg(int(speculation.enabled), speculation.m, speculation.lookahead)
        h = C.c_void_p()
        check(L.moe_create(C.byref(_model_desc(cfg)), C.byref(cc), C.byref(sc), device,
                           int(record_hidden), C.byref(h)))
        self._h = h
        self.ep_rank, self.ep_world = ep_rank, ep_world
        if ep_world > 1:
            check(L.moe_ep_configure(h, ep_rank, ep_world))
        if synth is not None:
            check(L.moe_synth_model(h, int(synth[0]), int(synth[1]), int(synth[2])))
        else:
            self._load(model, payloads, attn_blocks or {})
        check(L.moe_finalize(h))
        self._events: list[StoreEvent] = []
        self.store = _StoreView(self)
        self.reset_session()

    # ------------------------------------------------------------ loading
    def _load(self, model, payloads, attn_blocks):
        cfg, p, L = model.config, model.params, lib()

        def put(name, w, allow_half=False):
            if _is_serialized(w):  # quant.serialize_block bytes (e.g. read from disk)
                buf = bytes(w)
                check(L.moe_load_tensor_serialized(self._h, name.encode(), buf, len(buf)))
                return
            mk = _Marshal()
            m = mk.any(w, allow_half)
            check(L.moe_load_tensor(self._h, name.encode(), C.byref(m)))

        # wte and wpe are read by one embedding kernel: fp16 only if both are
        # exactly representable in fp16
        emb_half = all(_is_block(p[nm]) or np.array_equal(
            np.asarray(p[nm], np.float32).astype(np.float16).astype(np.float32),
            np.asarray(p[nm], np.float32)) for nm in ("wte", "wpe"))
        for nm in ("wte", "wpe"):
            put(nm, p[nm], allow_half=emb_half)
        put("lm_head", p["lm_head"], allow_half=True)
        put("ln_f.gamma", p["ln_f.gamma"])
        put("ln_f.beta", p["ln_f.beta"])
        for l in range(cfg.n_layers):
            pre = f"layers.{l}"
            for nm in ("ln1.gamma", "ln1.beta", "ln2.gamma", "ln2.beta", "gate"):
                put(f"{pre}.{nm}", p[f"{pre}.{nm}"])
            for nm in ("wq", "wk", "wv", "wo"):
                key = f"{pre}.attn.{nm}"
                put(key, attn_blocks[key] if key in attn_blocks else p[key])
        from .expert_parallel import owner_of
        for key, payload in payloads.items():
            k = ExpertKey(*key)
            if owner_of(k.expert, cfg.n_experts, self.ep_world) != self.ep_rank:
                continue  # another rank's expert
            trip = expert_triple(payload)
            if all(_is_serialized(w) for w in trip):  # serialized blocks, parsed in C++
                bufs = [bytes(w) for w in trip]
                check(L.moe_load_expert_serialized(self._h, k.layer, k.expert,
                                                   *[a for b in bufs for a in (b, len(b))]))
                continue
            mk = _Marshal()
            ms = [mk.any(w) for w in trip]
            check(L.moe_load_expert(self._h, k.layer, k.expert, *[C.byref(m) for m in ms]))

    # ------------------------------------------------------------ expert parallel
    def ep_handle(self) -> bytes:
        """This rank's 64-byte exchange-buffer handle (CUDA IPC)."""
        buf = C.create_string_buffer(64)
        check(lib().moe_ep_handle(self._h, buf))
        return buf.raw

    def ep_connect(self, handles) -> None:
        """Open every rank's exchange buffer (handles in rank order)."""
        blob = b"".join(handles)
        if len(blob) != 64 * self.ep_world:
            raise ValueError("need one 64-byte handle per rank")
        check(lib().moe_ep_connect(self._h, C.c_char_p(blob)))

    def ep_connect_nccl(self, unique_id: bytes) -> None:
        """NCCL transport: join the communicator named by rank 0's 128-byte
        ``nccl_unique_id()``; the slot exchange becomes one ncclAllGather per
        layer and position (include/moeb200.h)."""
        if len(unique_id) != 128:
            raise ValueError("an NCCL unique id is 128 bytes")
        check(lib().moe_ep_connect_nccl(self._h, C.c_char_p(unique_id)))

    def close(self):
        if self._h is not None:
            lib().moe_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    # ------------------------------------------------------------ session
    def reset_session(self) -> None:
        check(lib().moe_reset_session(self._h))
        self._pos = 0
        self._last_logits = None
        self._logits_on_device = False
        self._prompt_len = 0

    def prefill(self, tokens) -> np.ndarray:
        """engine.py:148-156: resets KV (not the store), returns (n, V) logits."""
        toks = np.ascontiguousarray(list(tokens), dtype=np.int32)
        V = self.model.config.vocab_size
        self._last_logits = None
        self._logits_on_device = False
        out = np.empty((max(toks.size, 1), V), np.float32)
        rc = lib().moe_prefill(self._h, toks.ctypes.data_as(_lib.IP), int(toks.size),
                               out.ctypes.data_as(_lib.FP))
        check(rc)
        self._pos = self._prompt_len = int(toks.size)
        self._last_logits = out[-1].copy()
        self._logits_on_device = True
        return out

    def run_token(self, token: int) -> np.ndarray:
        """engine.py:158-166."""
        if self._last_logits is None:
            raise RuntimeError("prefill must run before decoding")
        out = np.empty(self.model.config.vocab_size, np.float32)
        rc = lib().moe_step(self._h, int(token), out.ctypes.data_as(_lib.FP))
        check(rc)
        self._pos += 1
        self._last_logits = out
        self._logits_on_device = True
        return out

    def decode(self, n_tokens: int, sampler="greedy", sampler_seed: int = 0) -> GenerationResult:
        """engine.py:168-182.  The greedy sampler runs on device (argmax kernel);
        other samplers draw on the host from each step's logits."""
        if n_tokens < 1:
            raise ValueError("n_tokens must be >= 1")
        greedy = sampler == "greedy"
        if isinstance(sampler, str):
            sampler = make_sampler(sampler, sampler_seed)
        if self._last_logits is None:
            raise RuntimeError("prefill must run before decoding")
        if greedy and self._logits_on_device:
            V = self.model.config.vocab_size
            toks = np.empty(n_tokens, np.int32)
            fin = np.empty(V, np.float32)
            rc = lib().moe_decode_greedy(self._h, int(n_tokens), toks.ctypes.data_as(_lib.IP),
                                         fin.ctypes.data_as(_lib.FP))
            if rc:  # e.g. past max_seq_len: the tokens that fit were decoded (reference order)
                self._pos = int(lib().moe_num_trace(self._h)) // self.model.config.n_layers
            check(rc)
            self._pos += n_tokens
            self._last_logits = fin
            return GenerationResult([int(t) for t in toks], fin, self.trace())
        tokens = []
        logits = self._last_logits
        for _ in range(n_tokens):
            t = sampler(logits)
            tokens.append(t)
            logits = self.run_token(t)
        return GenerationResult(tokens, logits, self.trace())

    # ------------------------------------------------------------ records
    def _sync_events(self):
        L = lib()
        n = L.moe_num_events(self._h)
        have = len(self._events)
        if n > have:
            buf = (_lib.Event * (n - have))()
            check(L.moe_read_events(self._h, have, n - have, buf))
            for e in buf:
                self._events.append(StoreEvent(int(e.seq), _KIND_OF[e.kind],
                                               ExpertKey(int(e.layer), int(e.expert)),
                                               int(e.token_pos), int(e.bytes_moved)))

    @property
    def events(self) -> list[StoreEvent]:
        self._sync_events()  # materialised lazily: the engine keeps the log
        return self._events

    def recall(self, definition: str = "device_or_staging") -> float:
        return recall(self.events, definition)

    def trace(self) -> Trace:
        """engine.py:130-144 (records sorted by (token_pos, layer))."""
        cfg = self.model.config
        L = lib()
        n = L.moe_num_trace(self._h)
        recs = []
        if n:
            buf = (_lib.TraceRec * n)()
            hid = np.empty((n, cfg.d_model), np.float32) if self.record_hidden else None
            check(L.moe_read_trace(self._h, 0, n, buf,
                                   hid.ctypes.data_as(_lib.FP) if hid is not None else None))
            k = cfg.top_k_gate
            for i, r in enumerate(buf):
                recs.append(TraceRecord(int(r.token_pos), int(r.layer),
                                        tuple(int(x) for x in r.experts[:k]),
                                        np.array(r.weights[:k], dtype=np.float32),
                                        hid[i].copy() if hid is not None else None))
        gates = None
        if self.record_hidden:
            gates = np.stack([np.asarray(self.model.params[f"layers.{l}.gate"], np.float32)
                              for l in range(cfg.n_layers)])
        to_dict = cfg.to_dict() if hasattr(cfg, "to_dict") else dict(vars(cfg))
        tr = Trace(config_digest=config_digest(to_dict), n_layers=cfg.n_layers,
                   n_experts=cfg.n_experts, top_k=cfg.top_k_gate,
                   records_hidden=self.record_hidden, prompt_len=self._prompt_len,
                   d_model=cfg.d_model if self.record_hidden else None, gates=gates,
                   records=recs)
        tr.sort_records()
        tr.validate()
        return tr

    def stats(self) -> dict:
        s = _lib.Stats()
        check(lib().moe_get_stats(self._h, C.byref(s)))
        return {f: getattr(s, f) for f, _ in _lib.Stats._fields_}


class DenseRunner(OffloadEngine):
    """B200 counterpart of the reference ``DenseRunner`` (engine.py:185-197): the
    in-memory path, every expert resident (k = n_experts, no staging, no
    speculation).  It runs the same kernels in the same order as any
    OffloadEngine, so offloading and speculation stay bit-transparent against it
    (reference tests/test_engine.py:112-128)."""

    def __init__(self, model, record_hidden: bool = True, **kw):
        super().__init__(model, CacheConfig(k=model.config.n_experts, b=0),
                         SpeculationConfig(enabled=False), record_hidden=record_hidden, **kw)


def synthetic_model(cfg, seed: int = 0):
    """A model object for the device-synthesized weights (no host params).
    ``trace()`` gate matrices are regenerated from the counter hash on demand."""
    return SimpleNamespace(config=cfg, params=_LazyGates(cfg, seed))


class _LazyGates(dict):
    def __init__(self, cfg, seed):
        super().__init__()
        self._cfg, self._seed = cfg, seed

    def __missing__(self, key):
        if key.endswith(".gate"):
            l = int(key.split(".")[1])
            n = self._cfg.d_model * self._cfg.n_experts
            out = np.empty(n, np.float32)
            std = 1.0 / np.sqrt(self._cfg.d_model)
            scale = np.float32(std / 37837.22700)
            check(lib().moe_synth_tensor_device(self._seed, 1000 + 100 * l + 4, n, float(scale),
                                                out.ctypes.data_as(_lib.FP)))
            v = out.reshape(self._cfg.d_model, self._cfg.n_experts)
            v = v.astype(np.float16).astype(np.float32)
            self[key] = v
            return v
        raise KeyError(key)
