"""Oracle restatement of the reference decode math (TEST INFRASTRUCTURE ONLY).

Follows ``/root/reference/pkg/src/moe_offload/model.py``.  Every arithmetic step
is float32 numpy, in the reference's order:
  * ModelConfig ................ model.py:40-77
  * init_params draw order ..... model.py:145-175
  * layer_norm ................. model.py:186-189
  * top_k_select / gate ........ model.py:192-220
  * swiglu / _sigmoid .......... model.py:223-235
  * moe_forward ................ model.py:238-254
  * KVCache .................... model.py:257-277
  * attention_step ............. model.py:280-301
  * output_logits / embed ...... model.py:304-319
  * forward_token / prefill .... model.py:322-367
  * samplers ................... model.py:374-401

Also provides ``synth_params``: a counter-hash weight source whose integer
arithmetic is reproduced bit-for-bit by the B200 engine's device generator, so
Mixtral-shaped models can be regenerated on either side without shipping
weights.
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

LN_EPS = 1e-5


class NonFiniteError(ValueError):
    """reference model.py:36-37."""


@dataclass(frozen=True)
class ModelConfig:
    vocab_size: int
    d_model: int
    n_layers: int
    n_heads: int
    d_ffn: int
    n_experts: int
    top_k_gate: int = 2
    seed: int = 0
    max_seq_len: int = 256

    def __post_init__(self):
        dims = (self.vocab_size, self.d_model, self.n_layers, self.n_heads, self.d_ffn,
                self.n_experts, self.top_k_gate, self.max_seq_len)
        if min(dims) < 1:
            raise ValueError("all model dimensions must be >= 1")
        if self.d_model % self.n_heads:
            raise ValueError("d_model must be divisible by n_heads")
        if self.top_k_gate > self.n_experts:
            raise ValueError("top_k_gate cannot exceed n_experts")

    @property
    def head_dim(self) -> int:
        return self.d_model // self.n_heads

    def to_dict(self) -> dict:
        return {k: getattr(self, k) for k in (
            "vocab_size", "d_model", "n_layers", "n_heads", "d_ffn", "n_experts",
            "top_k_gate", "seed", "max_seq_len")}


@dataclass(frozen=True)
class ExpertKey:
    layer: int
    expert: int

    def __iter__(self):
        return iter((self.layer, self.expert))


@dataclass
class Model:
    config: ModelConfig
    params: dict

    def gate_matrix(self, layer: int) -> np.ndarray:
        return self.params[f"layers.{layer}.gate"]

    def expert(self, layer: int, e: int):
        b = f"layers.{layer}.experts.{e}"
        p = self.params
        return (p[f"{b}.w_gate_proj"], p[f"{b}.w_up_proj"], p[f"{b}.w_down_proj"])


def init_params(cfg: ModelConfig) -> dict:
    """Seeded normal init in the reference's exact draw order (model.py:145-175)."""
    gen = np.random.default_rng(cfg.seed)
    d, f, v = cfg.d_model, cfg.d_ffn, cfg.vocab_size

    def draw(shape, std):
        return (gen.standard_normal(shape) * std).astype(np.float32)

    p = {"wte": draw((v, d), 0.02), "wpe": draw((cfg.max_seq_len, d), 0.02),
         "lm_head": draw((d, v), 0.02),
         "ln_f.gamma": np.ones(d, np.float32), "ln_f.beta": np.zeros(d, np.float32)}
    std_d = 1.0 / np.sqrt(d)
    for l in range(cfg.n_layers):
        pre = f"layers.{l}"
        for nm in ("ln1", "ln2"):
            p[f"{pre}.{nm}.gamma"] = np.ones(d, np.float32)
            p[f"{pre}.{nm}.beta"] = np.zeros(d, np.float32)
        for nm in ("wq", "wk", "wv", "wo"):
            p[f"{pre}.attn.{nm}"] = draw((d, d), std_d)
        p[f"{pre}.gate"] = draw((d, cfg.n_experts), std_d)
        for e in range(cfg.n_experts):
            eb = f"{pre}.experts.{e}"
            p[f"{eb}.w_gate_proj"] = draw((d, f), std_d)
            p[f"{eb}.w_up_proj"] = draw((d, f), std_d)
            p[f"{eb}.w_down_proj"] = draw((f, d), 1.0 / np.sqrt(f))
    return p


# ----------------------------------------------------------- synthetic weights
# Counter-based integer hash -> sum of four 16-bit uniforms (Irwin-Hall(4)),
# centred and scaled by one float32 multiply.  Integer-exact, so the device
# generator (csrc/synth.cu) reproduces it bit for bit.

_M64 = (1 << 64) - 1
SYNTH_IHSTD = 37837.22700   # std of (sum of four U{0..65535}) = 65536/sqrt(3)


def _mix64(z: np.ndarray) -> np.ndarray:
    """splitmix64 finalizer on uint64 arrays."""
    z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
    z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def synth_scale(std: float) -> np.float32:
    return np.float32(std / SYNTH_IHSTD)


def synth_tensor(seed: int, tensor_id: int, shape, std: float, offset: int = 0,
                 count: int | None = None) -> np.ndarray:
    """Deterministic pseudo-normal float32 tensor (flat elements
    [offset, offset+count) of ``shape``)."""
    n = int(np.prod(shape))
    if count is None:
        count = n - offset
    base = np.uint64(((seed * 0x9E3779B97F4A7C15) ^ (tensor_id * 0xD1B54A32D192ED03)) & _M64)
    idx = np.arange(offset, offset + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        h = _mix64(idx * np.uint64(0x9E3779B97F4A7C15) + base)
    s = ((h & np.uint64(0xFFFF)) + ((h >> np.uint64(16)) & np.uint64(0xFFFF))
         + ((h >> np.uint64(32)) & np.uint64(0xFFFF)) + (h >> np.uint64(48)))
    z = s.astype(np.int64) - 131070
    out = z.astype(np.float32) * synth_scale(std)
    return out.reshape(shape) if offset == 0 and count == n else out


def synth_tensor_ids(cfg: ModelConfig):
    """Stable tensor ids for :func:`synth_params` (shared with the device)."""
    ids = {"wte": 1, "wpe": 2, "lm_head": 3}
    for l in range(cfg.n_layers):
        base = 1000 + 100 * l
        for j, nm in enumerate(("wq", "wk", "wv", "wo")):
            ids[f"layers.{l}.attn.{nm}"] = base + j
        ids[f"layers.{l}.gate"] = base + 4
        for e in range(cfg.n_experts):
            for j, nm in enumerate(("w_gate_proj", "w_up_proj", "w_down_proj")):
                ids[f"layers.{l}.experts.{e}.{nm}"] = base + 10 + 3 * e + j
    return ids


def synth_std(name: str, cfg: ModelConfig) -> float:
    if name in ("wte", "wpe", "lm_head"):
        return 0.02
    if name.endswith("w_down_proj"):
        return 1.0 / np.sqrt(cfg.d_ffn)
    return 1.0 / np.sqrt(cfg.d_model)


def synth_shape(name: str, cfg: ModelConfig):
    d, f = cfg.d_model, cfg.d_ffn
    if name == "wte":
        return (cfg.vocab_size, d)
    if name == "wpe":
        return (cfg.max_seq_len, d)
    if name == "lm_head":
        return (d, cfg.vocab_size)
    if name.endswith(".gate"):
        return (d, cfg.n_experts)
    if ".attn." in name:
        return (d, d)
    if name.endswith("w_down_proj"):
        return (f, d)
    return (d, f)


def synth_param(name: str, cfg: ModelConfig, seed: int) -> np.ndarray:
    ids = synth_tensor_ids(cfg)
    return synth_tensor(seed, ids[name], synth_shape(name, cfg), synth_std(name, cfg))


def synth_params(cfg: ModelConfig, seed: int = 0, layers=None) -> dict:
    """All (or selected layers') parameters from the counter hash."""
    d = cfg.d_model
    p = {nm: synth_param(nm, cfg, seed) for nm in ("wte", "wpe", "lm_head")}
    p["ln_f.gamma"], p["ln_f.beta"] = np.ones(d, np.float32), np.zeros(d, np.float32)
    for l in (range(cfg.n_layers) if layers is None else layers):
        pre = f"layers.{l}"
        for nm in ("ln1", "ln2"):
            p[f"{pre}.{nm}.gamma"] = np.ones(d, np.float32)
            p[f"{pre}.{nm}.beta"] = np.zeros(d, np.float32)
        for nm in ("wq", "wk", "wv", "wo"):
            p[f"{pre}.attn.{nm}"] = synth_param(f"{pre}.attn.{nm}", cfg, seed)
        p[f"{pre}.gate"] = synth_param(f"{pre}.gate", cfg, seed)
        for e in range(cfg.n_experts):
            for nm in ("w_gate_proj", "w_up_proj", "w_down_proj"):
                key = f"{pre}.experts.{e}.{nm}"
                p[key] = synth_param(key, cfg, seed)
    return p


# ----------------------------------------------------------------- pure math

def layer_norm(x, gamma, beta):
    """Population-variance LayerNorm (model.py:186-189)."""
    mu = x.mean(axis=-1, keepdims=True)
    var = x.var(axis=-1, keepdims=True)
    return (x - mu) / np.sqrt(var + LN_EPS) * gamma + beta


def top_k(logits, k):
    """Descending, ties -> lower index (model.py:192-195)."""
    return np.argsort(-logits, kind="stable")[:k]


@dataclass
class GateOutcome:
    layer: int
    token_pos: int
    experts: tuple           # expert indices, descending weight
    weights: np.ndarray      # float32
    logits: np.ndarray


def gate(model: Model, layer: int, h, token_pos: int = 0) -> GateOutcome:
    """Linear gate, top-k, softmax over the selected logits (model.py:198-220)."""
    h = np.asarray(h)
    if not np.all(np.isfinite(h)):
        raise NonFiniteError(f"gate input at layer {layer}, position {token_pos} is not finite")
    if not 0 <= layer < model.config.n_layers:
        raise ValueError(f"layer {layer} out of range")
    logits = h @ model.gate_matrix(layer)
    sel = top_k(logits, model.config.top_k_gate)
    z = logits[sel]
    z = z - z.max()
    ez = np.exp(z)
    w = ez / ez.sum()
    return GateOutcome(layer, token_pos, tuple(int(e) for e in sel), w.astype(np.float32), logits)


def sigmoid(x):
    """Branch-stable logistic (model.py:229-235)."""
    out = np.empty_like(x)
    pos = x >= 0
    out[pos] = 1.0 / (1.0 + np.exp(-x[pos]))
    ex = np.exp(x[~pos])
    out[~pos] = ex / (1.0 + ex)
    return out


def swiglu(w1, w3, w2, x):
    """((x@W1)·σ(x@W1)·(x@W3)) @ W2 (model.py:223-226)."""
    a = x @ w1
    b = x @ w3
    return (a * sigmoid(a) * b) @ w2


def moe_forward(h, outcome: GateOutcome, experts) -> np.ndarray:
    """h + Σ w_i·SwiGLU_i(h), descending-weight order (model.py:238-254)."""
    if len(experts) != len(outcome.experts):
        raise ValueError("resolved expert list does not match gate outcome")
    out = h
    for w, ew in zip(outcome.weights, experts):
        if ew is None:
            raise ValueError("expert weights were not resolved")
        out = out + w * swiglu(*ew, h)
    return out


class KVCache:
    """fp32 (max_seq, H, hd) per layer (model.py:257-277)."""

    def __init__(self, cfg: ModelConfig):
        shp = (cfg.max_seq_len, cfg.n_heads, cfg.head_dim)
        self.k = [np.zeros(shp, np.float32) for _ in range(cfg.n_layers)]
        self.v = [np.zeros(shp, np.float32) for _ in range(cfg.n_layers)]
        self.n = [0] * cfg.n_layers
        self.cap = cfg.max_seq_len

    def append(self, layer, k, v):
        t = self.n[layer]
        if t >= self.cap:
            raise ValueError(f"sequence exceeds max_seq_len={self.cap}")
        self.k[layer][t] = k
        self.v[layer][t] = v
        self.n[layer] = t + 1

    def view(self, layer):
        t = self.n[layer]
        return self.k[layer][:t], self.v[layer][:t]


def attention_step(model: Model, layer: int, x, kv: KVCache, pos: int):
    """LN1 -> q,k,v -> KV append -> softmax(qK^T/sqrt(hd)) V -> x + ctx@Wo -> LN2
    (model.py:280-301).  Returns the pre-MoE hidden state."""
    cfg, p = model.config, model.params
    pre = f"layers.{layer}"
    n1 = layer_norm(x, p[f"{pre}.ln1.gamma"], p[f"{pre}.ln1.beta"])
    hd = cfg.head_dim
    q = (n1 @ p[f"{pre}.attn.wq"]).reshape(cfg.n_heads, hd)
    k = (n1 @ p[f"{pre}.attn.wk"]).reshape(cfg.n_heads, hd)
    v = (n1 @ p[f"{pre}.attn.wv"]).reshape(cfg.n_heads, hd)
    kv.append(layer, k, v)
    K, V = kv.view(layer)
    s = np.einsum("hd,thd->ht", q, K) / np.float32(np.sqrt(hd))
    s = s - s.max(axis=1, keepdims=True)
    a = np.exp(s)
    a = a / a.sum(axis=1, keepdims=True)
    ctx = np.einsum("ht,thd->hd", a, V).reshape(cfg.d_model)
    r = x + ctx @ p[f"{pre}.attn.wo"]
    return layer_norm(r, p[f"{pre}.ln2.gamma"], p[f"{pre}.ln2.beta"])


def output_logits(model: Model, x):
    """LN_f -> lm_head (model.py:304-310)."""
    p = model.params
    z = layer_norm(x, p["ln_f.gamma"], p["ln_f.beta"]) @ p["lm_head"]
    if not np.all(np.isfinite(z)):
        raise NonFiniteError("output logits are not finite")
    return z


def embed(model: Model, token: int, pos: int):
    """wte[tok] + wpe[pos] (model.py:313-319)."""
    cfg = model.config
    if not 0 <= token < cfg.vocab_size:
        raise ValueError(f"token id {token} outside vocabulary of {cfg.vocab_size}")
    if pos >= cfg.max_seq_len:
        raise ValueError(f"position {pos} exceeds max_seq_len={cfg.max_seq_len}")
    return model.params["wte"][token] + model.params["wpe"][pos]


def forward_token(model, token, pos, kv, resolve, on_gate=None):
    """One token through every layer (model.py:322-340)."""
    x = embed(model, token, pos)
    for layer in range(model.config.n_layers):
        x = attention_step(model, layer, x, kv, pos)
        out = gate(model, layer, x, pos)
        if on_gate is not None:
            on_gate(layer, out, x)
        x = moe_forward(x, out, resolve(layer, out, x))
    return output_logits(model, x)


def prefill_pass(model, tokens, kv, resolve_layer, on_gate=None):
    """Layer-by-layer prompt encoding (model.py:343-367)."""
    if len(tokens) == 0:
        raise ValueError("prompt must contain at least one token")
    xs = [embed(model, t, i) for i, t in enumerate(tokens)]
    n = len(tokens)
    for layer in range(model.config.n_layers):
        for i in range(n):
            xs[i] = attention_step(model, layer, xs[i], kv, i)
        outs = [gate(model, layer, xs[i], i) for i in range(n)]
        if on_gate is not None:
            for i in range(n):
                on_gate(layer, outs[i], xs[i])
        table = resolve_layer(layer, outs)
        for i in range(n):
            xs[i] = moe_forward(xs[i], outs[i], [table[(layer, e)] for e in outs[i].experts])
    return np.stack([output_logits(model, x) for x in xs])


def sample_greedy(logits) -> int:
    return int(np.argmax(logits))


@dataclass
class CategoricalSampler:
    """numpy Generator.choice over softmax probabilities (model.py:378-393)."""

    seed: int
    _rng: np.random.Generator = field(init=False, repr=False)

    def __post_init__(self):
        self._rng = np.random.default_rng(self.seed)

    def __call__(self, logits) -> int:
        z = logits.astype(np.float64)
        z -= z.max()
        pr = np.exp(z)
        pr /= pr.sum()
        return int(self._rng.choice(pr.size, p=pr))


def make_sampler(name: str, seed: int = 0):
    if name == "greedy":
        return sample_greedy
    if name == "categorical":
        return CategoricalSampler(seed)
    raise ValueError(f"unknown sampler {name!r}")
