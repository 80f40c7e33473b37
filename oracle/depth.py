"""Full-depth oracle for the Mixtral-shape mixed-quant model (TEST INFRASTRUCTURE ONLY).

The same arithmetic as the reference decode path -- ``prefill_pass`` and
``forward_token`` (model.py:322-367), ``attention_step`` (model.py:280-301),
``gate`` (model.py:198-220), ``swiglu`` / ``moe_forward`` (model.py:223-254),
``output_logits`` (model.py:304-310), greedy sampling (model.py:374-375) -- run
for several independent sessions at once so that 32-layer, 4096-wide parity
checks finish in minutes: every projection of a layer is one pass over the
packed weights for all the sessions' positions (oracle/fastq.py C kernels,
x @ dequantize(W) accumulated in float64, then rounded to float32 like the
reference's fp32 result).  The per-session sequence of operations, and so every
routing decision, is the reference's; only the matmul summation order differs
(more exact).  Decision margins are recorded so a mismatch can be told apart
from a near-tie.

The store event log is replayed afterwards through ONE oracle store in session
order (prompts run one after another on one engine; prefill resets the KV cache,
not the store -- engine.py:100-110), with the reference's replay rules
(engine.py:263-313).
"""

from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import fastq as FQ
from . import model as M
from .store import CacheConfig, ExpertStore


def f32(a):
    return np.asarray(a, dtype=np.float32)


@dataclass
class DepthModel:
    """Mixed-quant model: dense tensors (fp16-valued float32 embeddings, lm_head,
    gates; LayerNorm 1/0), quantized attention projections, quantized experts."""

    cfg: M.ModelConfig
    dense: dict
    attn: dict = field(default_factory=dict)      # (layer, "wq") -> fastq prepared block
    experts: dict = field(default_factory=dict)   # (layer, e) -> (W1, W3, W2) prepared

    def gate_matrix(self, layer):
        return self.dense[f"layers.{layer}.gate"]


def mm(block, X):
    """X @ W for a prepared quantized block, float64 accumulation -> float32."""
    return FQ.gemv(block, X).astype(np.float32)


def ln_rows(X, g, b):
    return np.stack([M.layer_norm(x, g, b) for x in X])


@dataclass
class Rec:
    token_pos: int
    layer: int
    experts: tuple
    weights: np.ndarray
    hidden: np.ndarray
    gate_margin: float        # k-th vs (k+1)-th gate logit (routing decision)
    guess_margin: float = np.inf  # m-th vs (m+1)-th next-layer logit (speculation)


@dataclass
class Session:
    tokens: list
    kv: M.KVCache
    pos: int = 0
    recs: list = field(default_factory=list)
    logits: np.ndarray | None = None          # last logits
    prefill_last: np.ndarray | None = None
    out_tokens: list = field(default_factory=list)
    lm_margins: list = field(default_factory=list)


def _margin(logits, k):
    s = np.sort(np.asarray(logits, np.float64))[::-1]
    return float(s[k - 1] - s[k]) if k < s.size else np.inf


class DepthOracle:
    def __init__(self, model: DepthModel, spec_m: int = 0, lookahead: int = 1):
        self.m = model
        self.spec_m, self.lookahead = spec_m, lookahead

    # ---------------------------------------------------------------- pieces
    def _attention(self, layer, X, sess_pos):
        """attention_step for rows X[r] of (session, position) sess_pos[r]
        (model.py:280-301); appends K/V in row order."""
        cfg, d = self.m.cfg, self.m.dense
        pre = f"layers.{layer}"
        N1 = ln_rows(X, d[f"{pre}.ln1.gamma"], d[f"{pre}.ln1.beta"])
        Q = mm(self.m.attn[(layer, "wq")], N1)
        Kp = mm(self.m.attn[(layer, "wk")], N1)
        Vp = mm(self.m.attn[(layer, "wv")], N1)
        H, hd = cfg.n_heads, cfg.head_dim
        ctx = np.empty_like(X)
        for r, (s, pos) in enumerate(sess_pos):
            s.kv.append(layer, Kp[r].reshape(H, hd), Vp[r].reshape(H, hd))
            K, V = s.kv.view(layer)
            q = Q[r].reshape(H, hd)
            sc = np.einsum("hd,thd->ht", q, K) / np.float32(np.sqrt(hd))
            sc = sc - sc.max(axis=1, keepdims=True)
            a = np.exp(sc)
            a = a / a.sum(axis=1, keepdims=True)
            ctx[r] = np.einsum("ht,thd->hd", a, V).reshape(cfg.d_model)
        R = X + mm(self.m.attn[(layer, "wo")], ctx)
        return ln_rows(R, d[f"{pre}.ln2.gamma"], d[f"{pre}.ln2.beta"])

    def _gate(self, layer, h, pos):
        """gate (model.py:198-220) with float64 logits rounded to float32."""
        if not np.all(np.isfinite(h)):
            raise M.NonFiniteError(f"gate input at layer {layer}, position {pos} is not finite")
        G = self.m.gate_matrix(layer)
        logits = f32(h.astype(np.float64) @ G.astype(np.float64))
        k = self.m.cfg.top_k_gate
        sel = M.top_k(logits, k)
        z = logits[sel]
        z = z - z.max()
        ez = np.exp(z)
        w = ez / ez.sum()
        return tuple(int(e) for e in sel), f32(w), _margin(logits, k)

    def _guess_margin(self, layer, h):
        tgt = layer + self.lookahead
        if self.spec_m <= 0 or tgt >= self.m.cfg.n_layers:
            return np.inf
        lg = f32(h.astype(np.float64) @ self.m.gate_matrix(tgt).astype(np.float64))
        return _margin(lg, self.spec_m)

    def _experts(self, layer, H, routes):
        """moe_forward for every row (model.py:238-254): rows grouped by expert,
        one pass per expert matrix; then h + w0*y0 + w1*y1 in order per row."""
        ys = {}
        by_e = {}
        for r, (ex, _) in enumerate(routes):
            for slot, e in enumerate(ex):
                by_e.setdefault(e, []).append((r, slot))
        for e, uses in sorted(by_e.items()):
            W1, W3, W2 = self.m.experts[(layer, e)]
            Hs = H[[r for r, _ in uses]]
            a = mm(W1, Hs)
            b = mm(W3, Hs)
            u = a * M.sigmoid(a) * b                     # model.py:223-226
            y = mm(W2, u)
            for i, (r, slot) in enumerate(uses):
                ys[(r, slot)] = y[i]
        out = np.empty_like(H)
        for r, (ex, w) in enumerate(routes):
            o = H[r]
            for slot in range(len(ex)):
                o = o + w[slot] * ys[(r, slot)]
            out[r] = o
        return out

    def _logits(self, X):
        d = self.m.dense
        N = ln_rows(X, d["ln_f.gamma"], d["ln_f.beta"])
        z = f32(N.astype(np.float64) @ d["lm_head"].astype(np.float64))
        if not np.all(np.isfinite(z)):
            raise M.NonFiniteError("output logits are not finite")
        return z

    def _embed(self, tok, pos):
        return M.embed(SimpleModel(self.m), tok, pos)

    def _layers(self, X, sess_pos):
        for layer in range(self.m.cfg.n_layers):
            H = self._attention(layer, X, sess_pos)
            routes = []
            for r, (s, pos) in enumerate(sess_pos):
                ex, w, gm = self._gate(layer, H[r], pos)
                routes.append((ex, w))
                s.recs.append(Rec(pos, layer, ex, w, H[r].copy(), gm,
                                  self._guess_margin(layer, H[r])))
            X = self._experts(layer, H, routes)
        return X

    # ---------------------------------------------------------------- flows
    def run(self, prompts, n_new: int):
        """Prefill every prompt (model.py:343-367), then n_new greedy tokens
        (engine.py:168-182) per session, all sessions advanced together."""
        cfg = self.m.cfg
        sess = [Session(list(p), M.KVCache(cfg)) for p in prompts]
        rows, X = [], []
        for s in sess:
            for i, t in enumerate(s.tokens):
                rows.append((s, i))
                X.append(self._embed(t, i))
        X = self._layers(np.stack(X), rows)
        Z = self._logits(X)
        for s in sess:
            last = max(r for r, (ss, _) in enumerate(rows) if ss is s)
            s.prefill_last = s.logits = Z[last]
            s.pos = len(s.tokens)
        for _ in range(n_new):
            X, rows = [], []
            for s in sess:
                t = M.sample_greedy(s.logits)
                s.lm_margins.append(_margin(s.logits, 1))
                s.out_tokens.append(t)
                X.append(self._embed(t, s.pos))
                rows.append((s, s.pos))
            X = self._layers(np.stack(X), rows)
            Z = self._logits(X)
            for i, s in enumerate(sess):
                s.logits = Z[i]
                s.pos += 1
        return sess


class SimpleModel:
    """The attributes oracle.model.embed reads."""

    def __init__(self, dm: DepthModel):
        self.config = dm.cfg
        self.params = dm.dense


def replay_sessions(sessions, n_layers, n_experts, cache: CacheConfig, spec_m: int = 0,
                    lookahead: int = 1, gates=None):
    """One store, sessions in order; per session the reference replay rules
    (engine.py:263-313): prompt layers batched with first-use dedupe, generated
    positions token by token with speculative guesses from the recorded h."""
    st = ExpertStore(n_layers, n_experts, cache)
    for s in sessions:
        plen = len(s.tokens)
        by_t = {}
        for r in s.recs:
            by_t.setdefault(r.token_pos, []).append(r)
        for l in range(n_layers):
            seen = set()
            for t in range(plen):
                rec = next(r for r in by_t[t] if r.layer == l)
                for e in rec.experts:
                    if e not in seen:
                        st.acquire(l, e, t)
                        seen.add(e)
        for t in sorted(k for k in by_t if k >= plen):
            for rec in sorted(by_t[t], key=lambda r: r.layer):
                for e in rec.experts:
                    st.acquire(rec.layer, e, t)
                if spec_m > 0 and rec.layer + lookahead < n_layers:
                    g = M.top_k(f32(rec.hidden.astype(np.float64) @
                                    gates[rec.layer + lookahead].astype(np.float64)), spec_m)
                    st.speculative_load([(rec.layer + lookahead, int(e)) for e in g], t,
                                        current_layer=rec.layer)
    return st.events
