"""CPU oracle for the ProphetKV selective-recompute prefill path.

TEST INFRASTRUCTURE ONLY. Nothing in the product package imports this file;
only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py`` (its
``cpu_baseline`` leg and ``--impl reference``) may use it, and only as the
checker / the timed CPU baseline.

This is a numpy restatement of the reference ``pikv`` hot path
(``/root/reference/pkg/src/pikv``).  Every function names the reference
``file:line`` it follows.  The arithmetic contract is the reference's own:
float32 storage, float64 accumulation inside every kernel, float64 RoPE
angles, raw (not renormalised) softmax mass, head-mean before query-mean,
per-layer float32 rounding before the float64 layer mean, ``ceil`` budget
in Python double, stable top-k with ties toward the smaller index.

Parity of this restatement is pinned two ways:
  * ``tests/test_oracle_vs_reference.py`` runs it against the real reference
    package (importable in the build container) and requires bit-identical
    outputs on seeded models;
  * ``tests/golden/*.npz`` hold reference-generated outputs (script
    ``tests/golden/make_golden.py``) that ``tests/test_oracle_golden.py``
    checks on any machine, including the GPU box where the reference is absent.
"""

from __future__ import annotations

import hashlib
import json
import math
from dataclasses import dataclass, field

import numpy as np

f32 = np.float32
f64 = np.float64


class OracleError(Exception):
    """Raised where the reference raises an EngineError subclass."""

    def __init__(self, kind: str, msg: str):
        super().__init__(f"{kind}: {msg}")
        self.kind = kind


# --------------------------------------------------------------------------
# dense kernels (reference: pkg/src/pikv/tensor.py)
# --------------------------------------------------------------------------

def _finite(x, what):
    # tensor.py:31-34 -- every kernel output is finite-checked
    if not np.isfinite(x).all():
        raise OracleError("NumericsError", f"non-finite values in {what}")
    return x


def mm(a, b, macs=None):
    """f32 x f32 -> f32 with float64 accumulation (tensor.py:49-63)."""
    if a.ndim != 2 or b.ndim != 2 or a.shape[1] != b.shape[0]:
        raise OracleError("ShapeError", f"matmul shapes {a.shape} {b.shape}")
    res = (a.astype(f64) @ b.astype(f64)).astype(f32)
    if macs is not None:
        macs[0] += a.shape[0] * a.shape[1] * b.shape[1]
    return _finite(res, "matmul output")


def rmsnorm(x, gain, eps):
    """x / sqrt(mean(x^2) + eps) * gain, in float64 (tensor.py:78-86)."""
    if gain.shape != (x.shape[-1],):
        raise OracleError("ShapeError", "gain shape")
    w = x.astype(f64)
    msq = np.mean(w * w, axis=-1, keepdims=True)
    return _finite((w / np.sqrt(msq + eps) * gain.astype(f64)).astype(f32), "rms_norm output")


def rope_inv_freq(d, theta):
    """theta^(-2i/d) for pair i, float64 (tensor.py:105)."""
    return theta ** (-np.arange(0, d, 2, dtype=f64) / d)


def rope_cos_sin(positions, d, theta):
    """float64 cos/sin tables [t, d/2] for the given positions (tensor.py:104-107).

    The GPU path uploads exactly this table, so device and oracle rotate
    with identical float64 factors.
    """
    ang = np.asarray(positions, dtype=f64)[:, None] * rope_inv_freq(d, theta)[None, :]
    return np.cos(ang), np.sin(ang)


def rope(x, positions, theta):
    """Interleaved-pair rotation of x [t, heads, d] (tensor.py:89-114)."""
    if x.ndim != 3:
        raise OracleError("ShapeError", "rope expects [t, heads, d]")
    t, _, d = x.shape
    if d % 2:
        raise OracleError("ConfigError", "odd rotary dim")
    if np.asarray(positions).shape != (t,):
        raise OracleError("ShapeError", "positions length")
    c, s = rope_cos_sin(positions, d, theta)
    c = c[:, None, :]
    s = s[:, None, :]
    w = x.astype(f64)
    ev, od = w[..., 0::2], w[..., 1::2]
    out = np.empty_like(w)
    out[..., 0::2] = ev * c - od * s
    out[..., 1::2] = ev * s + od * c
    return _finite(out.astype(f32), "rope output")


def topk_ascending(scores, k):
    """k largest, ties toward smaller index, returned ascending (tensor.py:117-133)."""
    v = np.asarray(scores, dtype=f32)
    if v.ndim != 1:
        raise OracleError("ShapeError", "top-k expects 1-D")
    if k < 0 or k > v.shape[0]:
        raise OracleError("ArgumentError", f"bad k={k}")
    _finite(v, "top-k scores")
    order = np.argsort(-v, kind="stable")[:k]
    return sorted(int(i) for i in order)


def budget(p, n):
    """ceil(p*n) in Python double -- float artefacts included (tensor.py:136-140)."""
    if not 0.0 <= p <= 1.0:
        raise OracleError("ArgumentError", f"ratio {p}")
    return math.ceil(p * n)


def bf16_round(x):
    """Round-to-nearest-even to bfloat16, returned as float32 (test adapter)."""
    a = np.ascontiguousarray(x, dtype=f32)
    u = a.view(np.uint32).astype(np.uint64)
    u = (u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000
    return u.astype(np.uint32).view(f32).reshape(a.shape)


# --------------------------------------------------------------------------
# model (reference: pkg/src/pikv/model.py)
# --------------------------------------------------------------------------

@dataclass(frozen=True)
class Cfg:
    """Shape contract (model.py:24-63)."""
    n_layers: int
    n_heads: int
    n_kv_heads: int
    head_dim: int
    hidden_dim: int
    ffn_dim: int
    vocab_size: int
    rope_theta: float = 10000.0
    norm_eps: float = 1e-5

    @property
    def kv_dim(self):
        return self.n_kv_heads * self.head_dim

    def json(self):
        return {k: getattr(self, k) for k in (
            "n_layers", "n_heads", "n_kv_heads", "head_dim", "hidden_dim",
            "ffn_dim", "vocab_size", "rope_theta", "norm_eps")}


@dataclass
class Layer:
    attn_norm: np.ndarray
    wq: np.ndarray
    wk: np.ndarray
    wv: np.ndarray
    wo: np.ndarray
    ffn_norm: np.ndarray
    w_gate: np.ndarray
    w_up: np.ndarray
    w_down: np.ndarray


@dataclass
class Weights:
    embed: np.ndarray
    layers: list
    final_norm: np.ndarray
    lm_head: np.ndarray
    _fp: str | None = field(default=None, repr=False)

    def tensors(self):
        # canonical naming order (model.py:108-123)
        out = [("embed.weight", self.embed)]
        for i, lw in enumerate(self.layers):
            p = f"layers.{i}"
            out += [(f"{p}.attn_norm.gain", lw.attn_norm), (f"{p}.attn.wq", lw.wq),
                    (f"{p}.attn.wk", lw.wk), (f"{p}.attn.wv", lw.wv),
                    (f"{p}.attn.wo", lw.wo), (f"{p}.ffn_norm.gain", lw.ffn_norm),
                    (f"{p}.ffn.w_gate", lw.w_gate), (f"{p}.ffn.w_up", lw.w_up),
                    (f"{p}.ffn.w_down", lw.w_down)]
        out += [("final_norm.gain", self.final_norm), ("lm_head.weight", self.lm_head)]
        return out

    def fingerprint(self, cfg):
        """blake2b-8 of config JSON + (name, f32 bytes) (model.py:147-160)."""
        if self._fp is None:
            h = hashlib.blake2b(digest_size=8)
            h.update(json.dumps(cfg.json(), sort_keys=True).encode())
            for name, t in self.tensors():
                h.update(name.encode())
                h.update(np.ascontiguousarray(t, dtype=f32).tobytes())
            self._fp = h.hexdigest()
        return self._fp

    def rounded_bf16(self):
        """Same weights rounded to bf16 (RNE), kept as float32 -- the shared
        bf16-exact inputs for GPU-vs-oracle parity."""
        r = bf16_round
        return Weights(embed=r(self.embed), final_norm=r(self.final_norm), lm_head=r(self.lm_head),
                       layers=[Layer(**{k: r(getattr(lw, k)) for k in Layer.__dataclass_fields__})
                               for lw in self.layers])


def init_weights(cfg, seed):
    """PCG64 stream identical to random_weights (model.py:163-185)."""
    g = np.random.default_rng(seed)

    def proj(fan_in, fan_out):
        return (g.standard_normal((fan_in, fan_out)) / np.sqrt(fan_in)).astype(f32)

    D, Q, KV, F = cfg.hidden_dim, cfg.n_heads * cfg.head_dim, cfg.kv_dim, cfg.ffn_dim
    layers = []
    for _ in range(cfg.n_layers):
        wq, wk, wv, wo = proj(D, Q), proj(D, KV), proj(D, KV), proj(Q, D)
        wg, wu, wd = proj(D, F), proj(D, F), proj(F, D)
        layers.append(Layer(attn_norm=np.ones(D, f32), wq=wq, wk=wk, wv=wv, wo=wo,
                            ffn_norm=np.ones(D, f32), w_gate=wg, w_up=wu, w_down=wd))
    embed = g.standard_normal((cfg.vocab_size, D)).astype(f32)
    head = proj(D, cfg.vocab_size)
    return Weights(embed=embed, layers=layers, final_norm=np.ones(D, f32), lm_head=head)


def _ids(tokens, cfg):
    # model.py:231-237
    a = np.asarray(tokens, dtype=np.int64)
    if a.ndim != 1 or a.shape[0] == 0:
        raise OracleError("InputError", "empty token sequence")
    if a.min() < 0 or a.max() >= cfg.vocab_size:
        raise OracleError("InputError", "token id out of range")
    return a


def masked_softmax64(scores, visible):
    """Row softmax over visible entries in float64 -> f32 (model.py:247-257)."""
    z = scores.astype(f64)
    z[~visible] = -np.inf
    mx = z.max(axis=1, keepdims=True)
    if not np.isfinite(mx).all():
        raise OracleError("NumericsError", "attention row with no visible entry")
    e = np.exp(z - mx)
    e[~visible] = 0.0
    return (e / e.sum(axis=1, keepdims=True)).astype(f32)


def qkv_proj(lw, cfg, x, pos, macs):
    """(q_rot, k_raw, k_rot, v) from normalised x (model.py:265-275)."""
    n = x.shape[0]
    q = mm(x, lw.wq, macs).reshape(n, cfg.n_heads, cfg.head_dim)
    k = mm(x, lw.wk, macs).reshape(n, cfg.n_kv_heads, cfg.head_dim)
    qr = rope(q, pos, cfg.rope_theta)
    kr = rope(k, pos, cfg.rope_theta)
    v = mm(x, lw.wv, macs).reshape(n, cfg.n_kv_heads, cfg.head_dim)
    return qr, k, kr, v


def attention(cfg, qr, K, V, pos_q, pos_kv, macs, score_macs, want_rows):
    """GQA causal attention by position (model.py:278-308).

    Returns concatenated heads [n, H*dk] and, optionally, head-mean rows [n, t].
    """
    n, H, dk = qr.shape
    t = K.shape[0]
    grp = H // cfg.n_kv_heads
    visible = pos_kv[None, :] <= pos_q[:, None]
    scl = f32(1.0 / np.sqrt(dk))
    out = np.empty((n, H, dk), dtype=f32)
    acc = np.zeros((n, t), dtype=f64) if want_rows else None
    for h in range(H):
        g = h // grp
        sc = mm(qr[:, h, :], np.ascontiguousarray(K[:, g, :].T), macs) * scl
        if score_macs is not None:
            score_macs[0] += n * dk * t
        p = masked_softmax64(sc, visible)
        out[:, h, :] = mm(p, np.ascontiguousarray(V[:, g, :]), macs)
        if acc is not None:
            acc += p
    rows = (acc / H).astype(f32) if acc is not None else None
    return out.reshape(n, H * dk), rows


def silu(x):
    # model.py:260-262
    w = x.astype(f64)
    return (w / (1.0 + np.exp(-w))).astype(f32)


def block_tail(lw, cfg, h, qr, K, V, pos_q, pos_kv, macs, score_macs, want_rows=False):
    """Attention + o-proj residual + SiLU FFN residual (model.py:311-323)."""
    a, rows = attention(cfg, qr, K, V, pos_q, pos_kv, macs, score_macs, want_rows)
    h = h + mm(a, lw.wo, macs)
    y = rmsnorm(h, lw.ffn_norm, cfg.norm_eps)
    g = silu(mm(y, lw.w_gate, macs))
    u = mm(y, lw.w_up, macs)
    h = h + mm(g * u, lw.w_down, macs)
    return h, rows


def logits_of(w, cfg, h, macs):
    # model.py:326-329
    return mm(rmsnorm(h, w.final_norm, cfg.norm_eps), w.lm_head, macs)


@dataclass
class Prefill:
    tokens: np.ndarray
    keys: list            # rotated, per layer [n, Hkv, dk]
    values: list
    keys_norope: list
    logits: np.ndarray
    rows: list | None


def prefill(w, cfg, tokens, want_rows=False, macs=None, score_macs=None):
    """Whole-sequence forward at positions 0..n-1 (model.py:332-359)."""
    ids = _ids(tokens, cfg)
    pos = np.arange(ids.shape[0], dtype=np.int64)
    h = w.embed[ids].copy()
    ks, vs, knr, rws = [], [], [], []
    for lw in w.layers:
        x = rmsnorm(h, lw.attn_norm, cfg.norm_eps)
        qr, k, kr, v = qkv_proj(lw, cfg, x, pos, macs)
        h, rows = block_tail(lw, cfg, h, qr, kr, v, pos, pos, macs, score_macs, want_rows)
        ks.append(kr)
        vs.append(v)
        knr.append(k)
        rws.append(rows)
    return Prefill(tokens=ids, keys=ks, values=vs, keys_norope=knr,
                   logits=logits_of(w, cfg, h, macs), rows=rws if want_rows else None)


@dataclass
class QueryOut:
    last_logits: np.ndarray
    rows: list | None
    fresh_k: list
    fresh_v: list


def narrow_pass(w, cfg, kv_layers, kv_pos, query, want_rows=False, macs=None, score_macs=None):
    """Query tokens at positions t..t+m-1 over a fixed KV state (model.py:370-402)."""
    ids = _ids(query, cfg)
    m = ids.shape[0]
    t = int(kv_pos.shape[0])
    pq = t + np.arange(m, dtype=np.int64)
    pall = np.concatenate([kv_pos, pq])
    h = w.embed[ids].copy()
    rws, fk, fv = [], [], []
    for li, lw in enumerate(w.layers):
        x = rmsnorm(h, lw.attn_norm, cfg.norm_eps)
        qr, _, kr, v = qkv_proj(lw, cfg, x, pq, macs)
        ck, cv = kv_layers[li]
        h, rows = block_tail(lw, cfg, h, qr, np.concatenate([ck, kr], axis=0),
                             np.concatenate([cv, v], axis=0), pq, pall, macs, score_macs, want_rows)
        rws.append(rows)
        fk.append(kr)
        fv.append(v)
    lg = logits_of(w, cfg, h, macs)
    return QueryOut(last_logits=lg[-1], rows=rws if want_rows else None, fresh_k=fk, fresh_v=fv)


# --------------------------------------------------------------------------
# chunk store + assembly (reference: pkg/src/pikv/chunkstore.py)
# --------------------------------------------------------------------------

def content_id(fp, token_ids):
    # chunkstore.py:29-34
    h = hashlib.blake2b(digest_size=8)
    h.update(fp.encode())
    h.update(np.asarray(token_ids, dtype=np.int64).tobytes())
    return int.from_bytes(h.digest(), "little")


@dataclass
class Chunk:
    chunk_id: int
    fp: str
    token_ids: np.ndarray
    k_nr: list      # per layer [t, Hkv, dk], unrotated
    v: list


def make_chunk(w, cfg, tokens):
    """Isolated prefill; keys stored before rotation (chunkstore.py:52-62)."""
    tr = prefill(w, cfg, tokens)
    fp = w.fingerprint(cfg)
    return Chunk(chunk_id=content_id(fp, tr.tokens), fp=fp, token_ids=tr.tokens,
                 k_nr=tr.keys_norope, v=tr.values)


@dataclass
class Cache:
    fp: str
    token_ids: np.ndarray
    positions: np.ndarray
    chunk_ids: list
    bounds: list
    source_chunk: np.ndarray
    source_local: np.ndarray
    keys: list
    values: list
    recomputed: np.ndarray
    finalized: bool = False

    @property
    def s(self):
        return int(self.token_ids.shape[0])

    def kv(self):
        return [(self.keys[i], self.values[i]) for i in range(len(self.keys))]


def stitch(chunks, cfg):
    """Concatenate chunk KV and rotate keys at global positions (chunkstore.py:99-140)."""
    if not chunks:
        raise OracleError("InputError", "no chunks")
    fp = chunks[0].fp
    for c in chunks:
        if c.fp != fp:
            raise OracleError("IncompatibleError", "fingerprint mismatch")
        if len(c.k_nr) != cfg.n_layers:
            raise OracleError("IncompatibleError", "layer count")
    ids = np.concatenate([c.token_ids for c in chunks])
    s = ids.shape[0]
    pos = np.arange(s, dtype=np.int64)
    lens = [int(c.token_ids.shape[0]) for c in chunks]
    starts = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(int)
    bounds = [(int(a), int(a + n)) for a, n in zip(starts, lens)]
    src_c = np.concatenate([np.full(n, i, dtype=np.int32) for i, n in enumerate(lens)])
    src_l = np.concatenate([np.arange(n, dtype=np.int32) for n in lens])
    keys = [rope(np.concatenate([c.k_nr[li] for c in chunks], axis=0), pos, cfg.rope_theta)
            for li in range(cfg.n_layers)]
    vals = [np.concatenate([c.v[li] for c in chunks], axis=0) for li in range(cfg.n_layers)]
    return Cache(fp=fp, token_ids=ids, positions=pos, chunk_ids=[c.chunk_id for c in chunks],
                 bounds=bounds, source_chunk=src_c, source_local=src_l, keys=keys, values=vals,
                 recomputed=np.zeros((cfg.n_layers, s), dtype=bool))


def overwrite(cache, layer, idx, new_k, new_v):
    """In-place scatter of fresh K/V at one layer (chunkstore.py:143-160)."""
    if not 0 <= layer < len(cache.keys):
        raise OracleError("ArgumentError", "layer out of range")
    ix = np.asarray(idx, dtype=np.int64)
    if ix.ndim != 1:
        raise OracleError("ShapeError", "indices must be 1-D")
    if ix.size and (ix.min() < 0 or ix.max() >= cache.s):
        raise OracleError("InputError", "replacement index out of range")
    want = (ix.shape[0],) + cache.keys[layer].shape[1:]
    if new_k.shape != want or new_v.shape != want:
        raise OracleError("ShapeError", "replacement shape")
    cache.keys[layer][ix] = new_k
    cache.values[layer][ix] = new_v
    cache.recomputed[layer, ix] = True


# --------------------------------------------------------------------------
# scoring, fusion, selection (reference: pkg/src/pikv/selection.py)
# --------------------------------------------------------------------------

def layer_mean(per_layer):
    """Uniform float64 mean over layers -> f32 (selection.py:52-54)."""
    return per_layer.astype(f64).mean(axis=0).astype(f32)


def prophet_scores(w, cfg, cache, query, renorm=False, macs=None, score_macs=None):
    """Stage I: per-layer query->context attention mass (selection.py:64-86).

    Returns (per_layer [L, s] f32, fused [s] f32).
    """
    res = narrow_pass(w, cfg, cache.kv(), cache.positions, query, want_rows=True,
                      macs=macs, score_macs=score_macs)
    s = cache.s
    per = np.empty((cfg.n_layers, s), dtype=f32)
    for li, rows in enumerate(res.rows):
        ctx = rows[:, :s].astype(f64)
        if renorm:
            ctx = ctx / np.maximum(ctx.sum(axis=1, keepdims=True), 1e-30)
        per[li] = ctx.mean(axis=0).astype(f32)
    return per, layer_mean(per)


def low_layer_probe(w, cfg, cache, macs=None, score_macs=None):
    """Block 0 for every context token over the assembled layer-0 cache, then the fresh
    layer-1 values (selection.py:95-124): (dv [s, kv_dim] f64, attention column sums [s] f64)."""
    s = cache.s
    h = w.embed[cache.token_ids].copy()
    lw = w.layers[0]
    x = rmsnorm(h, lw.attn_norm, cfg.norm_eps)
    qr, _, _, _ = qkv_proj(lw, cfg, x, cache.positions, macs)
    h, rows = block_tail(lw, cfg, h, qr, cache.keys[0], cache.values[0], cache.positions, cache.positions, macs,
                         score_macs, want_rows=True)
    colsum = rows.astype(f64).sum(axis=0)
    if cfg.n_layers == 1:
        return np.zeros((s, cfg.kv_dim), dtype=f64), colsum
    lw1 = w.layers[1]
    x1 = rmsnorm(h, lw1.attn_norm, cfg.norm_eps)
    v1 = mm(x1, lw1.wv, macs)
    dv = v1.astype(f64) - cache.values[1].reshape(s, cfg.kv_dim).astype(f64)
    return dv, colsum


def cacheblend_l1(w, cfg, cache, macs=None, score_macs=None):
    """alpha = ||dV||_2 per token (selection.py:127-133); the layer-mean of identical rows."""
    dv, _ = low_layer_probe(w, cfg, cache, macs, score_macs)
    return np.linalg.norm(dv, axis=1).astype(f32)


def kvshare_l1(w, cfg, cache, macs=None, score_macs=None):
    """Attention column sums times ||dV||_1 (selection.py:136-142)."""
    dv, colsum = low_layer_probe(w, cfg, cache, macs, score_macs)
    return (colsum * np.abs(dv).sum(axis=1)).astype(f32)


def select(fused, p):
    """(indices ascending, k) for ratio p (selection.py:57-61)."""
    k = budget(p, fused.shape[0])
    return topk_ascending(fused, k), k


# --------------------------------------------------------------------------
# Stage II + finalize (reference: pkg/src/pikv/recompute.py)
# --------------------------------------------------------------------------

def repair(w, cfg, cache, sel, macs=None, score_macs=None, capture=None):
    """Fresh-peer selective recompute, in place (recompute.py:43-82).

    ``capture`` (optional dict) receives per-layer fresh K/V at the selection
    (f32, before any storage rounding) -- the oracle side of the K/V parity tap.
    """
    if cache.finalized:
        raise OracleError("StateError", "finalized")
    if cache.recomputed.any():
        raise OracleError("StateError", "already repaired")
    ix = np.asarray(sel, dtype=np.int64)
    if ix.size == 0:
        return cache
    if not np.all(np.diff(ix) > 0):
        raise OracleError("ArgumentError", "selection not strictly ascending")
    ps = cache.positions[ix]
    h = w.embed[cache.token_ids[ix]].copy()
    for li, lw in enumerate(w.layers):
        x = rmsnorm(h, lw.attn_norm, cfg.norm_eps)
        qr, _, kr, v = qkv_proj(lw, cfg, x, ps, macs)
        overwrite(cache, li, ix, kr, v)          # write first (recompute.py:63)
        if capture is not None:
            capture.setdefault("k", []).append(kr.copy())
            capture.setdefault("v", []).append(v.copy())
        K, V = cache.keys[li], cache.values[li]  # then read the updated layer
        h, _ = block_tail(lw, cfg, h, qr, K, V, ps, cache.positions, macs, score_macs)
    return cache


def finalize(w, cfg, cache, query, want_rows=False, macs=None, score_macs=None):
    """One-shot query pass over the repaired cache (recompute.py:105-125).

    Returns (first_logits [V], QueryOut).
    """
    if cache.finalized:
        raise OracleError("StateError", "already finalized")
    cache.finalized = True
    res = narrow_pass(w, cfg, cache.kv(), cache.positions, query, want_rows=want_rows,
                      macs=macs, score_macs=score_macs)
    return res.last_logits, res


def decode(w, cfg, kv_layers, kv_pos, tokens):
    """Teacher-forced decode steps (model.py:405-441): each token attends to the KV state
    plus its own fresh K/V, which is then appended.  Returns per-step logits."""
    ks = [np.array(k) for k, _ in kv_layers]
    vs = [np.array(v) for _, v in kv_layers]
    pos = np.array(kv_pos, dtype=np.int64)
    out = []
    for t in tokens:
        res = narrow_pass(w, cfg, list(zip(ks, vs)), pos, [int(t)])
        out.append(res.last_logits)
        ks = [np.concatenate([k, fk], axis=0) for k, fk in zip(ks, res.fresh_k)]
        vs = [np.concatenate([v, fv], axis=0) for v, fv in zip(vs, res.fresh_v)]
        pos = np.concatenate([pos, [pos.shape[0]]])
    return out


# --------------------------------------------------------------------------
# MAC books (reference FlopTally semantics, model.py:188-193; formulas in
# SURVEY.md Appendix B, verified against the reference tallies)
# --------------------------------------------------------------------------

def macs_query_pass(cfg, s, m):
    """(total, attn_scores) MACs of one narrow pass of m tokens over s entries."""
    H, dk, D, F, KV = cfg.n_heads, cfg.head_dim, cfg.hidden_dim, cfg.ffn_dim, cfg.kv_dim
    t = s + m
    per = m * D * (H * dk + 2 * KV) + 2 * H * m * dk * t + m * H * dk * D + 3 * m * D * F
    return cfg.n_layers * per + m * D * cfg.vocab_size, cfg.n_layers * H * m * dk * t


def macs_repair(cfg, s, k):
    """(total, attn_scores) MACs of the repair of k tokens over an s-entry cache."""
    if k == 0:
        return 0, 0
    H, dk, D, F, KV = cfg.n_heads, cfg.head_dim, cfg.hidden_dim, cfg.ffn_dim, cfg.kv_dim
    per = k * D * (H * dk + 2 * KV) + 2 * H * k * dk * s + k * H * dk * D + 3 * k * D * F
    return cfg.n_layers * per, cfg.n_layers * H * k * dk * s


def macs_probe(cfg, s):
    """MACs the reference books for one low-layer probe over s context tokens: block 0 with
    dense s x s attention, plus the layer-1 value projection when there is a layer 1."""
    H, dk, D, F, KV = cfg.n_heads, cfg.head_dim, cfg.hidden_dim, cfg.ffn_dim, cfg.kv_dim
    block0 = s * D * (H * dk + 2 * KV) + 2 * H * s * dk * s + s * H * dk * D + 3 * s * D * F
    return block0 + (s * D * KV if cfg.n_layers > 1 else 0)


def prophet_ttft_slice(w, cfg, chunks, query, p):
    """The timed reference slice assemble -> score -> select -> repair -> finalize.

    Used as the CPU baseline (bench.py) and by end-to-end parity tests.
    Returns a dict of the slice's outputs.
    """
    cache = stitch(chunks, cfg)
    per, fused = prophet_scores(w, cfg, cache, query)
    sel, k = select(fused, p)
    cap = {}
    repair(w, cfg, cache, sel, capture=cap)
    logits, _ = finalize(w, cfg, cache, query)
    return {"per_layer": per, "fused": fused, "sel": sel, "k": k, "fresh": cap,
            "first_logits": logits, "cache": cache}
