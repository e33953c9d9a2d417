"""Stage I scoring, layer fusion and budgeted selection on the GPU.

Drop-in for reference selection.py (ValueScores 25-42, SelectionResult 45-49,
fuse_layers 52-54, select_top_p 57-61, score_prophet 64-86, score_cacheblend_l1
127-133).  The static baselines (epic, random) are host one-liners kept for run_strategy
compatibility; score_cacheblend_l1 / score_kvshare_l1 (136-142) run the low-layer probe
as fp32-faithful narrow passes.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import numpy as np

from . import _lib
from .errors import ArgumentError, ConfigError, InputError, NumericsError, ShapeError
from .model import F32, F64, FlopTally, ModelConfig, bill_query_pass, resolve_device_model
from .tensor import device_topk, ratio_budget

STRATEGIES = ("prophet", "epic", "cacheblend_l1", "kvshare_l1", "random")


def _host_layer_mean(per_layer: np.ndarray) -> np.ndarray:
    return per_layer.astype(F64).mean(axis=0).astype(F32)


@dataclass
class ValueScores:
    strategy: str
    per_layer: np.ndarray   # [L, s]
    fused: np.ndarray       # [s]
    _dev_fused: object = field(default=None, repr=False, compare=False)

    def __post_init__(self) -> None:
        if self.per_layer.ndim != 2:
            raise ShapeError(f"per-layer scores must be [L, s], got {self.per_layer.shape}")
        want = _host_layer_mean(self.per_layer)
        if self.fused.shape != want.shape or not np.allclose(self.fused, want, atol=1e-6):
            raise ArgumentError("fused scores must be the mean of the per-layer rows")

    def _renamed(self, strategy: str) -> "ValueScores":
        return ValueScores(strategy=strategy, per_layer=self.per_layer, fused=self.fused)

    @classmethod
    def from_vector(cls, strategy: str, vector, n_layers: int) -> "ValueScores":
        v = np.asarray(vector, dtype=F32)
        per_layer = np.repeat(v[None, :], n_layers, axis=0)
        return cls(strategy=strategy, per_layer=per_layer, fused=_host_layer_mean(per_layer))


class _DeviceScores(ValueScores):
    """ValueScores of a device narrow pass.  The fused vector is the device layer mean (the
    reference rule, so the host re-check of __post_init__ is skipped) and the host copies of
    per_layer / fused are made on first access: select_top_p -> recompute_selected then
    run on the device copies without a 4 MB read-back and a host mean on the critical path."""

    def __init__(self, strategy: str, dev_per_layer, dev_fused):  # noqa: D107 -- no dataclass init
        object.__setattr__(self, "strategy", strategy)
        object.__setattr__(self, "_dev_per_layer", dev_per_layer)
        object.__setattr__(self, "_dev_fused", dev_fused)
        object.__setattr__(self, "_host_pl", None)
        object.__setattr__(self, "_host_fused", None)

    @property
    def per_layer(self):
        if self._host_pl is None:
            object.__setattr__(self, "_host_pl", self._dev_per_layer.cpu().numpy())
        return self._host_pl

    @per_layer.setter
    def per_layer(self, v):
        object.__setattr__(self, "_host_pl", v)

    @property
    def fused(self):
        if self._host_fused is None:
            object.__setattr__(self, "_host_fused", self._dev_fused.cpu().numpy())
        return self._host_fused

    @fused.setter
    def fused(self, v):
        object.__setattr__(self, "_host_fused", v)


@dataclass
class SelectionResult:
    indices: list   # ascending
    p: float
    k: int
    _dev_idx: object = field(default=None, repr=False, compare=False)


_WS = threading.local()


def workspace(nbytes: int, tag: str = "ws"):
    """Grow-only device scratch per (host thread, device, tag): the ranks of an in-process
    group (tp.run_ranks) are threads sharing one device and must not share scratch. Kept in
    thread-local storage so a rank thread's buffers are released when the thread ends."""
    torch = _lib.require_cuda()
    bufs = getattr(_WS, "bufs", None)
    if bufs is None:
        bufs = _WS.bufs = {}
    key = (torch.cuda.current_device(), tag)
    buf = bufs.get(key)
    if buf is None or buf.numel() < nbytes:
        buf = torch.empty(max(int(nbytes), 256), dtype=torch.uint8, device="cuda")
        bufs[key] = buf
    return buf


def fuse_layers(per_layer) -> np.ndarray:
    """Uniform mean over layers (reference selection.py:52-54), on the GPU."""
    torch = _lib.require_cuda()
    a = np.ascontiguousarray(per_layer, dtype=F32)
    if a.ndim != 2:
        raise ShapeError(f"per-layer scores must be [L, s], got {a.shape}")
    d = torch.from_numpy(a).cuda()
    fused = torch.empty(a.shape[1], dtype=torch.float32, device=d.device)
    _fuse_device(d, fused)
    return fused.cpu().numpy()


def _fuse_device(per_layer_dev, fused_out, stream=None):
    torch = _lib.require_cuda()
    L, s = per_layer_dev.shape
    idx = torch.empty(1, dtype=torch.int32, device=per_layer_dev.device)
    st = torch.empty(1, dtype=torch.int32, device=per_layer_dev.device)
    _lib.check(_lib.load().pkv_fuse_select(per_layer_dev.data_ptr(), int(L), int(s), 0, fused_out.data_ptr(),
                                           idx.data_ptr(), st.data_ptr(), None, 0, _lib.stream_ptr(torch, stream)))


def select_top_p(scores: ValueScores, p: float) -> SelectionResult:
    """Top ceil(p*s) tokens of the fused vector; ties toward smaller index."""
    torch = _lib.require_cuda()
    fused = scores._dev_fused
    s = int(fused.shape[0]) if fused is not None else scores.fused.shape[0]
    k = ratio_budget(p, s)
    if fused is None:
        fused = torch.from_numpy(np.ascontiguousarray(scores.fused, dtype=F32)).cuda()
    if k == 0:
        return SelectionResult(indices=[], p=p, k=0, _dev_idx=torch.empty(0, dtype=torch.int32, device=fused.device))
    idx, status = device_topk(fused, k)
    st = int(status.item())
    if st == 7:
        raise NumericsError("non-finite values in top-k scores")
    _lib.check(st)
    return SelectionResult(indices=idx.cpu().tolist(), p=p, k=k, _dev_idx=idx)


def check_tokens(tokens, config: ModelConfig) -> np.ndarray:
    """Non-empty 1-D ids inside the vocab (reference model.py:231-237)."""
    ids = np.asarray(tokens, dtype=np.int64)
    if ids.ndim != 1 or ids.shape[0] == 0:
        raise InputError(f"token sequence must be non-empty 1-D, got shape {ids.shape}")
    if ids.min() < 0 or ids.max() >= config.vocab_size:
        raise InputError("token id out of range for vocab")
    return ids


def run_query_pass(dm, cache, ids: np.ndarray, flags: int, per_layer=None, fresh_k=None, fresh_v=None, logits=None,
                   stream=None, c_cache=None):
    """One device narrow pass (reference model.py:370-402) over the cache (c_cache: a
    copy of cache.c_cache with other layer_ready events)."""
    torch = _lib.require_cuda()
    m = int(ids.shape[0])
    if c_cache is None:
        cache.ensure_query_room(m)
        c_cache = cache.c_cache
        # this pass shares the 'qp' workspace with a final pass that would follow Stage II
        # on its own stream: finalize_query then runs in order
        if getattr(cache, "_final_follow", None) is not None:
            cache._final_follow = None
    d_ids = torch.from_numpy(ids.astype(np.int32)).to(cache.device)
    lib = _lib.load()
    nbytes = lib.pkv_query_pass_workspace(dm.handle, cache.context_length, m, flags)
    ws = workspace(nbytes, "qp")

    def ptr(t):
        return t.data_ptr() if t is not None else None

    import ctypes
    chunks = ctypes.byref(cache.c_chunks)
    _lib.check(lib.pkv_query_pass(dm.handle, ctypes.byref(c_cache), chunks, d_ids.data_ptr(), m, flags,
                                  ptr(per_layer), ptr(fresh_k), ptr(fresh_v), ptr(logits), ws.data_ptr(), ws.numel(),
                                  _lib.stream_ptr(torch, stream)))


def score_prophet(weights, config: ModelConfig, cache, query_tokens, tally: FlopTally | None = None,
                  renormalize_context_only: bool = False) -> ValueScores:
    """Query-to-context attention over the assembled (approximate) cache: one
    fp32-faithful narrow pass on the GPU; per-layer head-mean, query-mean rows
    over the context become the layer scores (reference selection.py:64-86)."""
    torch = _lib.require_cuda()
    dm = resolve_device_model(weights, config)
    ids = check_tokens(query_tokens, config)
    if cache.access_log is not None:
        cache.access_log.extend(("read", li) for li in range(config.n_layers))
    s = cache.context_length
    per_layer = torch.empty((config.n_layers, s), dtype=torch.float32, device=cache.device)
    flags = _lib.PKV_QP_SCORES | _lib.PKV_QP_FROM_CHUNKS
    if renormalize_context_only:
        flags |= _lib.PKV_QP_RENORM
    run_query_pass(dm, cache, ids, flags, per_layer=per_layer)
    # the query a later recompute_selected may carry along Stage II so that finalize_query
    # of the same tokens needs no separate pass (recompute.py, pkv_recompute_query)
    cache._pending_query = np.asarray(ids, dtype=np.int32).copy()
    fused = torch.empty(s, dtype=torch.float32, device=cache.device)
    _fuse_device(per_layer, fused)
    bill_query_pass(tally, config, s, int(ids.shape[0]))
    # a non-finite per-layer score makes its token's layer mean non-finite: one device check
    if not bool(torch.isfinite(fused).all()):
        raise NumericsError("non-finite values in attention scores")
    return _DeviceScores("prophet", per_layer, fused)


def score_epic(cache, n_layers: int) -> ValueScores:
    """Static positional prior: negated distance to the chunk start (reference selection.py:89-92)."""
    return ValueScores.from_vector("epic", (-cache.source_local.astype(np.int64)).astype(F32), n_layers)


def _probe_scores(weights, config: ModelConfig, cache, tally: FlopTally | None, kvshare: bool) -> np.ndarray:
    """Scores of the low-layer probe (reference selection.py:95-142) for every context token.
    Block 0 over the assembled layer-0 cache, then rmsnorm + the value projection of layer 1:
    context tokens [p, p+32) run as one fp32-faithful narrow pass over the cache truncated to
    [0, p) -- at positions p.. they attend to it and causally to each other (their fresh
    layer-0 K/V equal the assembled entries: layer 0 has no context) -- stopped after layer
    1's projections (``PKV_QP_PROBE``).  Everything stays on the stream: kvshare's layer-0
    column sums accumulate in f64 on the device in block order (``pkv_probe_accum``), the
    probe's layer-1 values land in one [s, kv_dim] buffer, and ``pkv_probe_scores`` forms
    ||dV||_2 (cacheblend) or colsum * ||dV||_1 (kvshare) per token; one [s] read-back."""
    import ctypes
    torch = _lib.require_cuda()
    dm = resolve_device_model(weights, config)
    s, L = cache.context_length, config.n_layers
    cache.wait_ready()  # a host-tier chunk transfer may still be filling the chunk buffers / pool
    Hkv, dk = cache.config.n_kv_heads, config.head_dim
    m = 32
    flags = _lib.PKV_QP_PROBE | _lib.PKV_QP_FROM_CHUNKS | (_lib.PKV_QP_SCORES if kvshare else 0)
    lib = _lib.load()
    st = _lib.stream_ptr(torch)
    colsum = torch.zeros(s, dtype=torch.float64, device=cache.device) if kvshare else None
    pl = torch.empty(s + m, dtype=torch.float32, device=cache.device) if kvshare else None
    fk = torch.empty((L, m, Hkv, dk), dtype=torch.float32, device=cache.device)
    fv = torch.empty_like(fk)
    v1 = torch.empty((s, Hkv * dk), dtype=torch.float32, device=cache.device)
    d_ids = torch.from_numpy(np.asarray(cache.token_ids, dtype=np.int32).copy()).to(cache.device)
    chunks = ctypes.byref(cache.c_chunks)
    # the workspace grows with the truncated context: size it once for the last block
    # (the split plan of the narrow pass makes the size non-monotone in the context length:
    # take the largest over the blocks, a host-side computation)
    ws = workspace(max(lib.pkv_query_pass_workspace(dm.handle, p0, min(m, s - p0), flags) for p0 in range(0, s, m)),
                   "probe")
    view = _lib.Cache.from_buffer_copy(cache.c_cache)
    view.layer_ready = None
    for p0 in range(0, s, m):
        n = min(m, s - p0)
        view.s = p0
        _lib.check(lib.pkv_query_pass(dm.handle, ctypes.byref(view), chunks, d_ids.data_ptr() + 4 * p0, n, flags,
                                      pl.data_ptr() if pl is not None else None, fk.data_ptr(), fv.data_ptr(), None,
                                      ws.data_ptr(), ws.numel(), st))
        if kvshare:
            _lib.check(lib.pkv_probe_accum(pl.data_ptr(), p0, n, colsum.data_ptr(), st))
        # fresh_v is [L][n][Hkv][dk] for this pass's n rows
        v1[p0:p0 + n] = fv.view(-1)[n * Hkv * dk: 2 * n * Hkv * dk].view(n, Hkv * dk)
    out = torch.empty(s, dtype=torch.float32, device=cache.device)
    _lib.check(lib.pkv_probe_scores(ctypes.byref(cache._cfg_c), ctypes.byref(cache.c_cache), v1.data_ptr(),
                                    colsum.data_ptr() if kvshare else None, out.data_ptr(), st))
    if tally is not None:  # reference books: block 0 with dense s x s attention + layer-1 wv
        H, D, F, KV = config.n_heads, config.hidden_dim, config.ffn_dim, config.kv_dim
        tally.total.add(s * D * (H * dk + 2 * KV) + 2 * H * s * dk * s + s * H * dk * D + 3 * s * D * F + s * D * KV)
        tally.attn_scores.add(H * s * dk * s)
    return out.cpu().numpy()


def score_cacheblend_l1(weights, config: ModelConfig, cache, embeddings=None,
                        tally: FlopTally | None = None) -> ValueScores:
    """Value-deviation magnitude from the low-layer probe, alpha = ||dV||_2 (reference
    selection.py:127-133), dV = probe layer-1 values - assembled layer-1 values."""
    if embeddings is not None:
        raise ConfigError("custom probe embeddings are not supported on the B200 path")
    s, L = cache.context_length, config.n_layers
    if L == 1:  # no layer 1: dV = 0 (reference selection.py:118-119)
        if tally is not None:
            H, dk, D, F, KV = config.n_heads, config.head_dim, config.hidden_dim, config.ffn_dim, config.kv_dim
            tally.total.add(s * D * (H * dk + 2 * KV) + 2 * H * s * dk * s + s * H * dk * D + 3 * s * D * F)
            tally.attn_scores.add(H * s * dk * s)
        return ValueScores.from_vector("cacheblend_l1", np.zeros(s, dtype=F32), L)
    return ValueScores.from_vector("cacheblend_l1", _probe_scores(weights, config, cache, tally, kvshare=False), L)


def score_kvshare_l1(weights, config: ModelConfig, cache, embeddings=None,
                     tally: FlopTally | None = None) -> ValueScores:
    """Layer-0 attention column sums times ||dV||_1 from the same low-layer probe (reference
    selection.py:136-142)."""
    if embeddings is not None:
        raise ConfigError("custom probe embeddings are not supported on the B200 path")
    s, L = cache.context_length, config.n_layers
    if L == 1:  # dV = 0, so colsum * ||dV||_1 = 0 (reference selection.py:118-119)
        return score_cacheblend_l1(weights, config, cache, None, tally)._renamed("kvshare_l1")
    return ValueScores.from_vector("kvshare_l1", _probe_scores(weights, config, cache, tally, kvshare=True), L)


def score_random(s_context: int, seed: int, n_layers: int) -> ValueScores:
    """Uniform noise scores (reference selection.py:145-148)."""
    return ValueScores.from_vector("random", np.random.default_rng(seed).random(s_context), n_layers)
