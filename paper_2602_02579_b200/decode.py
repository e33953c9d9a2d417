"""Decoding after the first token on the device: reference
model.decode_step / greedy_generate (model.py:405-471).

A decode step is the fp32-faithful narrow pass with one query row (include/pkv.h
``pkv_query_pass``, flags LOGITS | APPEND_KV) over every cache entry so far -- the
assembled/repaired context, the finalized query and the tokens generated since, all in
the paged pool with their f32 keys (fp16 key + residual plane) -- appending
the new token's K/V at position ``cache.length``.  A KVCache from ``finalize_query``
keeps its device pools; a host KVCache (e.g. ``KVCache.from_prefill``) is uploaded once
(keys split into the fp16 key and its residual plane by ``pkv_replace_entries``).
"""

from __future__ import annotations

from dataclasses import dataclass

import numpy as np

from . import _lib
from .chunkstore import PAGE, QUERY_RESERVE, ctypes_ref, rope_device_tables
from .errors import StateError
from .model import FlopTally, KVCache, ModelConfig, bill_query_pass, resolve_device_model
from .selection import check_tokens, workspace


@dataclass
class GenerationResult:
    """Reference model.GenerationResult."""

    tokens: list
    step_attn: list | None = None


class DevicePools:
    """Paged fp16 K/V pools (+ key residual plane) holding `length` entries at positions
    0..length-1, with room to append; the device side of a decoding KVCache."""

    def __init__(self, config: ModelConfig, device, capacity: int):
        self.config = config
        self.device = device
        self.length = 0
        self._alloc(max(capacity, 1))

    def _alloc(self, capacity: int):
        torch = _lib.require_cuda()
        cfg = self.config
        self.pool_tokens = -(-capacity // PAGE) * PAGE
        shape = (cfg.n_layers, cfg.n_kv_heads, self.pool_tokens, cfg.layout().dkp)
        old = [getattr(self, n, None) for n in ("k_pool", "v_pool", "k2_pool")]
        self.k_pool, self.v_pool, self.k2_pool = (
            torch.zeros(shape, dtype=torch.float16, device=self.device) for _ in range(3))
        for new, o in zip((self.k_pool, self.v_pool, self.k2_pool), old):
            if o is not None:
                new[:, :, : o.shape[2]] = o
        self.pages = torch.arange(self.pool_tokens // PAGE, dtype=torch.int32, device=self.device)
        self.rope_len, self.rcos, self.rsin, self.rcs32 = rope_device_tables(cfg.rope_theta, cfg.head_dim,
                                                                            self.pool_tokens)
        self._no_tokens = torch.zeros(1, dtype=torch.int32, device=self.device)

    def ensure_room(self, n: int) -> None:
        if self.length + n > self.pool_tokens:
            self._alloc(2 * (self.length + n))

    def c_cache(self):
        """pkv_cache view with s = current length (keys read from the pool + planes)."""
        return _lib.Cache(self.k_pool.data_ptr(), self.v_pool.data_ptr(), self.pool_tokens, self.pages.data_ptr(),
                          self.length, self._no_tokens.data_ptr(), self.rcos.data_ptr(), self.rsin.data_ptr(),
                          self.rope_len, None, self.k2_pool.data_ptr(), None,
                          self.rcs32.data_ptr())

    @classmethod
    def from_assembled(cls, cache, length: int) -> "DevicePools":
        """Adopt a finalized AssembledCache's pools (context + query already appended)."""
        p = cls.__new__(cls)
        p.config, p.device = cache.config, cache.device
        p.k_pool, p.v_pool, p.k2_pool = cache.k_pool, cache.v_pool, cache.k2_pool
        p.pool_tokens, p.pages = cache.pool_tokens, cache._d_pages
        p.rope_len, p.rcos, p.rsin, p.rcs32 = cache.rope_len, cache._rcos, cache._rsin, cache._rcs32
        p._no_tokens = cache._d_tokens
        p.length = length
        return p

    @classmethod
    def from_host(cls, config: ModelConfig, keys, values, device) -> "DevicePools":
        """Upload host per-layer f32 [n][Hkv][dk] K/V (rotated keys) with exact key planes."""
        torch = _lib.require_cuda()
        n = int(np.asarray(keys[0]).shape[0])
        p = cls(config, device, n + QUERY_RESERVE)
        p.length = n
        idx = torch.arange(n, dtype=torch.int32, device=device)
        lib = _lib.load()
        cfg_c = config.c_struct()
        c = p.c_cache()
        for li in range(config.n_layers):
            tk = torch.from_numpy(np.ascontiguousarray(keys[li], dtype=np.float32)).to(device)
            tv = torch.from_numpy(np.ascontiguousarray(values[li], dtype=np.float32)).to(device)
            _lib.check(lib.pkv_replace_entries(ctypes_ref(cfg_c), ctypes_ref(c), li, idx.data_ptr(), n,
                                               tk.data_ptr(), tv.data_ptr(), _lib.stream_ptr(torch)))
        return p

    def host_layers(self, is_key: bool):
        """Per-layer f32 [length][Hkv][dk]: keys k + k2 (f32 to 2^-22), values from fp16."""
        dk = self.config.head_dim
        n = self.length
        if is_key:
            t = self.k_pool[:, :, :n, :dk].float() + self.k2_pool[:, :, :n, :dk].float()
        else:
            t = self.v_pool[:, :, :n, :dk].float()
        a = t.permute(0, 2, 1, 3).cpu().numpy()
        return [np.ascontiguousarray(a[li]) for li in range(self.config.n_layers)]


def _device_kv(weights, config: ModelConfig, cache: KVCache, dm) -> DevicePools:
    dev = getattr(cache, "_device_pools", None)
    if dev is None:
        dev = DevicePools.from_host(config, cache.keys, cache.values, dm.device)
        cache._device_pools = dev
    return dev


def _rebind_views(cache: KVCache, pools: DevicePools) -> None:
    cache._keys = lambda: pools.host_layers(True)
    cache._values = lambda: pools.host_layers(False)


def _decode_one(dm, config: ModelConfig, pools: DevicePools, token: int, tally: FlopTally | None):
    torch = _lib.require_cuda()
    ids = check_tokens([token], config)
    pools.ensure_room(1)
    logits = torch.empty(config.vocab_size, dtype=torch.float32, device=pools.device)
    d_ids = torch.from_numpy(ids.astype(np.int32)).to(pools.device)
    lib = _lib.load()
    flags = _lib.PKV_QP_LOGITS | _lib.PKV_QP_APPEND_KV
    nbytes = lib.pkv_query_pass_workspace(dm.handle, pools.length, 1, flags)
    ws = workspace(nbytes, "decode")
    c = pools.c_cache()
    _lib.check(lib.pkv_query_pass(dm.handle, ctypes_ref(c), None, d_ids.data_ptr(), 1, flags, None, None, None,
                                  logits.data_ptr(), ws.data_ptr(), ws.numel(), _lib.stream_ptr(torch)))
    bill_query_pass(tally, config, pools.length, 1)
    pools.length += 1
    return logits.cpu().numpy()


def decode_step(weights, config: ModelConfig, cache: KVCache, token: int, position: int,
                tally: FlopTally | None = None):
    """Append one token and return the next-token logits (reference model.py:431-441).
    Preconditions are checked before any mutation."""
    check_tokens([token], config)
    if position != cache.length:
        raise StateError(f"decode position {position} != cache length {cache.length}")
    dm = resolve_device_model(weights, config)
    pools = _device_kv(weights, config, cache, dm)
    logits = _decode_one(dm, config, pools, int(token), tally)
    cache.positions = np.concatenate([cache.positions, np.array([position], dtype=np.int64)])
    cache.last_logits = logits
    _rebind_views(cache, pools)
    return logits, cache


def greedy_generate(weights, config: ModelConfig, cache: KVCache, max_new_tokens: int, stop_ids=(),
                    include_stop: bool = False, capture_attn: bool = False,
                    tally: FlopTally | None = None) -> GenerationResult:
    """Argmax decoding from a finalized cache; ties go to the smaller token id
    (reference model.py:444-471)."""
    if cache.last_logits is None:
        raise StateError("cache has no pending logits; finalize or prefill first")
    if capture_attn:
        from .errors import ConfigError
        raise ConfigError("attention capture is not available on the B200 path")
    dm = resolve_device_model(weights, config)
    stop = set(int(s) for s in stop_ids)
    out: list = []
    logits = cache.last_logits
    pools = None
    for _ in range(max_new_tokens):
        nxt = int(np.argmax(logits))
        if nxt in stop:
            if include_stop:
                out.append(nxt)
            break
        out.append(nxt)
        if pools is None:
            pools = _device_kv(weights, config, cache, dm)
        logits = _decode_one(dm, config, pools, nxt, tally)
        cache.positions = np.concatenate([cache.positions, np.array([cache.length], dtype=np.int64)])
        cache.last_logits = logits
    if pools is not None:
        _rebind_views(cache, pools)
    return GenerationResult(tokens=out, step_attn=None)
