"""Full prefill on the device: the reference's ground-truth forward
``full_prefill`` (model.py:332-359) and the chunk producer ``precompute_chunk``
(chunkstore.py:52-62), both as the Stage-II kernels with every position selected.

``precompute_chunk`` leaves the chunk's unrotated keys and values in the device
chunk-store layout (bf16 ``[L][t][Hkv][dkp]``, include/pkv.h), captured inside the QKV
GEMM epilogue, so a freshly produced chunk is assembled without a host round trip; the
reference's f32 ``keys_norope``/``values`` are materialised lazily on access.
Numerics are the Stage-II contract (fp16 operands, fp32 accumulation and residual).
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np

from . import _lib
from .chunkstore import PAGE, ChunkKV, chunk_content_id, ctypes_ref, rope_device_tables
from .errors import ConfigError
from .model import FlopTally, ModelConfig, bill_query_pass, resolve_device_model
from .selection import check_tokens


@dataclass
class PrefillTrace:
    """Reference model.PrefillTrace (model.py:195-205)."""

    tokens: np.ndarray
    positions: np.ndarray
    keys: list                     # per layer [n, n_kv, d_k] f32, rotated
    values: list                   # per layer [n, n_kv, d_k] f32
    logits: np.ndarray             # [n, vocab]
    keys_norope: list | None = None
    attn: list | None = None
    attn_heads: list | None = None


class _SequenceCache:
    """Device pools + RoPE tables for one token sequence at positions 0..n-1."""

    def __init__(self, cfg: ModelConfig, ids: np.ndarray, dev):
        torch = _lib.require_cuda()
        lay = cfg.layout()
        n = int(ids.shape[0])
        self.n = n
        self.pool_tokens = -(-n // PAGE) * PAGE
        shape = (cfg.n_layers, cfg.n_kv_heads, self.pool_tokens, lay.dkp)
        self.k_pool = torch.zeros(shape, dtype=torch.float16, device=dev)
        self.v_pool = torch.zeros_like(self.k_pool)
        self.k2_pool = torch.zeros_like(self.k_pool)  # keys' residual plane: k_pool + k2 = f32 key
        self.pages = torch.arange(self.pool_tokens // PAGE, dtype=torch.int32, device=dev)
        self.tokens = torch.from_numpy(ids.astype(np.int32)).to(dev)
        self.rope_len, self.rcos, self.rsin, self.rcs32 = rope_device_tables(cfg.rope_theta, cfg.head_dim,
                                                                            self.pool_tokens)
        self.c = _lib.Cache(self.k_pool.data_ptr(), self.v_pool.data_ptr(), self.pool_tokens, self.pages.data_ptr(), n,
                            self.tokens.data_ptr(), self.rcos.data_ptr(), self.rsin.data_ptr(), self.rope_len, None,
                            self.k2_pool.data_ptr(), None, self.rcs32.data_ptr())

    def layer(self, pool, li: int, dk: int, plane=None) -> np.ndarray:
        """[n, Hkv, dk] f32 of one layer (pages are in order), plus a residual plane."""
        t = pool[li, :, : self.n, :dk].float()
        if plane is not None:
            t = t + plane[li, :, : self.n, :dk].float()
        return t.permute(1, 0, 2).cpu().numpy()


def _run(dm, cfg: ModelConfig, ids: np.ndarray, want_knr: bool, want_logits: bool, stream=None):
    torch = _lib.require_cuda()
    if dm.tp_world != 1:
        raise ConfigError("full prefill runs on an unsharded model")
    dev = dm.device
    seq = _SequenceCache(cfg, ids, dev)
    lay = cfg.layout()
    n, L, Hkv = seq.n, cfg.n_layers, cfg.n_kv_heads
    knr = v = logits = None
    if want_knr:
        knr = torch.zeros((L, n, Hkv, lay.dkp), dtype=torch.bfloat16, device=dev)
        v = torch.zeros_like(knr)
    if want_logits:
        logits = torch.empty((n, cfg.vocab_size), dtype=torch.float32, device=dev)
    lib = _lib.load()
    ws = torch.empty(lib.pkv_full_prefill_workspace(dm.handle, n), dtype=torch.uint8, device=dev)

    def ptr(t):
        return t.data_ptr() if t is not None else None

    _lib.check(lib.pkv_full_prefill(dm.handle, ctypes_ref(seq.c), ptr(knr), ptr(v), ptr(logits), ws.data_ptr(),
                                    ws.numel(), _lib.stream_ptr(torch, stream)))
    return seq, knr, v, logits


def full_prefill(weights, config: ModelConfig, tokens, capture_attn: bool = False, capture_attn_heads: bool = False,
                 capture_keys_norope: bool = False, tally: FlopTally | None = None) -> PrefillTrace:
    """Forward pass over the whole sequence at positions 0..n-1 (reference
    model.py:332-359) on the Stage-II kernels."""
    if capture_attn or capture_attn_heads:
        # attention-row capture is the reference's measurement apparatus (metrics.py),
        # not on the TTFT path
        raise ConfigError("attention capture is not available on the B200 path")
    dm = resolve_device_model(weights, config)
    ids = check_tokens(tokens, config)
    seq, knr, v, logits = _run(dm, config, ids, capture_keys_norope, True)
    dk = config.head_dim
    keys = [seq.layer(seq.k_pool, li, dk, seq.k2_pool) for li in range(config.n_layers)]
    values = [seq.layer(seq.v_pool, li, dk) for li in range(config.n_layers)]
    keys_nr = None
    if knr is not None:
        a = knr[..., :dk].float().cpu().numpy()
        keys_nr = [np.ascontiguousarray(a[li]) for li in range(config.n_layers)]
    bill_query_pass(tally, config, 0, int(ids.shape[0]), with_logits=True)
    return PrefillTrace(tokens=ids, positions=np.arange(ids.shape[0], dtype=np.int64), keys=keys, values=values,
                        logits=logits.cpu().numpy(), keys_norope=keys_nr)


def precompute_chunk(weights, config: ModelConfig, tokens) -> ChunkKV:
    """Isolated prefill of one chunk, keys stored before any rotation (reference
    chunkstore.py:52-62); the K/V stay on the device in the chunk-store layout."""
    dm = resolve_device_model(weights, config)
    ids = check_tokens(tokens, config)
    _, knr, v, _ = _run(dm, config, ids, True, False)
    fp = dm.fingerprint  # == weights.fingerprint(config) for host weights (set at upload)
    return ChunkKV.from_device(chunk_content_id(fp, ids), fp, ids, knr, v, config.head_dim)


def precompute_chunks_device(dm, config: ModelConfig, token_lists, fingerprint: str | None = None) -> list:
    """Batch of chunks from a DeviceModel (bench / serving helper)."""
    fp = fingerprint or dm.fingerprint
    out = []
    for toks in token_lists:
        ids = check_tokens(toks, config)
        _, knr, v, _ = _run(dm, config, ids, True, False)
        out.append(ChunkKV.from_device(chunk_content_id(fp, ids), fp, ids, knr, v, config.head_dim))
    return out
